"""The view partition of HotPath at world sizes 2, 3 and 4, emulated in one process on one GPU:
each "rank" is its own DeviceContext (own device buffers) that runs only its block of views
(pipeline.partition), and the exchange after SLIC (GRID_BUFFERS), after the sweep and after every
refine iteration (planes) is done as device-to-device copies of the owners' blocks into every
other rank's buffers — the bytes an NCCL all-gather / broadcast would deliver.  The ranks run one
after another (no kernel waits on another rank), so this is safe on one GPU.  Every rank must end
with the single-context result bit for bit (Jacobi updates + deterministic rasterize), and the
accepted counts summed over ranks must equal the single-context count."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 4])
def test_partitioned_run_equals_single(world):
    import torch

    from paper_1812_06856_b200 import _native as N
    from paper_1812_06856_b200 import api, scenes
    from paper_1812_06856_b200.pipeline import GRID_BUFFERS, HotPath, HotPathConfig, partition

    V = 5
    sc = scenes.render_scene("cluttered", V, 160, 120, 160.0, 0.1)
    cfg = HotPathConfig(api.SlicParams(12, 0.1, 10), api.SweepParams(24, 0.05, 0), api.EnergyParams(iterations=3), 7)

    single = HotPath(0, sc["lab"], sc["cams"], sc["range"], cfg, use_torch_stream=False)
    acc_single = single.run(with_stats=True)["accepted"]
    want = [single.ctx.get_planes(v) for v in range(V)]
    want_depth = [single.ctx.get_depth(v) for v in range(V)]

    ranks = [HotPath(0, sc["lab"], sc["cams"], sc["range"], cfg, use_torch_stream=False) for _ in range(world)]
    for r, hp in enumerate(ranks):
        hp.world, hp.rank = world, r
        hp.v0, hp.n = partition(V, world, r)

    def exchange(which):
        torch.cuda.synchronize()
        for r, owner in enumerate(ranks):
            src, stride = owner._tensor(which)
            lo, hi = owner.v0 * stride, (owner.v0 + owner.n) * stride
            for q, other in enumerate(ranks):
                if q != r and owner.n:
                    dst, _ = other._tensor(which)
                    dst[lo:hi].copy_(src[lo:hi])
        torch.cuda.synchronize()

    for hp in ranks:
        hp.ctx.slic_views(hp.v0, hp.n, cfg.slic)
    for which in GRID_BUFFERS:
        exchange(which)
    for hp in ranks:
        hp.ctx.mark_views_ready(0, V, 1)
        hp.ctx.sweep_views(hp.v0, hp.n, cfg.sweep, cfg.seed)
    exchange(N.BUF_PLANES)
    for hp in ranks:
        hp.ctx.mark_views_ready(0, V, 2)
        hp.ctx.rasterize()
        hp.ctx.make_refine_context(cfg.energy, cfg.sweep.levels)
        hp.ctx.set_refine_views(hp.v0, hp.n)
    acc = 0
    for l in range(1, cfg.energy.iterations + 1):
        for hp in ranks:
            acc += hp.ctx.refine_iteration(l, with_stats=True)[0]
        exchange(N.BUF_PLANES)
        for hp in ranks:
            hp.ctx.mark_views_ready(0, V, 2)
            hp.ctx.rasterize()
    assert acc == acc_single
    for r, hp in enumerate(ranks):
        for v in range(V):
            assert np.array_equal(hp.ctx.get_planes(v), want[v]), f"world {world} rank {r} view {v}"
            assert np.array_equal(hp.ctx.get_depth(v), want_depth[v]), f"world {world} rank {r} depth {v}"
