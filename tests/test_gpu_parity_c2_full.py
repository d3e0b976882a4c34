"""Full-pipeline parity on C2 (8 x 1024x768 linear rig, S=12, L=128, N=7, 5 iterations;
SURVEY.md §8d), with no sampling: the GPU and the reference (oracle/_ref, all host cores) each run
the whole hot path from the same images —

  slic_segment of every view -> sweep_view of every view -> rasterize -> make_refine_context ->
  refine_iteration l = 1..5 (+ rasterize after each) -> fuse_all

— and every intermediate is compared bit for bit: label maps, every sweep winner, every depth
raster, the planes and RefineStats after every iteration, and the fused depth maps.  Unlike
test_gpu_parity_configs.py (sampled lockstep from the GPU's own state) the two runs never exchange
state, so any divergence anywhere would propagate to the end."""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c2_whole_pipeline(ref):
    from paper_1812_06856_b200 import api, scenes

    c = scenes.CONFIGS["C2"]
    sc = scenes.render_config("C2", gt=False)
    V = sc["lab"].shape[0]
    workers = len(os.sched_getaffinity(0))
    rs = ref.Session(sc["lab"], sc["cams"], sc["range"])
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], sc["cams"], sc["range"])

    sp = api.SlicParams(c["S"], 0.1, 10)
    dc.slic_views(0, V, sp)
    for v in range(V):
        rs.slic(v, c["S"], 0.1, 10, workers)
        assert np.array_equal(dc.get_grid(v).label_map, rs.grid(v)["labels"]), f"SLIC labels of view {v}"

    dc.sweep_views(0, V, api.SweepParams(c["levels"], 0.05, c["max_neighbors"]), 0)
    for v in range(V):
        want = rs.sweep(v, c["levels"], 0.05, c["max_neighbors"], 0, workers)
        got = dc.get_planes(v)
        bad = np.any(got != want, axis=1)
        assert not bad.any(), f"sweep view {v}: {bad.sum()} of {len(got)} winners differ"
        rs.set_planes(v, want)
    rs.rasterize()
    dc.rasterize()
    for v in range(V):
        assert np.array_equal(dc.get_depth(v), rs.depth(v)), f"sweep-init depth of view {v}"

    it = c["iterations"]
    rs.refine_context(c["levels"], iterations=it, max_neighbors=c["max_neighbors"])
    dc.make_refine_context(api.EnergyParams(iterations=it, max_neighbors=c["max_neighbors"]), c["levels"])
    for l in range(1, it + 1):
        acc_r, vio_r = rs.refine_iteration(l, workers, with_stats=True)
        acc_g, vio_g = dc.refine_iteration(l)
        rs.rasterize()
        dc.rasterize()
        assert (acc_g, vio_g) == (acc_r, vio_r), f"RefineStats of iteration {l}"
        for v in range(V):
            want, got = rs.planes(v), dc.get_planes(v)
            bad = np.any(got != want, axis=1)
            assert not bad.any(), f"iteration {l} view {v}: {bad.sum()} planes differ"
            assert np.array_equal(dc.get_depth(v), rs.depth(v)), f"depth of view {v} after iteration {l}"

    want = rs.fuse_all(0.05, workers)
    dc.fuse_views(0.05)
    for v in range(V):
        assert np.array_equal(dc.get_fused(v).view(np.uint32), want[v].view(np.uint32)), f"fused view {v}"
