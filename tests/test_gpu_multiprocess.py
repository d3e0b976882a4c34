"""Process-level analogue of acceptance criterion 8 (tests/acceptance.cpp:435-468: 1 vs 8
workers byte-identical) for the multi-GPU path: two processes, each a HotPath rank on the one
B200 of the test box with a gloo process group (the device buffers are staged through the host
by pipeline.exchange_views; on a multi-GPU node the same code runs over NCCL in place).  Each
rank segments, sweeps and refines only its own views and exchanges grids and planes; every rank
must end with the single-process planes and depth rasters bit for bit, and the ranks' accepted
counts must add up to the single-process count.  Both partitions: equal blocks (all-gather) and
unequal blocks (per-owner broadcast).  The ranks never wait on one another inside a kernel."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    from paper_1812_06856_b200 import api
    from paper_1812_06856_b200.pipeline import HotPathConfig

    return HotPathConfig(api.SlicParams(12, 0.1, 10), api.SweepParams(24, 0.05, 0), api.EnergyParams(iterations=3), 0)


def _scene(V):
    from paper_1812_06856_b200 import scenes

    return scenes.render_scene("cluttered", V, 240, 180, 240.0, 0.08)


def _rank(rank, world, port, V, q):
    import torch.distributed as dist

    from paper_1812_06856_b200.pipeline import HotPath

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = _scene(V)
        hp = HotPath(0, sc["lab"], sc["cams"], sc["range"], _cfg(), group=dist.group.WORLD)
        r = hp.run(with_stats=True)
        planes = np.stack([hp.ctx.get_planes(v) for v in range(V)])
        depth = np.stack([hp.ctx.get_depth(v) for v in range(V)])
        q.put((rank, r["accepted"], (hp.v0, hp.n), planes, depth))
        hp.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("V", [4, 5])
def test_two_ranks_equal_single_process(V):
    import torch.multiprocessing as mp

    from paper_1812_06856_b200.pipeline import HotPath

    sc = _scene(V)
    single = HotPath(0, sc["lab"], sc["cams"], sc["range"], _cfg(), use_torch_stream=False)
    acc_single = single.run(with_stats=True)["accepted"]
    want_p = np.stack([single.ctx.get_planes(v) for v in range(V)])
    want_d = np.stack([single.ctx.get_depth(v) for v in range(V)])
    single.close()

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, V, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    owned = sorted(o[2] for o in out)
    assert owned[0][0] == 0 and owned[0][1] + owned[1][1] == V and owned[1][0] == owned[0][1]
    for rank, acc, _, planes, depth in out:
        assert np.array_equal(planes.view(np.uint64), want_p.view(np.uint64)), f"rank {rank} planes"
        assert np.array_equal(depth.view(np.uint32), want_d.view(np.uint32)), f"rank {rank} depth"
    assert sum(o[1] for o in out) == acc_single
