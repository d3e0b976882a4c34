"""Multi-GPU plumbing on CPU (gloo, world size 2): the view partition and the in-place exchange
of all-view buffers that pipeline.HotPath runs over NCCL after SLIC and after every refine
iteration.  Each rank fills only its own views; after the exchange every rank must hold the
same complete buffer, for equal (all-gather) and unequal (broadcast) partitions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1812_06856_b200.pipeline import exchange_views, partition


def test_partition_covers_views_once():
    for V in (1, 2, 5, 16, 25, 64):
        for world in (1, 2, 3, 4, 8):
            owned = []
            for r in range(world):
                v0, n = partition(V, world, r)
                owned += list(range(v0, v0 + n))
            assert owned == list(range(V))
            sizes = [partition(V, world, r)[1] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, V, stride, allgather, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        buf = torch.zeros(V * stride, dtype=torch.uint8)
        v0, n = partition(V, world, rank)
        for v in range(v0, v0 + n):  # "compute" own views: deterministic content per view
            g = np.random.default_rng(v).integers(0, 255, stride, dtype=np.uint8)
            buf[v * stride:(v + 1) * stride] = torch.from_numpy(g)
        exchange_views(buf, stride, V, world, rank, in_place_allgather=allgather)
        q.put((rank, buf.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("V,allgather", [(4, True), (5, False), (4, False)])
def test_exchange_views_gloo_world2(V, allgather):
    world, stride = 2, 96
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, V, stride, allgather, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.concatenate([np.random.default_rng(v).integers(0, 255, stride, dtype=np.uint8) for v in range(V)])
    for r in range(world):
        assert np.array_equal(out[r], want), f"rank {r} buffer incomplete"
