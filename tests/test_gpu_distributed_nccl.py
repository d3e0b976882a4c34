"""The multi-GPU exchange mechanics on one B200: a 1-rank NCCL process group runs the in-place
all-gather on the library's own device buffers (zero-copy tensors over lfdg_device_buffer) —
the code path HotPath uses per refine iteration at N > 1 — and the full HotPath run under the
group equals the single-process run bit for bit."""
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


def test_nccl_inplace_allgather_on_device_buffers():
    import torch
    import torch.distributed as dist

    from paper_1812_06856_b200 import _native as N
    from paper_1812_06856_b200 import api, scenes
    from paper_1812_06856_b200.pipeline import HotPath, HotPathConfig

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        sc = scenes.render_scene("cluttered", 4, 160, 120, 160.0, 0.1)
        cfg = HotPathConfig(api.SlicParams(12, 0.1, 10), api.SweepParams(16, 0.05, 0),
                            api.EnergyParams(iterations=2), 0)
        ref = HotPath(0, sc["lab"], sc["cams"], sc["range"], cfg)
        ref.run()
        want = [ref.ctx.get_planes(v) for v in range(4)]
        hp = HotPath(0, sc["lab"], sc["cams"], sc["range"], cfg, group=dist.group.WORLD)
        hp.run()
        # force the exchange path (a no-op for one rank) through NCCL on every buffer kind
        for which in (N.BUF_LABELS, N.BUF_CX, N.BUF_COLOR, N.BUF_MOFF, N.BUF_MPIX, N.BUF_CRAY, N.BUF_PLANES):
            t, stride = hp._tensor(which)
            before = t.clone()
            dist.all_gather_into_tensor(t, t[0:stride * 4])
            torch.cuda.synchronize()
            assert torch.equal(t, before)
        for v in range(4):
            assert np.array_equal(hp.ctx.get_planes(v), want[v])
    finally:
        dist.destroy_process_group()
