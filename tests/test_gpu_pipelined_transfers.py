"""Pipelined end-to-end transfers (lfdg_prefetch_images / lfdg_commit_images /
lfdg_download_results_async / lfdg_wait_downloads): two different view sets streamed through
one context with the next upload and the previous download overlapping the compute give exactly
the results of two separate one-shot runs (estimate_depth), and the reference's C1 golden."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_streamed_view_sets_equal_separate_runs():
    import torch

    from paper_1812_06856_b200 import api, scenes
    from paper_1812_06856_b200.pipeline import HotPath, HotPathConfig, estimate_depth

    a = scenes.render_config("C1")
    b = scenes.render_scene("occluder", 3, 320, 240, 320.0, 0.1)
    b_lab = b["lab"]  # a different image set under C1's cameras and range
    cfg = HotPathConfig(slic=api.SlicParams(12, 0.1, 10), sweep=api.SweepParams(32, 0.05, 0),
                        energy=api.EnergyParams(iterations=3), seed=0)
    want = [estimate_depth(x, a["cams"], a["range"], cfg) for x in (a["lab"], b_lab)]

    hp = HotPath(0, a["lab"], a["cams"], a["range"], cfg, use_torch_stream=False)
    nsp = 27 * 20
    pins = [torch.empty(x.size, dtype=torch.float32, pin_memory=True).numpy().reshape(x.shape) for x in (a["lab"], b_lab)]
    pins[0][...] = a["lab"]
    pins[1][...] = b_lab
    planes = [torch.empty(3 * nsp * 4, dtype=torch.float64, pin_memory=True).numpy().reshape(3, nsp, 4) for _ in range(2)]
    depth = [torch.empty(3 * 240 * 320, dtype=torch.float32, pin_memory=True).numpy().reshape(3, 240, 320)
             for _ in range(2)]
    hp.prefetch(pins[0])
    for k in range(2):
        hp.commit()
        if k == 0:
            hp.prefetch(pins[1])
        hp.run()
        hp.download_async(planes[k], depth[k])
    hp.wait_downloads()
    hp.ctx.synchronize()
    hp.close()
    for k in range(2):
        wp, wd = want[k]
        assert np.array_equal(planes[k].view(np.uint64), np.stack(wp).view(np.uint64)), f"set {k} planes"
        assert np.array_equal(depth[k].view(np.uint32), wd.view(np.uint32)), f"set {k} depth"
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1_golden.npz"))
    for v in range(3):
        assert np.array_equal(planes[0][v].view(np.uint64), g[f"refine3_{v}"].view(np.uint64))


def test_commit_without_prefetch_is_a_state_error():
    from paper_1812_06856_b200 import _native as N, api, scenes

    a = scenes.render_config("C1")
    dc = api.DeviceContext(0)
    dc.set_views(a["lab"], a["cams"], a["range"])
    assert N.lib().lfdg_commit_images(dc.h) == N.LFDG_STATE
    lab = np.ascontiguousarray(a["lab"])
    N.check(N.lib().lfdg_prefetch_images(dc.h, 0, 3, N.ptr(lab)))
    assert N.lib().lfdg_prefetch_images(dc.h, 0, 3, N.ptr(lab)) == N.LFDG_STATE  # still uncommitted
    N.check(N.lib().lfdg_commit_images(dc.h))
    dc.synchronize()
    dc.close()
