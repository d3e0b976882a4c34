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


def test_serial_and_pipelined_uploads_mixed():
    """upload_images (serial, compute stream) and prefetch (copy stream) share the
    staging buffer.  prefetch(A) -> commit -> run -> upload(B) -> prefetch(C) -> commit must run
    B's step on B's images and C's step on C's; a serial upload while a prefetch is uncommitted is
    refused."""
    import torch

    from paper_1812_06856_b200 import _native as N, api, scenes
    from paper_1812_06856_b200.pipeline import HotPath, HotPathConfig, estimate_depth

    a = scenes.render_config("C1")
    sets = [a["lab"], scenes.render_scene("occluder", 3, 320, 240, 320.0, 0.1)["lab"],
            scenes.render_scene("staircase", 3, 320, 240, 320.0, 0.1)["lab"]]
    cfg = HotPathConfig(slic=api.SlicParams(12, 0.1, 10), sweep=api.SweepParams(32, 0.05, 0),
                        energy=api.EnergyParams(iterations=2), seed=0)
    want = [estimate_depth(x, a["cams"], a["range"], cfg) for x in sets]
    hp = HotPath(0, a["lab"], a["cams"], a["range"], cfg, use_torch_stream=False)
    pins = []
    for x in sets:
        p = torch.empty(x.size, dtype=torch.float32, pin_memory=True).numpy().reshape(x.shape)
        p[...] = x
        pins.append(p)
    nsp = 27 * 20
    got = []

    def step():
        hp.run()
        pl = np.zeros((3, nsp, 4), np.float64)
        dp = np.zeros((3, 240, 320), np.float32)
        hp.download(pl, dp, sync=True)
        got.append((pl, dp))

    hp.prefetch(pins[0])
    hp.commit()
    step()
    hp.upload(pins[1])   # serial repack from the staging buffer ...
    hp.prefetch(pins[2])  # ... immediately followed by a prefetch into the same buffer
    with pytest.raises(api.StateError):
        hp.upload(pins[1])  # refused while C is staged
    # B's images are installed; C waits in the staging buffer until commit
    step()
    hp.commit()
    step()
    hp.close()
    for k, (pl, dp) in enumerate(got):
        wp, wd = want[k]
        assert np.array_equal(pl.view(np.uint64), np.stack(wp).view(np.uint64)), f"set {k} planes"
        assert np.array_equal(dp.view(np.uint32), wd.view(np.uint32)), f"set {k} depth"


def test_wrong_shapes_raise_before_the_abi():
    from paper_1812_06856_b200 import api, scenes
    from paper_1812_06856_b200.pipeline import HotPath, HotPathConfig

    a = scenes.render_config("C1")
    dc = api.DeviceContext(0)
    with pytest.raises(api.InvalidParams):
        dc.set_views(a["lab"], a["cams"][:2], a["range"])  # fewer cameras than views
    with pytest.raises(api.InvalidParams):
        dc.set_views(a["lab"][..., 0], a["cams"], a["range"])  # [V][H][W]
    dc.set_views(a["lab"], a["cams"], a["range"])
    with pytest.raises(api.InvalidParams):
        dc.update_images(0, np.zeros((1, 240, 320, 4), np.float32))
    with pytest.raises(api.InvalidParams):
        dc.update_images(0, np.zeros((1, 120, 320, 3), np.float32))
    with pytest.raises(api.InvalidParams):
        dc.upload_rgb(np.zeros((4, 240, 320, 3), np.float32))  # more views than the context holds
    with pytest.raises(api.InvalidParams):
        dc.upload_rgb8(np.zeros((1, 240, 321, 3), np.uint8))
    dc.close()
    hp = HotPath(0, a["lab"], a["cams"], a["range"], HotPathConfig(), use_torch_stream=False)
    with pytest.raises(api.InvalidParams):
        hp.prefetch(a["lab"][:2])
    with pytest.raises(api.InvalidParams):
        hp.upload(np.zeros((3, 240, 320, 4), np.float32))
    hp.close()


def test_views_of_2_31_pixels_rejected_by_the_abi():
    """Pixel indices are 32-bit: lfdg_set_views rejects a view of 2^31 pixels or more before it
    reads the images (a one-pixel buffer stands in for them)."""
    import ctypes as C

    from paper_1812_06856_b200 import _native as N, api

    dc = api.DeviceContext(0)
    L = N.lib()
    one = np.zeros(3, np.float32)
    cams = (N.Camera * 1)()
    rc = L.lfdg_set_views(dc.h, 1, 1 << 16, 1 << 15, N.ptr(one), C.cast(cams, C.c_void_p), 1.0, 2.0)
    assert rc == N.LFDG_INVALID_PARAMS
    assert b"2^31" in L.lfdg_last_error()
    dc.close()
