"""GPU sRGB -> scaled LAB (rgb_to_scaled_lab, image.hpp:97-107) against
the reference: the GPU conversion of rendered scenes equals the LAB the reference renderer
produced, bit for bit, and random / edge colours equal the host port (which tests/test_lab_port.py
pins to glibc).  The fused upload path (lfdg_upload_rgb) lands the same LAB in the context."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gpu_lab_matches_reference_render(ref):
    from paper_1812_06856_b200 import api

    sc = ref.render_scene("cluttered", 2, 320, 240, 320.0, 0.1)
    got = api.rgb_to_scaled_lab(sc["rgb"])
    assert np.array_equal(got.view(np.uint32), sc["lab"].view(np.uint32))


def test_gpu_lab_random_and_edges():
    from paper_1812_06856_b200 import _native as N, api

    rng = np.random.default_rng(3)
    rgb = rng.uniform(-0.05, 1.2, (1 << 20, 3)).astype(np.float32)
    edges = np.array([0.0, 0.04045, np.nextafter(np.float32(0.04045), np.float32(1)), 1.0, 1e-30, 0.5, 2.0, 1e20],
                     np.float32)
    rgb[: len(edges) ** 3] = np.stack(np.meshgrid(edges, edges, edges), -1).reshape(-1, 3)
    want = np.empty_like(rgb)
    N.check(N.lib().lfdg_rgb_to_scaled_lab(rgb.shape[0], N.ptr(rgb), N.ptr(want)))  # host port (scene.cpp)
    got = api.rgb_to_scaled_lab(rgb)
    same = (got.view(np.uint32) == want.view(np.uint32)) | (np.isnan(got) & np.isnan(want))
    assert same.all(), f"{(~same).any(axis=1).sum()} pixels differ"


def test_upload_rgb_lands_reference_lab(ref):
    from paper_1812_06856_b200 import api

    sc = ref.render_scene("cluttered", 3, 160, 120, 160.0, 0.1)
    dc = api.DeviceContext(0)
    dc.set_views(np.zeros_like(sc["lab"]), sc["cams"], sc["range"])
    dc.upload_rgb(sc["rgb"])
    rs = ref.Session(sc["lab"], sc["cams"], sc["range"])
    for v in range(3):
        rs.slic(v, 12, 0.1, 10)
        dc.slic(v, api.SlicParams(12, 0.1, 10))
        assert np.array_equal(dc.get_grid(v).label_map, rs.grid(v)["labels"])


def _device_lab(dc):
    import torch

    from paper_1812_06856_b200 import _native as N
    from paper_1812_06856_b200.pipeline import _CudaArray

    ptr, nbytes, _ = dc.device_buffer(N.BUF_LAB)
    t = torch.as_tensor(_CudaArray(ptr, nbytes), device="cuda:0")
    return t.cpu().numpy().view(np.float32).reshape(-1, 4)


def test_upload_rgb8_every_colour_equals_float_path():
    """lfdg_upload_rgb8 on all 2^24 8-bit colours (one 4096x4096 view) lands exactly the LAB that
    lfdg_upload_rgb produces from byte / 255.f (read_image, io.hpp:136-146), which the tests above
    pin to the reference; the w lane is 0."""
    from paper_1812_06856_b200 import api

    c = np.arange(1 << 24, dtype=np.uint32)
    rgb8 = np.stack([(c >> 16) & 255, (c >> 8) & 255, c & 255], -1).astype(np.uint8).reshape(1, 4096, 4096, 3)
    cams = np.zeros((1, 21))
    cams[0, [0, 4, 8]] = 1.0
    cams[0, [9, 13, 17]] = 1.0
    dc8, dcf = api.DeviceContext(0), api.DeviceContext(0)
    for dc in (dc8, dcf):
        dc.set_views(np.zeros((1, 4096, 4096, 3), np.float32), cams, (1.0, 2.0))
    dc8.upload_rgb8(rgb8)
    dcf.upload_rgb(rgb8.astype(np.float32) / np.float32(255.0))
    a, b = _device_lab(dc8), _device_lab(dcf)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert (a[:, 3] == 0).all()
    dc8.close()
    dcf.close()
