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
