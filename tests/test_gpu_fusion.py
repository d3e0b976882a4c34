"""Stability fusion (fusion.hpp:31-100) on the GPU against the
reference: fuse_all of the refined C1 depth maps and gather_candidates' ordered lists, bit for
bit; stability_fuse on hand-made lists (tests/test_fusion.cpp's cases)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def refined_c1(ref):
    from paper_1812_06856_b200 import api

    g = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "c1_golden.npz"))
    sc = ref.render_scene("cluttered", 3, 320, 240, 320.0, 0.1)
    rs = ref.Session(sc["lab"], sc["cams"], sc["range"])
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], sc["cams"], sc["range"])
    for v in range(3):
        rs.slic(v, 12, 0.1, 10)
        dc.slic(v, api.SlicParams(12, 0.1, 10))
        rs.set_planes(v, g[f"refine3_{v}"])
        dc.set_planes(v, g[f"refine3_{v}"])
    rs.rasterize()
    dc.rasterize()
    step = (1.0 / sc["range"][0] - 1.0 / sc["range"][1]) / 31
    return rs, dc, step


def test_fuse_all_matches_reference(refined_c1):
    rs, dc, eps = refined_c1
    want = rs.fuse_all(eps)
    dc.fuse_views(eps)
    for v in range(3):
        got = dc.get_fused(v)
        assert np.array_equal(got.view(np.uint32), want[v].view(np.uint32)), f"view {v}"
        assert (got > 0).mean() > 0.5


def test_gather_candidates_order_matches_reference(refined_c1):
    rs, dc, _ = refined_c1
    for ref_view in (0, 2):
        o1, d1, v1 = rs.gather_candidates(ref_view)
        o2, d2, v2 = dc.gather_candidates(ref_view)
        assert np.array_equal(o1, o2)
        assert np.array_equal(d1.view(np.uint32), d2.view(np.uint32)) and np.array_equal(v1, v2)


def test_stability_fuse_hand_cases():
    from paper_1812_06856_b200 import api

    def one(lst, eps):
        off = np.array([0, len(lst)], np.int32)
        d = np.array([c[0] for c in lst], np.float32)
        v = np.array([c[1] for c in lst], np.int32)
        return api.stability_fuse(off, d, v, eps)[0]

    eps = 1.0 / 4.0 - 1.0 / 4.5  # tests/test_fusion.cpp:23-38 style cases
    assert one([(4.0, 0), (4.1, 1), (9.0, 2)], 0.02) == np.float32(4.0)
    assert one([(5.0, 0)], eps) == np.float32(5.0)
    assert one([], eps) == 0.0
    assert one([(2.0, 0), (9.0, 1)], 0.01) == 0.0
    assert one([(5.0, 2), (4.99, 0), (5.01, 1)], 0.01) == np.float32(4.99)
    with pytest.raises(api.InvariantError):
        one([], 0.0)
