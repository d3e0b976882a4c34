"""Full-size parity at the bench workload (C3: 16 x 1920x1080, S=16, L=256, N=15, 5 iterations;
SURVEY.md §8d), nothing sampled:

* SLIC: label maps, records and member lists of all 16 views equal the reference's
  slic_segment (superpixel.hpp:179);
* sweep: all 16 x 8160 winning depths equal the reference's sweep_view output, bit for bit
  (tests/golden/c3_init_depths.npz, produced by the unmodified reference, make_c3_init.py);
* refinement, lockstep per iteration from the GPU's own evolving state: for l = 1..5 the GPU's
  planes and depth rasters are loaded into the reference, the reference's stock refine_iteration
  (refine.hpp:253-323, all 130,560 tasks, with RefineStats) runs on them, and every plane, the
  accepted count and the violation count must equal the GPU's refine_iteration; rasterize
  (sweep.hpp:44) of every view is compared on the way.  The GPU then continues from its own state.
"""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIXTURE = os.path.join(ROOT, "tests", "golden", "c3_init_depths.npz")


@pytest.fixture(scope="module")
def c3():
    from paper_1812_06856_b200 import api, scenes

    sc = scenes.render_config("C3", gt=False)
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], sc["cams"], sc["range"])
    dc.slic_views(0, 16, api.SlicParams(16, 0.1, 10))
    dc.sweep_views(0, 16, api.SweepParams(256, 0.05, 0), 0)
    dc.rasterize()
    return sc, dc


def test_sweep_matches_reference_fixture(c3):
    sc, dc = c3
    want = np.load(FIXTURE)["depths"]
    for v in range(16):
        got = dc.get_planes(v)
        assert np.array_equal(got[:, 0], want[v]), f"view {v}: {np.sum(got[:, 0] != want[v])} depths differ"
        assert np.all(got[:, 1:] == np.array([0.0, 0.0, -1.0]))


@pytest.fixture(scope="module")
def ref_c3(ref, c3):
    sc, dc = c3
    rs = ref.Session(sc["lab"], sc["cams"], sc["range"])
    workers = len(os.sched_getaffinity(0))
    for v in range(16):
        rs.slic(v, 16, 0.1, 10, workers)
    return rs, workers


def test_slic_full_size_all_views(ref_c3, c3):
    rs, _ = ref_c3
    sc, dc = c3
    for v in range(16):
        want, got = rs.grid(v), dc.get_grid(v)
        assert np.array_equal(got.label_map, want["labels"]), f"labels of view {v}"
        assert np.array_equal(got.offsets, want["offsets"]) and np.array_equal(got.members, want["members"])
        for k_got, k_want in (("cx", "cx"), ("cy", "cy"), ("mean_color", "color"), ("pixel_count", "count")):
            assert np.array_equal(got.sp[k_got], want["records"][k_want]), f"{k_got} of view {v}"


def test_refine_full_lockstep_all_iterations(ref_c3, c3):
    from paper_1812_06856_b200 import api

    rs, workers = ref_c3
    sc, dc = c3
    dc.make_refine_context(api.EnergyParams(iterations=5), 256)
    rs_ctx = False
    for l in range(1, 6):
        for v in range(16):
            rs.set_planes(v, dc.get_planes(v))
        rs.rasterize()
        for v in range(16):
            assert np.array_equal(rs.depth(v).view(np.uint32), dc.get_depth(v).view(np.uint32)), \
                f"rasterized depth of view {v} before iteration {l}"
        if not rs_ctx:
            rs.refine_context(256, iterations=5)
            rs_ctx = True
        acc_r, vio_r = rs.refine_iteration(l, workers, with_stats=True)
        acc_g, vio_g = dc.refine_iteration(l, with_stats=True)
        ndiff = 0
        for v in range(16):
            bad = np.any(dc.get_planes(v) != rs.planes(v), axis=1)
            ndiff += int(bad.sum())
        assert ndiff == 0, f"iteration {l}: {ndiff} of 130560 planes differ"
        assert (acc_g, vio_g) == (acc_r, vio_r), f"RefineStats of iteration {l}: GPU {(acc_g, vio_g)} ref {(acc_r, vio_r)}"
        dc.rasterize()
