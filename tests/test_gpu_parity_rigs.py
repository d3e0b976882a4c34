"""GPU parity on camera rigs that exercise every specialisation of the kernels:

* ``grid``    2x2 grid rig (make_grid_rig): kFlat with target rows that vary per target (row_inv = 0);
* ``tz``      identity rotations, canonical K, cameras at different depths: kIdR + kCanonK, not kFlat;
* ``rot``     small per-view rotations, canonical K: the general-R paths;
* ``skew``    identity rotations, K01 != 0: the general-K paths (rays depend on both coordinates);
* ``general`` rotations + skew + t.z: nothing specialised;
* ``converging`` the bench's C3G rig at small size (toed-in, rolled, skewed cameras) with images
  rendered through those cameras (lfdg_render_scene_cams), so the geometry is self-consistent.

Images come from the rectified renderer; the perturbed cameras are valid PinholeCameras
(orthonormal R, upper-triangular K with K22 = 1) but do not match the pixels, which is irrelevant
for parity: both implementations get identical inputs.  Every stage is compared bit for bit with
the reference (oracle/_ref): SLIC, sweep, rasterize, two refine iterations with RefineStats."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

V, W, H = 3, 160, 120


def _rot(ax, ay, az):
    cx, sx, cy, sy, cz, sz = np.cos(ax), np.sin(ax), np.cos(ay), np.sin(ay), np.cos(az), np.sin(az)
    rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    return rz @ ry @ rx


def _cams(kind, base):
    cams = base.copy()
    rng = np.random.default_rng({"tz": 1, "rot": 2, "skew": 3, "general": 4}.get(kind, 0))
    for v in range(cams.shape[0]):
        K = cams[v, 0:9].reshape(3, 3).copy()
        R = cams[v, 9:18].reshape(3, 3).copy()
        t = cams[v, 18:21].copy()
        if kind in ("rot", "general") and v > 0:
            R = _rot(*(rng.uniform(-0.02, 0.02, 3)))
            t = t + rng.uniform(-0.01, 0.01, 3)
        if kind in ("skew", "general"):
            K[0, 1] = 0.25 + 0.1 * v
        if kind in ("tz", "general"):
            t[2] = 0.05 * v
        cams[v, 0:9] = K.ravel()
        cams[v, 9:18] = R.ravel()
        cams[v, 18:21] = t
    return cams


@pytest.fixture(scope="module", params=["grid", "tz", "rot", "skew", "general", "converging"])
def rig(request, ref):
    from paper_1812_06856_b200 import api, scenes

    kind = request.param
    if kind == "converging":
        base = scenes.render_scene("cluttered", 4, W, H, 160.0, 0.1, gt=False, lab=False)
        cams = scenes.converging_rig(base["cams"], base["range"])
        sc = scenes.render_scene_cams("cluttered", 4, W, H, 160.0, 0.1, cams)
    elif kind == "grid":
        sc = ref.render_scene("cluttered", 0, W, H, 160.0, 0.1, grid=(2, 2))
        cams = sc["cams"]
    else:
        sc = ref.render_scene("cluttered", V, W, H, 160.0, 0.1)
        cams = _cams(kind, sc["cams"])
    rs = ref.Session(sc["lab"], cams, sc["range"])
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], cams, sc["range"])
    nv = sc["lab"].shape[0]
    for v in range(nv):
        rs.slic(v, 12, 0.1, 10)
        dc.slic(v, api.SlicParams(12, 0.1, 10))
    return kind, nv, rs, dc


def test_rig_sweep_rasterize_refine(rig):
    from paper_1812_06856_b200 import api

    kind, nv, rs, dc = rig
    for v in range(nv):
        assert np.array_equal(dc.get_grid(v).label_map, rs.grid(v)["labels"])
    for v in range(nv):
        want = rs.sweep(v, 32, 0.05, 0, 7)
        got = dc.sweep(v, api.SweepParams(32, 0.05, 0), 7)
        bad = np.any(got != want, axis=1)
        assert not bad.any(), f"{kind}: sweep view {v}: {bad.sum()} planes differ"
    rs.rasterize()
    dc.rasterize()
    for v in range(nv):
        assert np.array_equal(dc.get_depth(v), rs.depth(v)), f"{kind}: rasterize view {v}"
    rs.refine_context(32, iterations=2)
    dc.make_refine_context(api.EnergyParams(iterations=2), 32)
    for l in (1, 2):
        acc_r, vio_r = rs.refine_iteration(l, with_stats=True)
        acc_g, vio_g = dc.refine_iteration(l)
        rs.rasterize()
        dc.rasterize()
        for v in range(nv):
            want, got = rs.planes(v), dc.get_planes(v)
            bad = np.any(got != want, axis=1)
            assert not bad.any(), f"{kind}: iteration {l} view {v}: {bad.sum()} planes differ"
            assert np.array_equal(dc.get_depth(v), rs.depth(v)), f"{kind}: depth after iteration {l}"
        assert (acc_g, vio_g) == (acc_r, vio_r), f"{kind}: RefineStats after iteration {l}"


def test_rig_fusion(rig):
    """fuse_all (fusion.hpp:31-100) of the refined state of the test above: the general transfer
    paths of the fusion kernels against the reference, bit for bit."""
    kind, nv, rs, dc = rig
    eps = 0.05
    want = rs.fuse_all(eps)
    dc.fuse_views(eps)
    for v in range(nv):
        got = dc.get_fused(v)
        assert np.array_equal(got.view(np.uint32), want[v].view(np.uint32)), f"{kind}: fused view {v}"


@pytest.mark.parametrize("grid", [(4, 5), (0, 0), "jittered"])
def test_many_matching_views(ref, grid):
    """All-others matching with many targets, every stage bit-exact against the reference:
    a 4x5 grid rig, N = 19 (the many-target mode: groups of 8 lanes over three target rounds, the
    last one partial), the same grid with every camera centre jittered in x and y (every target
    translation distinct), and 70 views on a line, N = 69 (groups of 32
    lanes over three rounds, the wide photo cache).  Iteration 1 runs with RefineStats (the
    re-check instantiation), iteration 2 without (the hot instantiation)."""
    from paper_1812_06856_b200 import api

    sc = ref.render_scene("cluttered", 70, 64, 48, 64.0, 0.01, grid=(4, 5) if grid == "jittered" else grid)
    cams = sc["cams"].copy()
    if grid == "jittered":
        jit = np.random.default_rng(11).uniform(-0.002, 0.002, (cams.shape[0], 2))
        cams[:, 18:20] += jit  # t.x, t.y; t.z stays 0 (kFlat)
    nv = sc["lab"].shape[0]
    rs = ref.Session(sc["lab"], cams, sc["range"])
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], cams, sc["range"])
    for v in range(nv):
        rs.slic(v, 8, 0.1, 10)
        dc.slic(v, api.SlicParams(8, 0.1, 10))
    checked = (0, nv // 2, nv - 1)
    for v in checked:
        want = rs.sweep(v, 16, 0.05, 0, 1)
        assert np.array_equal(dc.sweep(v, api.SweepParams(16, 0.05, 0), 1), want), f"sweep view {v}"
    for v in range(nv):
        if v not in checked:
            p = rs.sweep(v, 16, 0.05, 0, 1)
            dc.set_planes(v, p)
    rs.rasterize()
    dc.rasterize()
    rs.refine_context(16, iterations=1)
    dc.make_refine_context(api.EnergyParams(iterations=1), 16)
    acc_r, _ = rs.refine_iteration(1, with_stats=True)
    acc_g, _ = dc.refine_iteration(1)
    for v in range(nv):
        assert np.array_equal(dc.get_planes(v), rs.planes(v)), f"refine view {v}"
    assert acc_g == acc_r
    rs.rasterize()
    dc.rasterize()
    rs.refine_iteration(2, with_stats=False)
    dc.refine_iteration(2, with_stats=False)
    for v in range(nv):
        assert np.array_equal(dc.get_planes(v), rs.planes(v)), f"refine l=2 view {v}"


def test_hundreds_of_matching_views(ref):
    """Inputs the reference accepts at any size: 320 views (N = 319 matching views, off-plane
    camera centres so the general refine kernel runs with its per-target tables; shared memory
    then holds two warps per CTA instead of four) and 5000 / 20000 sweep levels.  Sampled sweep winners and
    refine tasks are compared with the reference."""
    from paper_1812_06856_b200 import api

    V, w, h = 320, 48, 36
    sc = ref.render_scene("cluttered", V, w, h, 48.0, 0.002)
    cams = sc["cams"].copy()
    cams[:, 20] = 0.001 * np.arange(V)  # t.z != 0: not kFlat
    rs = ref.Session(sc["lab"], cams, sc["range"])
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], cams, sc["range"])
    dc.slic_views(0, V, api.SlicParams(12, 0.1, 10))
    for v in range(V):
        rs.set_grid_from_labels(v, dc.get_grid(v).label_map, 12)
    for v in (0, 7):
        rs.slic(v, 12, 0.1, 10)
        assert np.array_equal(dc.get_grid(v).label_map, rs.grid(v)["labels"])
    dc.sweep_views(0, V, api.SweepParams(4, 0.05, 0), 0)
    want = rs.sweep_sample(5, np.arange(12, dtype=np.int32), 4, 0.05, 0, 0)
    assert np.array_equal(dc.get_planes(5), want)
    for v in range(V):
        rs.set_planes(v, dc.get_planes(v))
    rs.rasterize()
    dc.rasterize()
    rs.refine_context(4, iterations=1, size_init=24)
    dc.make_refine_context(api.EnergyParams(iterations=1, size_init=24), 4)
    rng = np.random.default_rng(3)
    tv = rng.integers(0, V, 200)
    ts = rng.integers(0, 12, 200)
    want, _ = rs.refine_tasks(1, tv, ts)
    dc.refine_iteration(1, with_stats=False)
    got = np.stack([dc.get_planes(int(v))[int(s)] for v, s in zip(tv, ts)])
    assert np.array_equal(got, want)
    # 5000 sweep levels (the reference accepts any L >= 2)
    dc2 = api.DeviceContext(0)
    sc2 = ref.render_scene("cluttered", 3, 64, 48, 64.0, 0.1)
    rs2 = ref.Session(sc2["lab"], sc2["cams"], sc2["range"])
    dc2.set_views(sc2["lab"], sc2["cams"], sc2["range"])
    dc2.slic(0, api.SlicParams(12, 0.1, 10))
    rs2.slic(0, 12, 0.1, 10)
    for v in (1, 2):
        dc2.slic(v, api.SlicParams(12, 0.1, 10))
        rs2.slic(v, 12, 0.1, 10)
    got = dc2.sweep(0, api.SweepParams(5000, 0.05, 0), 3)
    assert np.array_equal(got, rs2.sweep(0, 5000, 0.05, 0, 3))
    # 20000 levels: beyond shared memory, the hypotheses live in global scratch slots and the
    # superpixels are swept in waves of resident CTAs
    got = dc2.sweep(1, api.SweepParams(20000, 0.05, 0), 5)
    assert np.array_equal(got, rs2.sweep(1, 20000, 0.05, 0, 5))
    dc2.sweep_views(0, 3, api.SweepParams(20000, 0.05, 0), 5)
    assert np.array_equal(dc2.get_planes(1), got)
