"""Randomised whole-path parity (edge cases the reference's tests exercise, plus
parameter combinations they do not): each seed draws a scene kind, a camera rig (line or grid,
optionally perturbed into rotated / skewed / shifted cameras that select the general kernel
paths), the image size, the SLIC / sweep / energy parameters (including the ablation switches,
sigma, alpha, eta, size_init, steps_init and max_neighbors) and the sweep seed, then runs the
whole hot path on the GPU and on the reference (oracle/_ref) and compares every stage bit for
bit: label maps, sweep winners, depth rasters, planes + RefineStats after every iteration and the
fused depth."""
import numpy as np
import pytest

from test_gpu_parity_rigs import _cams

pytestmark = pytest.mark.gpu


def _draw(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = ["cluttered", "staircase", "wall", "slanted", "occluder"][seed % 5]
    grid = [(0, 0), (0, 0), (2, 2), (2, 3)][rng.integers(4)]
    nv = int(rng.integers(2, 6))
    W, H = int(rng.integers(48, 161)), int(rng.integers(40, 121))
    if rng.random() < 0.2:  # many targets: the 16- and 8-lane group layouts over target rounds
        grid = [(0, 0), (4, 5), (5, 5), (3, 6)][rng.integers(4)]
        nv = int(rng.integers(10, 26))
        W, H = int(rng.integers(40, 81)), int(rng.integers(32, 61))
    rig = ["none", "none", "tz", "rot", "skew", "general"][rng.integers(6)]
    S = int(rng.choice([5, 7, 8, 10, 12, 16]))
    slic = (S, float(rng.choice([0.02, 0.1, 0.4])), int(rng.integers(1, 11)))
    levels = int(rng.choice([2, 8, 17, 32, 48]))
    K = int(rng.choice([0, 0, 1, 2]))
    energy = dict(sigma=float(rng.choice([0.0, 0.0, 0.05])), alpha=float(rng.choice([0.075, 0.2])),
                  eta=float(rng.choice([0.5, 0.0, 1.0])), size_init=int(rng.choice([0, 0, 40])),
                  steps_init=int(rng.choice([5, 5, 2, 9])), iterations=int(rng.integers(1, 4)),
                  max_neighbors=K, use_smoothness=bool(rng.random() > 0.2),
                  use_consistency=bool(rng.random() > 0.2), use_occlusion=bool(rng.random() > 0.3))
    return dict(kind=kind, grid=grid, nv=nv, W=W, H=H, rig=rig, slic=slic, levels=levels, K=K,
                thr=float(rng.choice([0.05, 0.01, 0.3])), seed=int(rng.integers(0, 2**31)), energy=energy)


@pytest.mark.parametrize("seed", range(64))
def test_fuzz_whole_path(ref, seed):
    from paper_1812_06856_b200 import api

    p = _draw(seed)
    # extra > 0 widens the depth range (a single fronto-parallel wall has d_min == d_max otherwise)
    extra = 0.3 if p["kind"] == "wall" else 0.0
    sc = ref.render_scene(p["kind"], p["nv"], p["W"], p["H"], float(p["W"]), 0.1, extra, grid=p["grid"])
    cams = sc["cams"] if p["rig"] == "none" else _cams(p["rig"], sc["cams"])
    nv = sc["lab"].shape[0]
    rs = ref.Session(sc["lab"], cams, sc["range"])
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], cams, sc["range"])
    S, m, it = p["slic"]
    for v in range(nv):
        rs.slic(v, S, m, it)
        dc.slic(v, api.SlicParams(S, m, it))
        assert np.array_equal(dc.get_grid(v).label_map, rs.grid(v)["labels"]), f"{p}: SLIC view {v}"
    for v in range(nv):
        want = rs.sweep(v, p["levels"], p["thr"], p["K"], p["seed"])
        got = dc.sweep(v, api.SweepParams(p["levels"], p["thr"], p["K"]), p["seed"])
        bad = np.any(got != want, axis=1)
        assert not bad.any(), f"{p}: sweep view {v}: {bad.sum()} winners differ"
    rs.rasterize()
    dc.rasterize()
    for v in range(nv):
        assert np.array_equal(dc.get_depth(v), rs.depth(v)), f"{p}: rasterize view {v}"
    e = p["energy"]
    rs.refine_context(p["levels"], **e)
    dc.make_refine_context(api.EnergyParams(**e), p["levels"])
    for l in range(1, e["iterations"] + 1):
        acc_r, vio_r = rs.refine_iteration(l, with_stats=True)
        acc_g, vio_g = dc.refine_iteration(l)
        rs.rasterize()
        dc.rasterize()
        assert (acc_g, vio_g) == (acc_r, vio_r), f"{p}: RefineStats of iteration {l}"
        for v in range(nv):
            bad = np.any(dc.get_planes(v) != rs.planes(v), axis=1)
            assert not bad.any(), f"{p}: iteration {l} view {v}: {bad.sum()} planes differ"
            assert np.array_equal(dc.get_depth(v), rs.depth(v)), f"{p}: depth view {v} after {l}"
    want = rs.fuse_all(0.05)
    dc.fuse_views(0.05)
    for v in range(nv):
        assert np.array_equal(dc.get_fused(v).view(np.uint32), want[v].view(np.uint32)), f"{p}: fused view {v}"


def test_fuzz_invalid_energy_params_rejected_like_reference(ref):
    """EnergyParams::validate (refine.hpp:28-31): both implementations reject the same values."""
    from paper_1812_06856_b200 import _native as N
    from paper_1812_06856_b200 import api

    sc = ref.render_scene("cluttered", 2, 64, 48, 64.0, 0.1)
    rs = ref.Session(sc["lab"], sc["cams"], sc["range"])
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], sc["cams"], sc["range"])
    for v in range(2):
        rs.slic(v, 8, 0.1, 10)
        dc.slic(v, api.SlicParams(8, 0.1, 10))
    for bad in (dict(eta=1.5), dict(eta=-0.1), dict(alpha=0.0), dict(sigma=-1.0), dict(steps_init=0),
                dict(size_init=-1), dict(iterations=-1)):
        with pytest.raises(RuntimeError):
            rs.refine_context(16, **bad)
        with pytest.raises(N.InvalidParams):
            dc.make_refine_context(api.EnergyParams(**bad), 16)
