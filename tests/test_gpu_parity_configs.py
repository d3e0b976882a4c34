"""Sampled-task lockstep parity on the other BASELINE configs ("sampled-task
lockstep checks on C3-C5"; C2 is run the same way to keep the test minutes bounded):

* C2  8 x 1024x768 linear rig, S=12, L=128, N=7;
* C4  5x5 grid rig 1920x1080 (kFlat with per-target rows), S=16, L=256, N=24;
* C5  64 x 1920x1080, S=16, L=256, max_neighbors = 8 (matching_views' nearest-K selection).

The GPU runs the whole path (SLIC of every view, sweep of every view, rasterize).  The reference
(oracle/_ref) then checks: slic_segment on two views bit for bit; sweep_view's winner for 96
random superpixels of those views; and, from the GPU's sweep state loaded into the reference,
refine_iteration (l = 1) on 256 random tasks, planes bit for bit.  The reference's other grids are
rebuilt from the GPU label maps by its own recompute_stats (pipeline.hpp:188 resume path)."""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module", params=["C2", "C4", "C5"])
def cfg(request, ref):
    from paper_1812_06856_b200 import api, scenes

    name = request.param
    c = scenes.CONFIGS[name]
    sc = scenes.render_config(name, gt=False)
    V = sc["lab"].shape[0]
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], sc["cams"], sc["range"])
    dc.slic_views(0, V, api.SlicParams(c["S"], 0.1, 10))
    dc.sweep_views(0, V, api.SweepParams(c["levels"], 0.05, c["max_neighbors"]), 0)
    dc.rasterize()
    rs = ref.Session(sc["lab"], sc["cams"], sc["range"])
    workers = len(os.sched_getaffinity(0))
    checked = (0, V // 2 + 1)
    for v in range(V):
        if v in checked:
            rs.slic(v, c["S"], 0.1, 10, workers)
        else:
            rs.set_grid_from_labels(v, dc.get_grid(v).label_map, c["S"])
    return name, c, V, dc, rs, workers, checked


def test_config_slic(cfg):
    name, c, V, dc, rs, workers, checked = cfg
    for v in checked:
        want, got = rs.grid(v), dc.get_grid(v)
        assert np.array_equal(got.label_map, want["labels"]), f"{name}: labels of view {v}"
        assert np.array_equal(got.offsets, want["offsets"]) and np.array_equal(got.members, want["members"])
        assert np.array_equal(got.sp["cx"], want["records"]["cx"]) and np.array_equal(got.sp["cy"], want["records"]["cy"])
        assert np.array_equal(got.sp["mean_color"], want["records"]["color"])


def test_config_sweep_sample(cfg):
    name, c, V, dc, rs, workers, checked = cfg
    rng = np.random.default_rng(5)
    for v in checked:
        planes = dc.get_planes(v)
        sps = rng.choice(len(planes), 96, replace=False).astype(np.int32)
        want = rs.sweep_sample(v, sps, c["levels"], 0.05, c["max_neighbors"], 0, workers)
        got = planes[sps]
        bad = np.any(got != want, axis=1)
        assert not bad.any(), f"{name}: view {v}: {bad.sum()} of {len(sps)} sampled sweep winners differ"


def test_config_refine_sample(cfg):
    from paper_1812_06856_b200 import api

    name, c, V, dc, rs, workers, checked = cfg
    for v in range(V):
        rs.set_planes(v, dc.get_planes(v))
    rs.rasterize()
    for v in checked:
        assert np.array_equal(rs.depth(v), dc.get_depth(v)), f"{name}: rasterized depth of view {v}"
    rs.refine_context(c["levels"], iterations=c["iterations"], max_neighbors=c["max_neighbors"])
    dc.make_refine_context(api.EnergyParams(iterations=c["iterations"], max_neighbors=c["max_neighbors"]), c["levels"])
    rng = np.random.default_rng(11)
    nsp = len(dc.get_planes(0))
    tv = rng.integers(0, V, 256)
    ts = rng.integers(0, nsp, 256)
    want, _ = rs.refine_tasks(1, tv, ts, workers)
    dc.refine_iteration(1, with_stats=False)
    got = np.stack([dc.get_planes(int(v))[int(s)] for v, s in zip(tv, ts)])
    bad = np.any(got != want, axis=1)
    assert not bad.any(), f"{name}: {bad.sum()} of {len(tv)} sampled refine tasks differ"
