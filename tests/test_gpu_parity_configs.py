"""Sampled-task lockstep parity on the other BASELINE workloads ("~10^4 random
(view, sp) tasks from the same snapshot"), at every refinement iteration:

* C4  5x5 grid rig 1920x1080 (kFlat with per-target rows, the many-target refine mode with the
      8-byte raster), S=16, L=256, N=24, 5 iterations;
* C5  64 x 1920x1080, S=16, L=256, max_neighbors = 8 (matching_views' nearest-K selection).

The GPU runs the whole path (SLIC of every view, sweep of every view, rasterize, five
refine_iteration + rasterize).  The reference (oracle/_ref, all host cores) checks:
  * slic_segment of EVERY view: label maps, records and member lists bit for bit;
  * sweep_view's winner for 10^4 random superpixels spread over the views;
  * for l = 1..5, from the GPU's own evolving state loaded into the reference (planes, then the
    reference's rasterize, compared with the GPU's depth of every view): refine_iteration's task
    body (refine.hpp:269-320) on 10^4 random tasks, planes bit for bit.
"""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N_TASKS = 10_000


@pytest.fixture(scope="module", params=["C4", "C5"])
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
    for v in range(V):
        rs.slic(v, c["S"], 0.1, 10, workers)
    return name, c, V, dc, rs, workers


def test_config_slic_all_views(cfg):
    name, c, V, dc, rs, workers = cfg
    for v in range(V):
        want, got = rs.grid(v), dc.get_grid(v)
        assert np.array_equal(got.label_map, want["labels"]), f"{name}: labels of view {v}"
        assert np.array_equal(got.offsets, want["offsets"]) and np.array_equal(got.members, want["members"])
        assert np.array_equal(got.sp["cx"], want["records"]["cx"]) and np.array_equal(got.sp["cy"], want["records"]["cy"])
        assert np.array_equal(got.sp["mean_color"], want["records"]["color"])


def test_config_sweep_sample(cfg):
    name, c, V, dc, rs, workers = cfg
    rng = np.random.default_rng(5)
    views = np.arange(V) if V <= 25 else np.linspace(0, V - 1, 16).round().astype(int)
    per = -(-N_TASKS // len(views))
    checked = 0
    for v in views:
        planes = dc.get_planes(int(v))
        sps = rng.choice(len(planes), per, replace=False).astype(np.int32)
        want = rs.sweep_sample(int(v), sps, c["levels"], 0.05, c["max_neighbors"], 0, workers)
        bad = np.any(planes[sps] != want, axis=1)
        assert not bad.any(), f"{name}: view {v}: {bad.sum()} of {len(sps)} sampled sweep winners differ"
        checked += len(sps)
    assert checked >= N_TASKS


def test_config_refine_lockstep_every_iteration(cfg):
    from paper_1812_06856_b200 import api

    name, c, V, dc, rs, workers = cfg
    it = c["iterations"]
    dc.make_refine_context(api.EnergyParams(iterations=it, max_neighbors=c["max_neighbors"]), c["levels"])
    nsp = len(dc.get_planes(0))
    for l in range(1, it + 1):
        for v in range(V):
            rs.set_planes(v, dc.get_planes(v))
        rs.rasterize()
        for v in range(V):
            assert np.array_equal(rs.depth(v).view(np.uint32), dc.get_depth(v).view(np.uint32)), \
                f"{name}: rasterized depth of view {v} before iteration {l}"
        if l == 1:
            rs.refine_context(c["levels"], iterations=it, max_neighbors=c["max_neighbors"])
        rng = np.random.default_rng(100 + l)
        tv = rng.integers(0, V, N_TASKS)
        ts = rng.integers(0, nsp, N_TASKS)
        want, _ = rs.refine_tasks(l, tv, ts, workers)
        dc.refine_iteration(l, with_stats=False)
        all_planes = np.stack([dc.get_planes(v) for v in range(V)])
        got = all_planes[tv, ts]
        bad = np.any(got != want, axis=1)
        assert not bad.any(), f"{name}: iteration {l}: {bad.sum()} of {N_TASKS} sampled refine tasks differ"
        dc.rasterize()
