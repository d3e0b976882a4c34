#!/usr/bin/env python3
"""Validate bench.py's reference-arm extrapolator against a full, timed run of the reference
(oracle/_ref, the unmodified reference headers) on the host cores (VERDICT r1 "measurement hygiene").

For each config: the full hot path on the CPU — slic_segment of every view, sweep_view of every
view, rasterize, make_refine_context, refine_iteration l = 1..iters each followed by rasterize —
timed stage by stage (ms/view = total / V, as pipeline.hpp:383-385 amortises refinement), and
beside it bench.py's bounded-sample estimate (reference_sample: one view's SLIC, n_sw sweep task
bodies, n_rf refine task bodies per l on the sweep-init state, scaled by the task counts) taken
on the same state.  Prints one JSON line per config.
  python tools/validate_cpu_extrapolation.py C1 C2
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from oracle import ref
    from paper_1812_06856_b200.scenes import CONFIGS

    workers = bench.cpu_cores()
    for name in sys.argv[1:] or ["C1", "C2"]:
        c = CONFIGS[name]
        sc = ref.render_scene(c["kind"], c["n_views"], c["width"], c["height"], c["f"], c["baseline"], 0.0, c["grid"])
        V = sc["lab"].shape[0]
        s = ref.Session(sc["lab"], sc["cams"], sc["range"])
        for v in range(V):  # warm-up (first-touch page faults, thread start-up)
            s.slic(v, c["S"], 0.1, 10, workers)
        s.sweep(0, c["levels"], 0.05, c["max_neighbors"], 0, workers)
        full = {}
        t = time.time()
        for v in range(V):
            s.slic(v, c["S"], 0.1, 10, workers)
        full["slic_s"] = time.time() - t
        t = time.time()
        init = [s.sweep(v, c["levels"], 0.05, c["max_neighbors"], 0, workers) for v in range(V)]
        full["sweep_s"] = time.time() - t
        for v in range(V):
            s.set_planes(v, init[v])
        t = time.time()
        s.rasterize()
        t_rast = time.time() - t
        s.refine_context(c["levels"], iterations=c["iterations"], max_neighbors=c["max_neighbors"])
        nsp = s.grid(0)["grid_w"] * s.grid(0)["grid_h"]
        # ---- bench.py's estimate on this (sweep-init) state
        st = dict(session=s, cfg=c, V=V, nsp=nsp, t_rast=t_rast, init_kind="reference sweep_view", setup_s=0.0)
        est = [bench.reference_sample(st, k, workers)["ms_per_view"] for k in range(3)]
        for v in range(V):  # the sample's SLIC re-segments a view with the same result; restore the state
            s.set_planes(v, init[v])
        s.rasterize()
        # ---- the full refinement, timed
        t_ref = []
        t = time.time()
        for l in range(1, c["iterations"] + 1):
            t0 = time.time()
            s.refine_iteration(l, workers)
            s.rasterize()
            t_ref.append(time.time() - t0)
        full["refine_s"] = t_ref
        full["rasterize_init_s"] = t_rast
        total = full["slic_s"] + full["sweep_s"] + t_rast + sum(t_ref)
        ms_full = 1e3 * total / V
        print(json.dumps({"config": name, "views": V, "workers": workers, "full_ms_per_view": ms_full,
                          "estimated_ms_per_view": est, "estimate_over_full": float(np.mean(est)) / ms_full,
                          "full_stages_s": full}), flush=True)


if __name__ == "__main__":
    main()
