#!/usr/bin/env python3
"""A/B stage timing on one config (dev tool; not collected by pytest).

  python tools/ab_probe.py C3 VAR=0,VAR=1 ...

Renders the config once, then for each variant (a comma-separated list of environment
assignments read by the library at launch time, e.g. LFDG_REFINE_LEGACY=1) runs SLIC, sweep,
rasterize, make_refine_context and the refine iterations twice, timing every stage with CUDA
events on the context's stream; prints one JSON line per variant (second repetition) and checks
that every variant produces the same planes."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1812_06856_b200 import api, scenes

    name = sys.argv[1]
    variants = sys.argv[2:] or [""]
    c = scenes.CONFIGS[name]
    sc = scenes.render_config(name, gt=False)
    V = sc["lab"].shape[0]
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    dc = api.DeviceContext(0)
    dc.set_stream(stream.cuda_stream)
    dc.set_views(sc["lab"], sc["cams"], sc["range"])
    ref_planes = None
    for var in variants:
        env = dict(kv.split("=") for kv in var.split(",") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        for rep in range(2):
            ev = {}

            def mark(k):
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                ev[k] = e

            mark("t0")
            dc.slic_views(0, V, api.SlicParams(c["S"], 0.1, 10))
            mark("slic")
            dc.sweep_views(0, V, api.SweepParams(c["levels"], 0.05, c["max_neighbors"]), 0)
            mark("sweep")
            dc.rasterize()
            dc.make_refine_context(api.EnergyParams(iterations=c["iterations"], max_neighbors=c["max_neighbors"]),
                                   c["levels"])
            mark("ctx")
            for l in range(1, c["iterations"] + 1):
                dc.refine_iteration(l, with_stats=False)
                mark(f"refine{l}")
                dc.rasterize()
                mark(f"rast{l}")
            torch.cuda.synchronize()
        keys = list(ev)
        out = {"variant": var or "default"}
        for a, b in zip(keys, keys[1:]):
            out[b] = round(ev[a].elapsed_time(ev[b]), 2)
        out["refine_total"] = round(sum(v for k, v in out.items() if k.startswith("refine")), 2)
        out["total"] = round(ev[keys[0]].elapsed_time(ev[keys[-1]]), 2)
        pe, ce = dc.refine_work(reset=False)
        out["pix_evals_2reps"] = pe
        out["cand_evals_2reps"] = ce
        try:
            wc = dc.work_counters(reset=True)
            out["idle_pix_evals_2reps"] = wc["refine_idle_slot_evals"]
            out["sweep_samples_2reps"] = wc["sweep_samples"]
        except Exception:  # an older library without lfdg_work_counters
            pass
        planes = np.stack([dc.get_planes(v) for v in range(V)])
        if ref_planes is None:
            ref_planes = planes
        out["same_planes"] = bool(np.array_equal(planes.view(np.uint64), ref_planes.view(np.uint64)))
        print(json.dumps(out), flush=True)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


if __name__ == "__main__":
    main()
