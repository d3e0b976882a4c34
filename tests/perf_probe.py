"""Stage timing probe (dev tool, not collected by pytest): renders a config with the reference
fixtures (oracle/_ref) and times each GPU stage with CUDA events.  Usage:
  python tests/perf_probe.py C3 [--cache DIR]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C1": dict(kind="cluttered", n=3, w=320, h=240, f=320.0, b=0.1, S=12, L=32, iters=3, K=0),
    "C2": dict(kind="cluttered", n=8, w=1024, h=768, f=1024.0, b=0.05, S=12, L=128, iters=5, K=0),
    "C3s": dict(kind="cluttered", n=16, w=480, h=270, f=480.0, b=0.04, S=16, L=64, iters=2, K=0),
    "C4": dict(kind="cluttered", n=25, w=1920, h=1080, f=1920.0, b=0.04, S=16, L=256, iters=5, K=0, grid=(5, 5)),
    "C5": dict(kind="cluttered", n=64, w=1920, h=1080, f=1920.0, b=0.02, S=16, L=256, iters=5, K=8),
    "C3": dict(kind="cluttered", n=16, w=1920, h=1080, f=1920.0, b=0.04, S=16, L=256, iters=5, K=0),
}


def main():
    import torch
    from oracle import ref
    from paper_1812_06856_b200 import api

    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    c = CONFIGS[name]
    t0 = time.time()
    sc = ref.render_scene(c["kind"], c["n"], c["w"], c["h"], c["f"], c["b"], grid=c.get("grid", (0, 0)))
    print(f"render {time.time() - t0:.1f}s", flush=True)
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], sc["cams"], sc["range"])
    V = sc["lab"].shape[0]
    ev = lambda: torch.cuda.Event(enable_timing=True)
    for rep in range(2):
        marks = {}
        e0 = ev(); e0.record(); torch.cuda.synchronize()
        t = time.time()
        dc.slic_views(0, V, api.SlicParams(c["S"], 0.1, 10)); dc.synchronize(); marks["slic"] = time.time() - t
        t = time.time()
        dc.sweep_views(0, V, api.SweepParams(c["L"], 0.05, c["K"]), 0); dc.rasterize(); dc.synchronize()
        marks["sweep"] = time.time() - t
        t = time.time()
        dc.make_refine_context(api.EnergyParams(iterations=c["iters"], max_neighbors=c["K"]), c["L"])
        dc.synchronize(); marks["ctx"] = time.time() - t
        for l in range(1, c["iters"] + 1):
            t = time.time()
            dc.refine_iteration(l, with_stats=False); acc = -1
            dc.rasterize(); dc.synchronize()
            marks[f"refine{l}"] = (round(time.time() - t, 4), acc, dc.refine_work(reset=True))
        print(rep, marks, flush=True)


if __name__ == "__main__":
    main()
