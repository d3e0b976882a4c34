"""Generate tests/golden/c3_init_depths.npz with the REFERENCE (oracle/_ref, unmodified headers):
C3 scene (cluttered_scene(16, 1920, 1080, f=1920, B=0.04)) -> slic_segment(S=16) -> sweep_view
(L=256, T=0.05, all-others matching, seed 0) for every view, using all host threads.

The fixture pins (a) full-size GPU sweep parity (tests/test_gpu_parity_full.py) and (b) the
sweep-init state on which bench.py's reference arm samples refine_iteration tasks.  It also
records the reference's measured per-view CPU times.  Takes ~25 min on 8 cores.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    from oracle import ref

    workers = os.cpu_count()
    t = time.time()
    sc = ref.render_scene("cluttered", 16, 1920, 1080, 1920.0, 0.04)
    s = ref.Session(sc["lab"], sc["cams"], sc["range"])
    times = {"render_s": time.time() - t, "workers": workers, "slic_s": [], "sweep_s": []}
    for v in range(16):
        t = time.time()
        s.slic(v, 16, 0.1, 10, workers)
        times["slic_s"].append(time.time() - t)
    print("slic done", times["slic_s"], flush=True)
    depths = np.zeros((16, 120 * 68), np.float64)
    for v in range(16):
        t = time.time()
        p = s.sweep(v, 256, 0.05, 0, 0, workers)
        times["sweep_s"].append(time.time() - t)
        assert np.all(p[:, 1:] == np.array([0.0, 0.0, -1.0]))
        depths[v] = p[:, 0]
        print("sweep view", v, times["sweep_s"][-1], flush=True)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c3_init_depths.npz")
    np.savez_compressed(out, depths=depths)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c3_init_times.json"), "w") as f:
        json.dump(times, f, indent=1)


if __name__ == "__main__":
    main()
