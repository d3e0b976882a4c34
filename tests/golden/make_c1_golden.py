"""Generate tests/golden/c1_golden.npz with the REFERENCE (oracle/_ref, unmodified headers):
C1 = cluttered_scene(3, 320, 240, f=320, B=0.1), slic_segment(S=12), sweep_view(L=32, seed 0),
rasterize, make_refine_context(L=32, 3 iterations), 3 x (refine_iteration with RefineStats;
rasterize).  Stores labels, sweep planes, refined planes per iteration, final depth and the
accepted counts.  Pins the oracle build (tests/test_oracle_pinning.py) and the GPU path
(tests/test_gpu_parity_c1.py compares against the live oracle; this file against the frozen one).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    from oracle import ref

    sc = ref.render_scene("cluttered", 3, 320, 240, 320.0, 0.1)
    s = ref.Session(sc["lab"], sc["cams"], sc["range"])
    out = {}
    for v in range(3):
        s.slic(v, 12, 0.1, 10)
        out[f"labels{v}"] = s.grid(v)["labels"]
        out[f"sweep{v}"] = s.sweep(v, 32, 0.05, 0, 0)
    s.rasterize()
    s.refine_context(32, iterations=3)
    acc = []
    for l in range(1, 4):
        a, vio = s.refine_iteration(l, with_stats=True)
        assert vio == 0
        acc.append(a)
        s.rasterize()
        for v in range(3):
            out[f"refine{l}_{v}"] = s.planes(v)
    for v in range(3):
        out[f"depth{v}"] = s.depth(v)
    out["accepted"] = np.array(acc, np.int64)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c1_golden.npz"), **out)


if __name__ == "__main__":
    main()
