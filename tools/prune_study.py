#!/usr/bin/env python3
"""Candidate-evaluation study on the reference (oracle/_ref; analysis tool, CPU only).

For random refine tasks of a config (from the reference's sweep-init state) it takes every
candidate's E_s and E_c and counts how many consistency evaluations each evaluation order needs
to reproduce the task's result:
  index   the reference order with the kernel's prune E_s * m_task <= e_cur (current GPU kernel);
  best    best-first by upper bound E_s * m_task within each phase, stopping when the next bound
          cannot beat (or tie at a smaller index) the best energy found — enough for the final
          plane (first-index argmax, strictly above the initial energy), not for the accepted count.
  python tools/prune_study.py C3 200
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from oracle import ref
    from paper_1812_06856_b200.scenes import CONFIGS

    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    ntask = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    c = CONFIGS[name]
    sc = ref.render_scene(c["kind"], c["n_views"], c["width"], c["height"], c["f"], c["baseline"], 0.0, c["grid"])
    s = ref.Session(sc["lab"], sc["cams"], sc["range"])
    V = sc["lab"].shape[0]
    W = os.cpu_count()
    for v in range(V):
        s.slic(v, c["S"], 0.1, 10, W)
    fx = os.path.join(ROOT, "tests", "golden", f"{name.lower()}_init_depths.npz")
    for v in range(V):
        g = s.grid(v)
        p = np.zeros((g["grid_w"] * g["grid_h"], 4))
        p[:, 3] = -1
        p[:, 0] = np.load(fx)["depths"][v]
        s.set_planes(v, p)
    s.rasterize()
    s.refine_context(c["levels"], iterations=c["iterations"], max_neighbors=c["max_neighbors"])
    nsp = s.grid(0)["grid_w"] * s.grid(0)["grid_h"]
    eta = 0.5
    mins = [s.min_nb_sim(v, nsp) for v in range(V)]
    rng = np.random.default_rng(0)
    for l in range(1, c["iterations"] + 1):
        tot = {"cands": 0, "index": 0, "best": 0}
        for _ in range(ntask):
            v, sp = int(rng.integers(V)), int(rng.integers(nsp))
            e0, planes, es, ec, ph = s.task_candidates(l, v, sp)
            m_task = (1.0 + eta * (1.0 - float(mins[v][sp]))) * (1.0 + 2 ** -30)
            e = es * ec
            # repeats of an earlier plane (or of the initial plane) are never evaluated
            seen = {tuple(s.planes(v)[sp])}
            rep = np.zeros(len(e), bool)
            for i, pl in enumerate(map(tuple, planes)):
                rep[i] = pl in seen
                seen.add(pl)
            tot["cands"] += len(e)
            for phase in (1, 2):
                idx = np.where((ph == phase) & ~rep)[0]
                # index order
                e_cur = e0 if phase == 1 else e_cur_a
                ecur = e_cur
                for i in idx:
                    if es[i] * m_task <= ecur:
                        continue
                    tot["index"] += 1
                    if e[i] > ecur:
                        ecur = e[i]
                # best-first
                best, best_i = e_cur, -1
                for i in sorted(idx, key=lambda k: (-es[k], k)):
                    ub = es[i] * m_task
                    if ub < best or (ub == best and (best_i < 0 or i > best_i)):
                        break
                    tot["best"] += 1
                    if e[i] > best or (e[i] == best and best_i >= 0 and i < best_i):
                        best, best_i = e[i], i
                assert best == ecur
                if phase == 1:
                    e_cur_a = ecur
        print(f"l={l}: candidates {tot['cands']}, evaluated index-order {tot['index']}, best-first {tot['best']} "
              f"({tot['best'] / max(1, tot['index']):.2f}x)", flush=True)


if __name__ == "__main__":
    main()
