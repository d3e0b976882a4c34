#!/usr/bin/env python3
"""Hot SASS instructions of one kernel in an ncu report, with their execution frequency relative to
the hottest instruction and the average active threads per warp-instruction (divergence):
  python tools/ncu_sass_hot.py <rep> [min_rel]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
min_rel = float(sys.argv[2]) if len(sys.argv) > 2 else 0.15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ie, st, at = (hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"),
              hdr.index("Avg. Threads Executed"))
data = [(r[1], int(r[ie] or 0), int(r[st] or 0), float(r[at] or 0)) for r in rows[2:] if len(r) > ie]
tot = sum(d[1] for d in data) or 1
mx = max(d[1] for d in data) or 1
hot = [d for d in data if d[1] >= min_rel * mx]
print(f"# {rows[0][1][:120]}")
print(f"# warp instructions {tot}; {len(hot)} instructions at >= {min_rel} of the hottest carry "
      f"{100 * sum(d[1] for d in hot) / tot:.1f}% of them")
print("# rel_freq avg_threads stall_samples sass")
for src, n, smp, thr in hot:
    print(f"{n / mx:5.2f} {thr:5.1f} {smp:7d}  {src.strip()[:90]}")
