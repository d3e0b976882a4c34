#!/usr/bin/env python3
"""Per-source-line instruction and stall-sample shares of one kernel in an ncu report
(needs -lineinfo and --import-source on):  python tools/ncu_lines.py <rep> [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
rows = []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        rows.append((int(r[7]), int(r[4]), f, r[0], r[1][:100]))
    except (ValueError, IndexError):
        pass
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
for ins, smp, fn, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * ins / ti:5.1f}% inst {100 * smp / ts:5.1f}% smp  {fn}:{ln}  {src}")
