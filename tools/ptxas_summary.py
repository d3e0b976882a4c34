#!/usr/bin/env python3
"""Registers / spills per kernel of one TU:  python tools/ptxas_summary.py <file.cu> [filter]"""
import re
import subprocess
import sys

src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
                      "-std=c++17", "-Xcompiler", "-fPIC", "-c", src, "-o", "/tmp/_ptxas.o", "-Xptxas", "-v"],
                     capture_output=True, text=True)
cur = None
rows = {}
for line in out.stderr.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    m = re.search(r"Function properties for (\w+)", line)
    if m:
        cur2 = m.group(1)
        if cur2 != cur:
            cur = None
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
if out.returncode:
    print(out.stderr)
for k, v in rows.items():
    name = re.sub(r"_ZN4lfdg\d+_GLOBAL__N__\w+?_cu_[0-9a-f]+", "", k)
    if flt in name:
        print(f"{name[:70]:70s} regs {v.get('regs')} spill st/ld {v.get('spill')}")
