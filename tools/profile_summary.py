#!/usr/bin/env python3
"""Summarise ncu output into the tracked profiles/ directory.

  python tools/profile_summary.py launches <launch-list.csv> <out.csv> "<command that produced it>"
  python tools/profile_summary.py kernel <capture.ncu-rep> <out.txt>

`launches` folds an `ncu --metrics gpu__time_duration.sum --csv` launch list into a per-kernel
table (launches, total ms, share of the GPU time).  `kernel` extracts the metrics DESIGN.md and
bench.py's roofline cite (duration, pipe utilisation, issue activity, DRAM bytes, stall reasons)
from one `ncu --set full` capture.  Needs `ncu` on PATH for `kernel` (it reads the report with
`ncu -i ... --page raw --csv`).
"""
import collections
import csv
import re
import subprocess
import sys

KEYS = [
    "Kernel Name",
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
]


def short_name(name):
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("void ", "")
    return name


def launches(src, dst, command):
    per = collections.OrderedDict()
    with open(src) as f:
        lines = [l for l in f if l.startswith('"')]
    for row in csv.DictReader(lines):
        if row["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(row["Metric Value"].replace(",", ""))
        unit = row["Metric Unit"]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}[unit]
        k = short_name(row["Kernel Name"])
        n, t = per.get(k, (0, 0.0))
        per[k] = (n + 1, t + ns * scale)
    total = sum(t for _, t in per.values())
    with open(dst, "w") as f:
        f.write(f"# ncu launch list summary: {command}\n")
        f.write("# gpu__time_duration.sum, --clock-control none; cold-cache serialised launches: compare shares\n")
        f.write(f"# total GPU time {total:.3f} ms\n")
        f.write("kernel,launches,total_ms,share_pct\n")
        for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k},{n},{t:.3f},{100 * t / total:.2f}\n")


def kernel(rep, dst):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(dst, "w") as f:
        f.write(f"# ncu --set full summary of {rep.split('/')[-1]}\n")
        for vals in rows[2:]:
            d = dict(zip(hdr, vals))
            u = dict(zip(hdr, units))
            for k in KEYS:
                if k in d:
                    f.write(f"{k} = {d[k]} {u.get(k, '')}".rstrip() + "\n")
            st = []
            for h, v in d.items():
                if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                    try:
                        st.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            f.write("stalls_per_issue = " + ", ".join(f"{n}:{v:.2f}" for v, n in st[:10]) + "\n\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4])
    elif sys.argv[1] == "kernel":
        kernel(sys.argv[2], sys.argv[3])
    else:
        sys.exit(__doc__)
