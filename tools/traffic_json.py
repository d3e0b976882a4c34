#!/usr/bin/env python3
"""profiles/r2_traffic.json from an `ncu --set full` capture of k_refine: DRAM bytes (read + write)
of the launch, keyed to the sha256 of the refine.cu that was profiled (bench.py uses the figure
only while that source is the one being benched).
  python tools/traffic_json.py <rep> <refine.cu as profiled> "<capture command>" """
import csv
import hashlib
import json
import subprocess
import sys

rep, src, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
r = rows[2]
def val(k):
    i = hdr.index(k)
    return float(r[i].replace(",", "")) * scale.get(units[i], 1)
out = {"k_refine": {"dram_bytes_per_launch": int(val("dram__bytes_read.sum") + val("dram__bytes_write.sum")),
                    "dram_read": int(val("dram__bytes_read.sum")), "dram_write": int(val("dram__bytes_write.sum")),
                    "duration_ms": val("gpu__time_duration.sum") / 1e6 if units[hdr.index("gpu__time_duration.sum")] == "ns"
                    else val("gpu__time_duration.sum"),
                    "kernel": r[hdr.index("Kernel Name")][:80],
                    "refine_cu_sha256": hashlib.sha256(open(src, "rb").read()).hexdigest(),
                    "capture": cmd}}
json.dump(out, open("profiles/r2_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
