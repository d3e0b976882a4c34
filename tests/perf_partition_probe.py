"""Dev probe: refine only views [v0, v0 + n) of C3 (the per-rank work of an N-GPU partition) and
time each iteration with CUDA events.  Usage: perf_partition_probe.py n [v0]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1812_06856_b200 import api, scenes

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
v0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sc = scenes.render_config("C3", gt=False)
dc = api.DeviceContext(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); dc.set_stream(s.cuda_stream)
dc.set_views(sc["lab"], sc["cams"], sc["range"])
dc.slic_views(0, 16, api.SlicParams(16, 0.1, 10)); dc.sweep_views(0, 16, api.SweepParams(256, 0.05, 0), 0); dc.rasterize()
for rep in range(2):
    dc.make_refine_context(api.EnergyParams(iterations=5), 256)
    dc.set_refine_views(v0, n)
    for v in range(16): pass
    tot = 0
    out = []
    for l in range(1, 6):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s); dc.refine_iteration(l, with_stats=False); e1.record(s); torch.cuda.synchronize()
        dc.rasterize()
        out.append(round(e0.elapsed_time(e1), 1))
    print(f"views=[{v0},{v0 + n}) rep={rep} per-iteration ms={out} total={sum(out):.1f}", flush=True)
