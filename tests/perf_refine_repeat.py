"""Dev probe: time refine_iteration(l) repeatedly on an identical snapshot (C3)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1812_06856_b200 import api, scenes

sc = scenes.render_config("C3", gt=False)
dc = api.DeviceContext(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); dc.set_stream(s.cuda_stream)
dc.set_views(sc["lab"], sc["cams"], sc["range"])
dc.slic_views(0, 16, api.SlicParams(16, 0.1, 10))
dc.sweep_views(0, 16, api.SweepParams(256, 0.05, 0), 0)
dc.rasterize()
dc.make_refine_context(api.EnergyParams(iterations=5), 256)
dc.refine_iteration(1, with_stats=False); dc.rasterize()
snap = [dc.get_planes(v) for v in range(16)]
for l in (2, 4, 1):
    for rep in range(4):
        for v in range(16): dc.set_planes(v, snap[v])
        dc.rasterize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s); dc.refine_iteration(l, with_stats=False); e1.record(s); torch.cuda.synchronize()
        pe, ce = dc.refine_work(reset=True)
        print(f"l={l} rep={rep} ms={e0.elapsed_time(e1):.1f} pixel_evals={pe} cand_evals={ce}", flush=True)
