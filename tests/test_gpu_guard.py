"""Out-of-bounds-write detection without compute-sanitizer (closed on this GPU pool): the whole
hot path at C1, C2-shaped, ragged, C3 and C4 (many-target refine mode) sizes runs with LFDG_GUARD=1 (every device buffer bracketed
by 64 KiB guard zones, exact-size allocations) and no guard zone may change.  The detector itself
is checked by writing one element past a buffer (lfdg_debug_guard_selftest).  Each case runs in
a subprocess because the guard mode is fixed at the library's first allocation."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_1812_06856_b200 import api, scenes, _native as N
L = N.lib()
assert L.lfdg_debug_guard_enabled() == 1
det = C.c_uint64()
N.check(L.lfdg_debug_guard_selftest(0, C.byref(det)))
assert det.value == 1, "guard self-test did not detect the overrun"
kind, nv, w, h, f, b, grid, S, levels, iters, knn = {case!r}
sc = scenes.render_scene(kind, nv, w, h, f, b, 0.0, grid, rgb=True)
V = sc["lab"].shape[0]
dc = api.DeviceContext(0)
dc.set_views(sc["lab"], sc["cams"], sc["range"])
dc.upload_rgb(sc["rgb"])
dc.slic_views(0, V, api.SlicParams(S, 0.1, 10))
dc.sweep_views(0, V, api.SweepParams(levels, 0.05, knn), 0)
dc.rasterize()
dc.make_refine_context(api.EnergyParams(iterations=iters, max_neighbors=knn), levels)
acc, vio = dc.run_refinement()
dc.fuse_views(0.05)
dc.gather_candidates(0)
for v in range(V):
    dc.get_planes(v); dc.get_depth(v); dc.get_fused(v); dc.get_grid(v)
nb, nc = C.c_uint64(), C.c_uint64()
N.check(L.lfdg_debug_check_guards(C.byref(nb), C.byref(nc)))
print("buffers", nb.value, "corrupt", nc.value, "violations", vio)
assert nb.value > 20 and nc.value == 0 and vio == 0
dc.close()
"""

CASES = {
    "c1": ("cluttered", 3, 320, 240, 320.0, 0.1, (0, 0), 12, 32, 3, 0),
    "ragged": ("staircase", 4, 203, 131, 200.0, 0.08, (0, 0), 13, 24, 3, 2),
    "grid3x3": ("occluder", 9, 250, 190, 250.0, 0.05, (3, 3), 11, 16, 2, 0),
    "c2_shape": ("cluttered", 8, 1024, 768, 1024.0, 0.05, (0, 0), 12, 128, 5, 0),
    "c3": ("cluttered", 16, 1920, 1080, 1920.0, 0.04, (0, 0), 16, 256, 5, 0),
    "c4_many_targets": ("cluttered", 25, 1920, 1080, 1920.0, 0.04, (5, 5), 16, 256, 5, 0),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_no_out_of_bounds_writes(name):
    env = dict(os.environ, LFDG_GUARD="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, case=CASES[name])], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "corrupt 0" in r.stdout
