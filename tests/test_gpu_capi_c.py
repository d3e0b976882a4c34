"""The C-ABI from plain C (tests/native/capi_pipeline.c, only include/lfdg.h and liblfdg.so): the
whole path on a 3-view scene equals the reference (oracle/_ref) run on the same inputs — planes
and depth rasters bit for bit, RefineStats.accepted equal — and an invalid parameter returns
LFDG_INVALID_PARAMS."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1812_06856_b200")


def test_c_program_matches_reference(ref, tmp_path):
    exe = str(tmp_path / "capi_pipeline")
    subprocess.run(["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "capi_pipeline.c"), "-o", exe, "-L", LIBDIR, "-llfdg",
                    "-Wl,-rpath," + LIBDIR], check=True)
    out = str(tmp_path / "result.bin")
    r = subprocess.run([exe, out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    nsp = int(r.stdout.split()[1])
    accepted = int(r.stdout.split()[3])
    raw = open(out, "rb").read()
    V, W, H = 3, 160, 120
    planes = np.frombuffer(raw[: V * nsp * 32], np.float64).reshape(V, nsp, 4)
    depth = np.frombuffer(raw[V * nsp * 32:], np.float32).reshape(V, H, W)

    sc = ref.render_scene("cluttered", V, W, H, 160.0, 0.1)
    rs = ref.Session(sc["lab"], sc["cams"], sc["range"])
    for v in range(V):
        rs.slic(v, 12, 0.1, 10)
    for v in range(V):
        rs.set_planes(v, rs.sweep(v, 32, 0.05, 0, 0))
    rs.rasterize()
    rs.refine_context(32, iterations=2)
    acc = 0
    for l in (1, 2):
        a, _ = rs.refine_iteration(l, with_stats=True)
        acc += a
        rs.rasterize()
    for v in range(V):
        assert np.array_equal(planes[v], rs.planes(v)), f"planes of view {v}"
        assert np.array_equal(depth[v].reshape(-1), rs.depth(v).reshape(-1)), f"depth of view {v}"
    assert accepted == acc
