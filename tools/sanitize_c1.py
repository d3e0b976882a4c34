"""Whole hot path at C1 (SLIC, sweep, rasterize, 3 refine iterations, fusion, sRGB->LAB upload,
evaluation) for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_c1.py

Checks the result against the frozen reference golden so a sanitizer run is also a parity run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1812_06856_b200 import api, scenes  # noqa: E402


def main():
    sc = scenes.render_config("C1", rgb=True)
    g = np.load(os.path.join(ROOT, "tests", "golden", "c1_golden.npz"))
    dc = api.DeviceContext(0)
    dc.set_views(sc["lab"], sc["cams"], sc["range"])
    dc.upload_rgb(sc["rgb"])  # the GPU sRGB -> LAB conversion overwrites the LAB with equal bytes
    dc.slic_views(0, 3, api.SlicParams(12, 0.1, 10))
    dc.sweep_views(0, 3, api.SweepParams(32, 0.05, 0), 0)
    dc.rasterize()
    dc.make_refine_context(api.EnergyParams(iterations=3), 32)
    acc, vio = dc.run_refinement()
    dc.fuse_views(0.05)
    ok = True
    for v in range(3):
        ok &= np.array_equal(dc.get_planes(v).view(np.uint64), g[f"refine3_{v}"].view(np.uint64))
        ok &= np.array_equal(dc.get_depth(v).view(np.uint32), g[f"depth{v}"].view(np.uint32))
        dc.get_fused(v)
    dc.close()
    print("sanitize_c1: parity", "OK" if ok else "MISMATCH", "accepted", acc, "violations", vio)
    sys.exit(0 if ok and vio == 0 else 1)


if __name__ == "__main__":
    main()
