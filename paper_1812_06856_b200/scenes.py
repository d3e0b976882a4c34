"""Synthetic camera-array scenes of BASELINE.json's configs (host C++ restatement of the
reference's fixtures.hpp in liblfdg.so; byte-identical to the reference's renderer)."""
from __future__ import annotations

import numpy as np

from . import _native as N

KINDS = {"cluttered": 0, "staircase": 1, "wall": 2, "slanted": 3, "occluder": 4}

# BASELINE.md §2 / SURVEY.md §8(d) config table.
CONFIGS = {
    "C1": dict(kind="cluttered", n_views=3, width=320, height=240, f=320.0, baseline=0.1, grid=(0, 0),
               S=12, levels=32, iterations=3, max_neighbors=0),
    "C2": dict(kind="cluttered", n_views=8, width=1024, height=768, f=1024.0, baseline=0.05, grid=(0, 0),
               S=12, levels=128, iterations=5, max_neighbors=0),
    "C3": dict(kind="cluttered", n_views=16, width=1920, height=1080, f=1920.0, baseline=0.04, grid=(0, 0),
               S=16, levels=256, iterations=5, max_neighbors=0),
    "C4": dict(kind="cluttered", n_views=25, width=1920, height=1080, f=1920.0, baseline=0.04, grid=(5, 5),
               S=16, levels=256, iterations=5, max_neighbors=0),
    "C5": dict(kind="cluttered", n_views=64, width=1920, height=1080, f=1920.0, baseline=0.02, grid=(0, 0),
               S=16, levels=256, iterations=5, max_neighbors=8),
}


def render_scene(kind="cluttered", n_views=3, width=320, height=240, f=320.0, baseline=0.1, extra=0.0,
                 grid=(0, 0), threads=0, rgb=False, gt=True):
    """fixtures.hpp render_scene + rgb_to_scaled_lab. Returns dict(lab, rgb, gt, cams, range)."""
    L = N.lib()
    nv = grid[0] * grid[1] if grid[0] > 0 else n_views
    lab = np.zeros((nv, height, width, 3), np.float32)
    rgb_a = np.zeros_like(lab) if rgb else None
    gt_a = np.zeros((nv, height, width), np.float32) if gt else None
    cams = np.zeros((nv, 21), np.float64)
    rng = np.zeros(2, np.float64)
    N.check(L.lfdg_render_scene(KINDS[kind], n_views, width, height, f, baseline, extra, grid[0], grid[1], threads,
                                N.ptr(lab), None if rgb_a is None else N.ptr(rgb_a),
                                None if gt_a is None else N.ptr(gt_a), N.ptr(cams), N.ptr(rng)))
    return dict(lab=lab, rgb=rgb_a, gt=gt_a, cams=cams, range=(float(rng[0]), float(rng[1])))


def render_config(name: str, threads: int = 0, gt: bool = True, rgb: bool = False):
    c = CONFIGS[name]
    return render_scene(c["kind"], c["n_views"], c["width"], c["height"], c["f"], c["baseline"], 0.0, c["grid"],
                        threads=threads, gt=gt, rgb=rgb)
