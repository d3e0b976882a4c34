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
    # C3 through a converging, non-rectified rig (the general camera paths measured at the
    # headline size): every camera toed in towards the scene centre, rolled, with a skewed K
    "C3G": dict(kind="cluttered", n_views=16, width=1920, height=1080, f=1920.0, baseline=0.04, grid=(0, 0),
                S=16, levels=256, iterations=5, max_neighbors=0, rig="converging"),
}


def converging_rig(cams: np.ndarray, d_range, roll_deg: float = 0.5, skew: float = 0.5) -> np.ndarray:
    """The rig `cams` (rectified line, centres on x) re-aimed: camera v keeps its centre c_v and
    looks at (x_mid, 0, Z0) — x_mid the middle of the rig, Z0 the depth of the mid inverse depth
    of the range (toe-in) — rolled by
    +-roll_deg (alternating) about its optical axis, with K01 = skew.  R maps world to camera
    (x_cam = R x + t), so R = Rz(roll) Ry(-phi), t = -R c."""
    out = np.array(cams, np.float64, copy=True)
    z0 = 2.0 / (1.0 / d_range[0] + 1.0 / d_range[1])
    centres = [-(out[v, 9:18].reshape(3, 3).T @ out[v, 18:21]) for v in range(out.shape[0])]
    x_mid = 0.5 * (min(c[0] for c in centres) + max(c[0] for c in centres))
    for v in range(out.shape[0]):
        K = out[v, 0:9].reshape(3, 3).copy()
        R0 = out[v, 9:18].reshape(3, 3)
        t0 = out[v, 18:21]
        c = -R0.T @ t0
        phi = np.arctan2(x_mid - c[0], z0 - c[2])
        cy, sy = np.cos(-phi), np.sin(-phi)
        ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
        rho = np.deg2rad(roll_deg) * (1 if v % 2 == 0 else -1)
        cz, sz = np.cos(rho), np.sin(rho)
        rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
        R = rz @ ry
        K[0, 1] = skew
        out[v, 0:9] = K.ravel()
        out[v, 9:18] = R.ravel()
        out[v, 18:21] = -R @ c
    return out


def render_scene(kind="cluttered", n_views=3, width=320, height=240, f=320.0, baseline=0.1, extra=0.0,
                 grid=(0, 0), threads=0, rgb=False, gt=True, lab=True):
    """fixtures.hpp render_scene + rgb_to_scaled_lab. Returns dict(lab, rgb, gt, cams, range)."""
    L = N.lib()
    nv = grid[0] * grid[1] if grid[0] > 0 else n_views
    lab_a = np.zeros((nv, height, width, 3), np.float32) if lab else None
    rgb_a = np.zeros((nv, height, width, 3), np.float32) if rgb else None
    gt_a = np.zeros((nv, height, width), np.float32) if gt else None
    cams = np.zeros((nv, 21), np.float64)
    rng = np.zeros(2, np.float64)
    N.check(L.lfdg_render_scene(KINDS[kind], n_views, width, height, f, baseline, extra, grid[0], grid[1], threads,
                                None if lab_a is None else N.ptr(lab_a), None if rgb_a is None else N.ptr(rgb_a),
                                None if gt_a is None else N.ptr(gt_a), N.ptr(cams), N.ptr(rng)))
    return dict(lab=lab_a, rgb=rgb_a, gt=gt_a, cams=cams, range=(float(rng[0]), float(rng[1])))


def render_scene_cams(kind, n_views, width, height, f, baseline, cams, extra=0.0, threads=0, rgb=False, gt=True):
    """The scene of (kind, n_views, W, H, f, baseline) rendered through the given cameras [V][21]."""
    L = N.lib()
    cams = np.ascontiguousarray(cams, np.float64)
    nv = cams.shape[0]
    lab = np.zeros((nv, height, width, 3), np.float32)
    rgb_a = np.zeros_like(lab) if rgb else None
    gt_a = np.zeros((nv, height, width), np.float32) if gt else None
    rng = np.zeros(2, np.float64)
    N.check(L.lfdg_render_scene_cams(KINDS[kind], n_views, width, height, f, baseline, extra, N.ptr(cams), nv, threads,
                                     N.ptr(lab), None if rgb_a is None else N.ptr(rgb_a),
                                     None if gt_a is None else N.ptr(gt_a), N.ptr(rng)))
    return dict(lab=lab, rgb=rgb_a, gt=gt_a, cams=cams, range=(float(rng[0]), float(rng[1])))


def render_config(name: str, threads: int = 0, gt: bool = True, rgb: bool = False):
    c = CONFIGS[name]
    if c.get("rig") == "converging":
        base = render_scene(c["kind"], c["n_views"], c["width"], c["height"], c["f"], c["baseline"], 0.0, c["grid"],
                            gt=False, lab=False)  # the rectified rig and range only
        cams = converging_rig(base["cams"], base["range"])
        return render_scene_cams(c["kind"], c["n_views"], c["width"], c["height"], c["f"], c["baseline"], cams,
                                 threads=threads, gt=gt, rgb=rgb)
    return render_scene(c["kind"], c["n_views"], c["width"], c["height"], c["f"], c["baseline"], 0.0, c["grid"],
                        threads=threads, gt=gt, rgb=rgb)
