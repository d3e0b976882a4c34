"""ctypes wrapper over oracle/_ref/liblfdref.so (the UNMODIFIED reference headers + shims).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
reference / cpu_baseline leg as the checker and the CPU timing arm.  The product package
(paper_1812_06856_b200) never imports anything under oracle/.

All arithmetic happens inside the reference's own code (see oracle/ref_harness.cpp for the
file:line of every wrapped function).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "liblfdref.so")

SCENE_KINDS = {"cluttered": 0, "staircase": 1, "wall": 2, "slanted": 3, "occluder": 4}

RECORD_DTYPE = np.dtype(
    [("cx", "<f8"), ("cy", "<f8"), ("color", "<f4", (3,)), ("count", "<i4"), ("gx", "<i4"), ("gy", "<i4")]
)
assert RECORD_DTYPE.itemsize == 40

_lib = None


def build_if_possible() -> bool:
    """Build _ref/liblfdref.so from /root/reference when the sources are present."""
    if os.path.exists(LIB_PATH):
        return True
    if not os.path.isdir("/root/reference/proj/include"):
        return False
    subprocess.run(["make", "-s", "ref"], cwd=HERE, check=True)
    return os.path.exists(LIB_PATH)


def available() -> bool:
    return os.path.exists(LIB_PATH) or build_if_possible()


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not available():
        raise RuntimeError("oracle/_ref/liblfdref.so is not built (needs /root/reference to build)")
    L = C.CDLL(LIB_PATH)
    P, I, D, F, U64 = C.c_void_p, C.c_int, C.c_double, C.c_float, C.c_uint64
    L.ref_last_error.restype = C.c_char_p
    L.ref_render_scene.argtypes = [I, I, I, I, D, D, D, I, I, P, P, P, P, P]
    L.ref_rgb_to_scaled_lab.argtypes = [C.c_int64, P, P]
    L.ref_session_create.restype = P
    L.ref_session_create.argtypes = [I, I, I, P, P, D, D]
    L.ref_session_destroy.argtypes = [P]
    L.ref_slic.argtypes = [P, I, I, F, I, I]
    L.ref_set_grid_from_labels.argtypes = [P, I, P, I]
    L.ref_grid_dims.argtypes = [P, I, C.POINTER(I), C.POINTER(I)]
    L.ref_get_grid.argtypes = [P, I, P, P, P, P]
    L.ref_matching_views.argtypes = [P, I, I, P]
    L.ref_sweep.argtypes = [P, I, I, F, I, U64, I, P]
    L.ref_sweep_cost.restype = D
    L.ref_sweep_cost.argtypes = [P, I, I, D, P, I, F]
    L.ref_set_planes.argtypes = [P, I, P]
    L.ref_get_planes.argtypes = [P, I, P]
    L.ref_rasterize.argtypes = [P]
    L.ref_get_depth.argtypes = [P, I, P]
    L.ref_set_depth.argtypes = [P, I, P]
    L.ref_refine_context.argtypes = [P, D, F, F, I, I, I, I, I, I, I, I, P, P]
    L.ref_min_nb_sim.argtypes = [P, I, P]
    L.ref_refine_iteration.argtypes = [P, I, I, I, P, P]
    for name in ("ref_energy", "ref_smoothness_term", "ref_consistency_term"):
        getattr(L, name).restype = D
        getattr(L, name).argtypes = [P, I, I, P]
    L.ref_pair_stats.argtypes = [P, I, I, P, I, P]
    L.ref_normal_candidates.argtypes = [P, I, I, P]
    L.ref_grid_neighbors.argtypes = [P, I, I, I, I, I, P]
    L.ref_sweep_sample.argtypes = [P, I, P, I, I, F, I, U64, I, P]
    L.ref_refine_tasks.argtypes = [P, I, P, P, I, I, P, P, P, P]
    L.ref_fuse_all.argtypes = [P, D, I, P]
    L.ref_task_candidates.argtypes = [P, I, I, I, I, P, P, P, P, P]
    L.ref_gather_candidates.argtypes = [P, I, P, P, P, C.c_int64, P]
    L.ref_bad_pixel_rate.restype = D
    L.ref_bad_pixel_rate.argtypes = [I, I, I, P, P, I, P, D, D, D, I, D]
    _lib = L
    return L


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc: int):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def render_scene(kind="cluttered", n_views=3, width=320, height=240, f=320.0, baseline=0.1, extra=0.0,
                 grid=(0, 0)):
    """inc/fixtures.hpp render_scene + rgb_to_scaled_lab. Returns dict(lab, rgb, gt, cams, range)."""
    L = lib()
    nv = grid[0] * grid[1] if grid[0] > 0 else n_views
    lab = np.zeros((nv, height, width, 3), np.float32)
    rgb = np.zeros_like(lab)
    gt = np.zeros((nv, height, width), np.float32)
    cams = np.zeros((nv, 21), np.float64)
    rng = np.zeros(2, np.float64)
    _check(L.ref_render_scene(SCENE_KINDS[kind], n_views, width, height, f, baseline, extra, grid[0], grid[1],
                              _p(lab), _p(rgb), _p(gt), _p(cams), _p(rng)))
    return dict(lab=lab, rgb=rgb, gt=gt, cams=cams, range=(float(rng[0]), float(rng[1])))


class Session:
    """A reference MultiViewSet + grids + PlaneMap + RefineContext (inc/sweep.hpp, inc/refine.hpp)."""

    def __init__(self, images: np.ndarray, cams: np.ndarray | None, d_range=(1.0, 10.0)):
        self.L = lib()
        self.images = np.ascontiguousarray(images, np.float32)
        self.V, self.H, self.W = self.images.shape[:3]
        self.cams = None if cams is None else np.ascontiguousarray(cams, np.float64)
        self.h = self.L.ref_session_create(self.V, self.W, self.H, _p(self.images),
                                           None if self.cams is None else _p(self.cams), d_range[0], d_range[1])

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_session_destroy(self.h)
            self.h = None

    def slic(self, view, size=12, compactness=0.1, iterations=10, workers=1):
        _check(self.L.ref_slic(self.h, view, size, compactness, iterations, workers))

    def set_grid_from_labels(self, view, labels, cell_size):
        labels = np.ascontiguousarray(labels, np.int32)
        _check(self.L.ref_set_grid_from_labels(self.h, view, _p(labels), cell_size))

    def grid(self, view):
        gw, gh = C.c_int(), C.c_int()
        self.L.ref_grid_dims(self.h, view, C.byref(gw), C.byref(gh))
        n = gw.value * gh.value
        labels = np.zeros(self.H * self.W, np.int32)
        rec = np.zeros(n, RECORD_DTYPE)
        off = np.zeros(n + 1, np.int32)
        mem = np.zeros(self.H * self.W, np.int32)
        self.L.ref_get_grid(self.h, view, _p(labels), _p(rec), _p(off), _p(mem))
        return dict(labels=labels, records=rec, offsets=off, members=mem, grid_w=gw.value, grid_h=gh.value)

    def sweep_sample(self, view, sps, levels, threshold=0.05, max_neighbors=0, seed=0, workers=1):
        sps = np.ascontiguousarray(sps, np.int32)
        out = np.zeros((len(sps), 4), np.float64)
        _check(self.L.ref_sweep_sample(self.h, view, _p(sps), len(sps), levels, threshold, max_neighbors, seed,
                                       workers, _p(out)))
        return out

    def refine_tasks(self, l, views, sps, workers=1, counts=False):
        """refine_iteration's task body on the listed tasks -> (planes, accepted[, cons_evals, pixel_evals])."""
        views = np.ascontiguousarray(views, np.int32)
        sps = np.ascontiguousarray(sps, np.int32)
        out = np.zeros((len(sps), 4), np.float64)
        acc = np.zeros(3, np.uint64)
        _check(self.L.ref_refine_tasks(self.h, l, _p(views), _p(sps), len(sps), workers, _p(out), _p(acc[0:1]),
                                       _p(acc[1:2]), _p(acc[2:3])))
        if counts:
            return out, int(acc[0]), int(acc[1]), int(acc[2])
        return out, int(acc[0])

    def task_candidates(self, l, view, sp, max_out=512):
        """Analysis helper: (e_init, planes [k][4], E_s [k], E_c [k], phase [k]) of one task."""
        planes = np.zeros((max_out, 4), np.float64)
        es = np.zeros(max_out, np.float64)
        ec = np.zeros(max_out, np.float64)
        ph = np.zeros(max_out, np.int32)
        e0 = np.zeros(1, np.float64)
        k = self.L.ref_task_candidates(self.h, l, view, sp, max_out, _p(planes), _p(es), _p(ec), _p(ph), _p(e0))
        if k < 0:
            _check(1)
        return float(e0[0]), planes[:k], es[:k], ec[:k], ph[:k]

    def fuse_all(self, epsilon, workers=1):
        out = np.zeros((self.V, self.H, self.W), np.float32)
        _check(self.L.ref_fuse_all(self.h, epsilon, workers, _p(out)))
        return out

    def gather_candidates(self, ref_view):
        off = np.zeros(self.H * self.W + 1, np.int32)
        total = np.zeros(1, np.int64)
        _check(self.L.ref_gather_candidates(self.h, ref_view, _p(off), None, None, 0, _p(total)))
        n = int(total[0])
        dep = np.zeros(max(n, 1), np.float32)
        vw = np.zeros(max(n, 1), np.int32)
        _check(self.L.ref_gather_candidates(self.h, ref_view, _p(off), _p(dep), _p(vw), n, _p(total)))
        return off, dep[:n], vw[:n]

    def matching_views(self, view, max_neighbors=0):
        out = np.zeros(self.V, np.int32)
        n = self.L.ref_matching_views(self.h, view, max_neighbors, _p(out))
        return out[:n].tolist()

    def sweep(self, view, levels=80, threshold=0.05, max_neighbors=0, seed=0, workers=1):
        gw, gh = C.c_int(), C.c_int()
        self.L.ref_grid_dims(self.h, view, C.byref(gw), C.byref(gh))
        planes = np.zeros((gw.value * gh.value, 4), np.float64)
        _check(self.L.ref_sweep(self.h, view, levels, threshold, max_neighbors, seed, workers, _p(planes)))
        return planes

    def sweep_cost(self, view, sp, depth, targets, threshold=0.05):
        t = np.ascontiguousarray(targets, np.int32)
        return self.L.ref_sweep_cost(self.h, view, sp, depth, _p(t), len(t), threshold)

    def set_planes(self, view, planes):
        planes = np.ascontiguousarray(planes, np.float64)
        self.L.ref_set_planes(self.h, view, _p(planes))

    def planes(self, view):
        gw, gh = C.c_int(), C.c_int()
        self.L.ref_grid_dims(self.h, view, C.byref(gw), C.byref(gh))
        out = np.zeros((gw.value * gh.value, 4), np.float64)
        self.L.ref_get_planes(self.h, view, _p(out))
        return out

    def rasterize(self):
        self.L.ref_rasterize(self.h)

    def depth(self, view):
        out = np.zeros((self.H, self.W), np.float32)
        self.L.ref_get_depth(self.h, view, _p(out))
        return out

    def set_depth(self, view, depth):
        depth = np.ascontiguousarray(depth, np.float32)
        self.L.ref_set_depth(self.h, view, _p(depth))

    def refine_context(self, sweep_levels, sigma=0.0, alpha=0.075, eta=0.5, size_init=0, steps_init=5,
                       iterations=5, max_neighbors=0, use_smoothness=True, use_consistency=True,
                       use_occlusion=True):
        s = np.zeros(1, np.float64)
        k = np.zeros(1, np.int32)
        _check(self.L.ref_refine_context(self.h, sigma, alpha, eta, size_init, steps_init, iterations,
                                         max_neighbors, int(use_smoothness), int(use_consistency),
                                         int(use_occlusion), sweep_levels, _p(s), _p(k)))
        return float(s[0]), int(k[0])

    def min_nb_sim(self, view, n):
        out = np.zeros(n, np.float32)
        self.L.ref_min_nb_sim(self.h, view, _p(out))
        return out

    def refine_iteration(self, l, workers=1, with_stats=False):
        acc = np.zeros(1, np.uint64)
        vio = np.zeros(1, np.uint64)
        _check(self.L.ref_refine_iteration(self.h, l, workers, int(with_stats), _p(acc), _p(vio)))
        return int(acc[0]), int(vio[0])

    def energy(self, view, sp, plane):
        return self.L.ref_energy(self.h, view, sp, _p(np.ascontiguousarray(plane, np.float64)))

    def smoothness_term(self, view, sp, plane):
        return self.L.ref_smoothness_term(self.h, view, sp, _p(np.ascontiguousarray(plane, np.float64)))

    def consistency_term(self, view, sp, plane):
        return self.L.ref_consistency_term(self.h, view, sp, _p(np.ascontiguousarray(plane, np.float64)))

    def pair_stats(self, view, sp, plane, target):
        out = np.zeros(5, np.float64)
        self.L.ref_pair_stats(self.h, view, sp, _p(np.ascontiguousarray(plane, np.float64)), target, _p(out))
        return out

    def normal_candidates(self, view, sp):
        out = np.zeros((8, 3), np.float64)
        n = self.L.ref_normal_candidates(self.h, view, sp, _p(out))
        return out[:n]

    def grid_neighbors(self, view, sp, kernel=False, size_px=0, step_sp=1):
        out = np.zeros(4096, np.int32)
        n = self.L.ref_grid_neighbors(self.h, view, sp, int(kernel), size_px, step_sp, _p(out))
        return out[:n].tolist()


def bad_pixel_rate(gt_all, cams, view, est, inv_depth_tol, focal=0.0, baseline=0.0, region=0, threshold=1.0):
    gt_all = np.ascontiguousarray(gt_all, np.float32)
    cams = np.ascontiguousarray(cams, np.float64)
    est = np.ascontiguousarray(est, np.float32)
    V, H, W = gt_all.shape
    return lib().ref_bad_pixel_rate(V, W, H, _p(gt_all), _p(cams), view, _p(est), inv_depth_tol, focal, baseline,
                                    region, threshold)
