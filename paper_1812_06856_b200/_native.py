"""ctypes binding of the C-ABI in include/lfdg.h (liblfdg.so, built in-tree by build.py).

There is no CPU fallback: importing this module on a machine without the built library, or
calling into it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LFDG_LIB") or os.path.join(HERE, "liblfdg.so")  # override: A/B experiments

LFDG_OK = 0
LFDG_INVALID_PARAMS = 1
LFDG_INVARIANT = 2
LFDG_CUDA = 3
LFDG_STATE = 4

# Buffer ids of lfdg_device_buffer.
BUF_LABELS, BUF_CX, BUF_CY, BUF_COLOR, BUF_COUNT, BUF_MOFF, BUF_MPIX, BUF_PLANES, BUF_DEPTH, BUF_CRAY, BUF_LAB = range(11)


class Camera(C.Structure):
    _fields_ = [("K", C.c_double * 9), ("R", C.c_double * 9), ("t", C.c_double * 3)]


class SlicParamsC(C.Structure):
    _fields_ = [("size", C.c_int), ("compactness", C.c_float), ("iterations", C.c_int)]


class SweepParamsC(C.Structure):
    _fields_ = [("levels", C.c_int), ("tssd_threshold", C.c_float), ("max_neighbors", C.c_int)]


class EnergyParamsC(C.Structure):
    _fields_ = [
        ("sigma", C.c_double),
        ("alpha", C.c_float),
        ("eta", C.c_float),
        ("size_init", C.c_int),
        ("steps_init", C.c_int),
        ("iterations", C.c_int),
        ("max_neighbors", C.c_int),
        ("use_smoothness", C.c_int),
        ("use_consistency", C.c_int),
        ("use_occlusion", C.c_int),
    ]


RECORD_DTYPE = np.dtype(
    [("cx", "<f8"), ("cy", "<f8"), ("mean_color", "<f4", (3,)), ("pixel_count", "<i4"), ("gx", "<i4"),
     ("gy", "<i4")]
)
assert RECORD_DTYPE.itemsize == 40

EXPORTED = [
    "lfdg_create", "lfdg_destroy", "lfdg_last_error", "lfdg_set_stream", "lfdg_synchronize", "lfdg_launch_count",
    "lfdg_set_views", "lfdg_update_images", "lfdg_slic_segment", "lfdg_slic_segment_views", "lfdg_grid_shape",
    "lfdg_get_grid", "lfdg_set_grid", "lfdg_sweep_view", "lfdg_sweep_views", "lfdg_matching_views",
    "lfdg_set_planes", "lfdg_get_planes", "lfdg_rasterize", "lfdg_rasterize_views", "lfdg_get_depth",
    "lfdg_set_depth", "lfdg_make_refine_context", "lfdg_set_refine_views", "lfdg_refine_iteration",
    "lfdg_run_refinement", "lfdg_get_min_nb_sim", "lfdg_device_buffer", "lfdg_mark_views_ready",
    "lfdg_selftest_exp", "lfdg_selftest_expf", "lfdg_render_scene", "lfdg_render_scene_cams", "lfdg_rgb_to_scaled_lab",
    "lfdg_upload_images", "lfdg_download_results", "lfdg_selftest_fp64_peak", "lfdg_selftest_fp32_peak", "lfdg_refine_work", "lfdg_work_counters", "lfdg_selftest_exp_nonpos",
    "lfdg_fuse_views", "lfdg_get_fused", "lfdg_gather_candidates", "lfdg_stability_fuse", "lfdg_upload_rgb",
    "lfdg_rgb_to_scaled_lab_gpu", "lfdg_eval_bad_pixel", "lfdg_debug_guard_enabled", "lfdg_debug_check_guards",
    "lfdg_debug_guard_selftest", "lfdg_upload_rgb8", "lfdg_prefetch_images", "lfdg_commit_images",
    "lfdg_download_results_async", "lfdg_wait_downloads",
]

_lib = None


class LfdgError(RuntimeError):
    """Base error; subclasses mirror the reference's exception classes."""

    code = LFDG_CUDA


class InvalidParams(LfdgError):  # lfd::InvalidParams (superpixel.hpp:14)
    code = LFDG_INVALID_PARAMS


class InvariantError(LfdgError):  # lfd::InvariantError (geometry.hpp:17)
    code = LFDG_INVARIANT


class CudaError(LfdgError):
    code = LFDG_CUDA


class StateError(LfdgError):
    code = LFDG_STATE


_ERRORS = {LFDG_INVALID_PARAMS: InvalidParams, LFDG_INVARIANT: InvariantError, LFDG_CUDA: CudaError,
           LFDG_STATE: StateError}


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python build.py` (or __graft_entry__.build()) first; "
                          "there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P, I, D, U64 = C.c_void_p, C.c_int, C.c_double, C.c_uint64
    PI, PU64 = C.POINTER(C.c_int), C.POINTER(C.c_uint64)
    sig = {
        "lfdg_create": (I, [I, C.POINTER(P)]),
        "lfdg_destroy": (None, [P]),
        "lfdg_last_error": (C.c_char_p, []),
        "lfdg_set_stream": (I, [P, P]),
        "lfdg_synchronize": (I, [P]),
        "lfdg_launch_count": (U64, [P]),
        "lfdg_set_views": (I, [P, I, I, I, P, P, D, D]),
        "lfdg_update_images": (I, [P, I, I, P]),
        "lfdg_slic_segment": (I, [P, I, C.POINTER(SlicParamsC)]),
        "lfdg_slic_segment_views": (I, [P, I, I, C.POINTER(SlicParamsC)]),
        "lfdg_grid_shape": (I, [P, I, PI, PI, PI]),
        "lfdg_get_grid": (I, [P, I, P, P, P, P]),
        "lfdg_set_grid": (I, [P, I, I, P]),
        "lfdg_sweep_view": (I, [P, I, C.POINTER(SweepParamsC), U64, P]),
        "lfdg_sweep_views": (I, [P, I, I, C.POINTER(SweepParamsC), U64]),
        "lfdg_matching_views": (I, [P, I, I, P, PI]),
        "lfdg_set_planes": (I, [P, I, P]),
        "lfdg_get_planes": (I, [P, I, P]),
        "lfdg_rasterize": (I, [P]),
        "lfdg_rasterize_views": (I, [P, I, I]),
        "lfdg_get_depth": (I, [P, I, P]),
        "lfdg_set_depth": (I, [P, I, P]),
        "lfdg_make_refine_context": (I, [P, C.POINTER(EnergyParamsC), I, C.POINTER(D), PI]),
        "lfdg_set_refine_views": (I, [P, I, I]),
        "lfdg_refine_iteration": (I, [P, I, PU64, PU64]),
        "lfdg_run_refinement": (I, [P, PU64, PU64]),
        "lfdg_get_min_nb_sim": (I, [P, I, P]),
        "lfdg_device_buffer": (I, [P, I, C.POINTER(P), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
        "lfdg_mark_views_ready": (I, [P, I, I, I]),
        "lfdg_selftest_exp": (I, [I, P, P, C.c_size_t]),
        "lfdg_selftest_expf": (I, [I, P, P, C.c_size_t]),
        "lfdg_render_scene": (I, [I, I, I, I, D, D, D, I, I, I, P, P, P, P, P]),
        "lfdg_render_scene_cams": (I, [I, I, I, I, D, D, D, P, I, I, P, P, P, P]),
        "lfdg_rgb_to_scaled_lab": (I, [C.c_int64, P, P]),
        "lfdg_upload_images": (I, [P, I, I, P]),
        "lfdg_upload_rgb": (I, [P, I, I, P]),
        "lfdg_eval_bad_pixel": (I, [I, I, I, I, P, P, I, P, C.c_double, C.c_double, C.c_double, P, I, P, P]),
        "lfdg_rgb_to_scaled_lab_gpu": (I, [I, P, P, C.c_size_t]),
        "lfdg_download_results": (I, [P, I, I, P, P, I]),
        "lfdg_selftest_fp64_peak": (I, [I, C.POINTER(D)]),
        "lfdg_selftest_fp32_peak": (I, [I, C.POINTER(D)]),
        "lfdg_refine_work": (I, [P, PU64, PU64, I]),
        "lfdg_work_counters": (I, [P, P, I]),
        "lfdg_selftest_exp_nonpos": (I, [I, P, P, C.c_size_t]),
        "lfdg_fuse_views": (I, [P, I, I, D]),
        "lfdg_get_fused": (I, [P, I, P]),
        "lfdg_gather_candidates": (I, [P, I, P, P, P, C.c_int64, C.POINTER(C.c_int64)]),
        "lfdg_stability_fuse": (I, [I, I, P, P, P, D, P]),
        "lfdg_upload_rgb8": (I, [P, I, I, P]),
        "lfdg_prefetch_images": (I, [P, I, I, P]),
        "lfdg_commit_images": (I, [P]),
        "lfdg_download_results_async": (I, [P, I, I, P, P]),
        "lfdg_wait_downloads": (I, [P]),
        "lfdg_debug_guard_enabled": (I, []),
        "lfdg_debug_check_guards": (I, [PU64, PU64]),
        "lfdg_debug_guard_selftest": (I, [I, PU64]),
    }
    allow_missing = os.environ.get("LFDG_ALLOW_MISSING_SYMBOLS") == "1"  # dev A/B against older builds
    for name, (res, args) in sig.items():
        if allow_missing and not hasattr(L, name):
            continue
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != LFDG_OK:
        msg = lib().lfdg_last_error().decode()
        raise _ERRORS.get(rc, LfdgError)(msg)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)
