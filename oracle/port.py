"""ctypes wrapper over oracle/_build/liblfdoracle.so, the plain-C restatement (lfd_oracle.c).

TEST INFRASTRUCTURE ONLY (tests/, bench.py cpu_baseline kind "port").  Pinned against the
reference (oracle/_ref) by tests/test_oracle_restatement.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liblfdoracle.so")

REC = np.dtype([("cx", "<f8"), ("cy", "<f8"), ("color", "<f4", (3,)), ("count", "<i4"), ("gx", "<i4"),
                ("gy", "<i4")])


class Grid(C.Structure):
    _fields_ = [("W", C.c_int), ("H", C.c_int), ("S", C.c_int), ("gw", C.c_int), ("gh", C.c_int),
                ("labels", C.c_void_p), ("rec", C.c_void_p), ("off", C.c_void_p), ("mem", C.c_void_p)]


class Energy(C.Structure):
    _fields_ = [("sigma", C.c_double), ("alpha", C.c_float), ("eta", C.c_float), ("size_init", C.c_int),
                ("steps_init", C.c_int), ("iterations", C.c_int), ("max_neighbors", C.c_int),
                ("use_smoothness", C.c_int), ("use_consistency", C.c_int), ("use_occlusion", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-s", "_build/liblfdoracle.so"], cwd=HERE, check=True)
        L = C.CDLL(LIB_PATH)
        P, I, D, F, U64 = C.c_void_p, C.c_int, C.c_double, C.c_float, C.c_uint64
        L.lfdo_slic_segment.argtypes = [I, I, P, I, F, I, C.POINTER(Grid)]
        L.lfdo_sweep_view.argtypes = [I, P, P, D, D, P, I, I, F, I, U64, P]
        L.lfdo_rasterize.argtypes = [P, C.POINTER(Grid), P, P]
        L.lfdo_refine_iteration.argtypes = [I, P, D, D, P, C.POINTER(Energy), P, P, I, P, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class PortGrid:
    def __init__(self, W, H, S):
        gw, gh = (W + S - 1) // S, (H + S - 1) // S
        self.labels = np.zeros(W * H, np.int32)
        self.rec = np.zeros(gw * gh, REC)
        self.off = np.zeros(gw * gh + 1, np.int32)
        self.mem = np.zeros(W * H, np.int32)
        self.c = Grid(W, H, S, gw, gh, _p(self.labels).value, _p(self.rec).value, _p(self.off).value,
                      _p(self.mem).value)


class Port:
    """One view set: images [V][H][W][3], cams [V][21], range."""

    def __init__(self, images, cams, d_range):
        self.images = np.ascontiguousarray(images, np.float32)
        self.cams = np.ascontiguousarray(cams, np.float64)
        self.V, self.H, self.W = self.images.shape[:3]
        self.range = d_range
        self.grids = [None] * self.V

    def slic(self, v, S=12, m=0.1, iters=10):
        g = PortGrid(self.W, self.H, S)
        rc = lib().lfdo_slic_segment(self.W, self.H, _p(self.images[v]), S, m, iters, C.byref(g.c))
        if rc:
            raise ValueError("invalid SLIC parameters")
        self.grids[v] = g
        return g

    def _grid_array(self):
        arr = (Grid * self.V)(*[g.c for g in self.grids])
        return arr

    def sweep(self, v, levels, T=0.05, max_nb=0, seed=0):
        nsp = self.grids[v].c.gw * self.grids[v].c.gh
        out = np.zeros((nsp, 4), np.float64)
        arr = self._grid_array()
        rc = lib().lfdo_sweep_view(self.V, _p(self.images), _p(self.cams), self.range[0], self.range[1],
                                   C.cast(arr, C.c_void_p), v, levels, T, max_nb, seed, _p(out))
        if rc:
            raise ValueError(f"sweep error {rc}")
        return out

    def rasterize(self, v, planes):
        out = np.zeros(self.W * self.H, np.float32)
        lib().lfdo_rasterize(_p(self.cams[v]), C.byref(self.grids[v].c), _p(np.ascontiguousarray(planes)), _p(out))
        return out.reshape(self.H, self.W)

    def refine_iteration(self, l, planes_all, depth_all, sigma, size_init, alpha=0.075, eta=0.5, steps_init=5,
                         max_nb=0, flags=(1, 1, 1)):
        planes_all = np.ascontiguousarray(planes_all, np.float64)
        depth_all = np.ascontiguousarray(depth_all, np.float32)
        out = np.zeros_like(planes_all)
        acc = np.zeros(1, np.uint64)
        e = Energy(sigma, alpha, eta, size_init, steps_init, 5, max_nb, *flags)
        arr = self._grid_array()
        rc = lib().lfdo_refine_iteration(self.V, _p(self.cams), self.range[0], self.range[1], C.cast(arr, C.c_void_p),
                                         C.byref(e), _p(planes_all), _p(depth_all), l, _p(out), _p(acc))
        if rc:
            raise ValueError(f"refine error {rc}")
        return out, int(acc[0])
