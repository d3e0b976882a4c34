"""Device ports of glibc exp/expf (csrc/glibc_math.cuh) against the host libm the reference uses."""
import ctypes
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _libm():
    L = ctypes.CDLL("libm.so.6")
    L.exp.restype = ctypes.c_double
    L.exp.argtypes = [ctypes.c_double]
    return L


def test_exp_matches_host_libm():
    from paper_1812_06856_b200 import _native as N

    rng = np.random.default_rng(7)
    x = np.concatenate([rng.uniform(-800, 5, 400000), rng.uniform(-745, -700, 100000), rng.uniform(-30, 0, 400000),
                        rng.uniform(-1100, 1100, 100000),
                        rng.integers(0, 2**63, 100000, dtype=np.int64).view(np.float64)])
    x = np.ascontiguousarray(x)
    out = np.zeros_like(x)
    N.check(N.lib().lfdg_selftest_exp(0, N.ptr(x), N.ptr(out), x.size))
    # numpy's exp is not glibc's; compare with the libm that the reference links
    L = _libm()
    want = np.array([L.exp(float(v)) for v in x])
    same = (out.view(np.uint64) == want.view(np.uint64)) | (np.isnan(out) & np.isnan(want))
    assert same.all(), f"{(~same).sum()} mismatches, e.g. x={x[~same][:3]}"


def test_expf_matches_host_libm_exhaustive_slice():
    from paper_1812_06856_b200 import _native as N

    # every float in [-110, 90] with a stride (the full exhaustive check runs on the CPU port)
    bits = np.arange(0, 2**32, 97, dtype=np.uint64).astype(np.uint32)
    x = np.ascontiguousarray(bits.view(np.float32))
    out = np.zeros_like(x)
    N.check(N.lib().lfdg_selftest_expf(0, N.ptr(x), N.ptr(out), x.size))
    L = ctypes.CDLL("libm.so.6")
    L.expf.restype = ctypes.c_float
    L.expf.argtypes = [ctypes.c_float]
    idx = np.random.default_rng(3).choice(x.size, 300000, replace=False)
    want = np.array([L.expf(float(x[i])) for i in idx], np.float32)
    got = out[idx]
    same = (got.view(np.uint32) == want.view(np.uint32)) | (np.isnan(got) & np.isnan(want))
    assert same.all(), f"{(~same).sum()} mismatches"


def test_exp_nonpos_matches_host_libm():
    from paper_1812_06856_b200 import _native as N

    rng = np.random.default_rng(11)
    x = np.concatenate([rng.uniform(-1100, 0, 300000), rng.uniform(-800, -500, 200000), rng.uniform(-1e-15, 0, 10000),
                        np.array([0.0, -0.0, -2.0**-54, -512.0, -745.1332191019411, -746.0, -1024.0, -np.inf])])
    x = np.ascontiguousarray(x)
    out = np.zeros_like(x)
    N.check(N.lib().lfdg_selftest_exp_nonpos(0, N.ptr(x), N.ptr(out), x.size))
    L = _libm()
    want = np.array([L.exp(float(v)) for v in x])
    assert np.array_equal(out.view(np.uint64), want.view(np.uint64))
