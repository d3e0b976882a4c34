// Bit-exact ports of the glibc 2.39 exp / expf that the reference calls (x86-64, FMA IFUNC
// variants __exp_fma / __expf_fma), usable on host and device.
//
// Why: the refinement energy (refine.hpp:36 depth_consistency, :149 photo weight, :158
// visibility) calls std::exp(double) and the colour weights (superpixel.hpp:347) call
// std::exp(float).  CUDA's exp/expf differ from glibc in the last bit on a fraction of inputs,
// which would perturb energies and flip near-ties.  These ports reproduce glibc's algorithm
// (ARM optimized-routines exp/expf, table sizes 128 / 32) with the FMA placement that GCC chose
// for the FMA variants, read off `objdump -d` of libm.so.6; tables are the
// libm bytes (libm_tables.h).  tests/test_libm_port.py checks them against the host libm
// (expf exhaustively over every float, exp on 2e8 samples); tests/test_gpu_math.py on device.
// Attribution and licence: the algorithms, constants and tables below are derived from the GNU C
// Library 2.39 (sysdeps/ieee754/dbl-64/e_exp.c + e_exp_data.c, sysdeps/ieee754/flt-32/e_expf.c,
// e_exp2f_data.c, e_powf.c + e_powf_log2_data.c, s_cbrtf.c), Copyright (C) 1991-2024 Free
// Software Foundation, Inc., distributed under the GNU Lesser General Public License v2.1 or
// later (https://www.gnu.org/licenses/lgpl-2.1.html).  The exp / expf / powf routines in glibc
// originate from ARM Optimized Routines (Copyright (c) 2017-2018 Arm Ltd., MIT licence).  This
// file is a derivative work under those terms; it is compiled into liblfdg.so only so that the
// GPU reproduces the host libm bit for bit.
#pragma once

#include <math.h>
#include <stdint.h>

#include "libm_tables.h"

#if defined(__CUDACC__)
#define LFDG_HD __host__ __device__ __forceinline__
#else
#define LFDG_HD inline
#endif

namespace lfdg {
namespace libm {

#if defined(__CUDACC__)
__device__ const __align__(16) uint64_t kExpTabDev[256] = LFDG_EXP_TAB_INIT;
__device__ const uint64_t kExpfTabDev[32] = LFDG_EXPF_TAB_INIT;
#endif
static const uint64_t kExpTabHost[256] = LFDG_EXP_TAB_INIT;
static const uint64_t kExpfTabHost[32] = LFDG_EXPF_TAB_INIT;

LFDG_HD uint64_t exp_tab(unsigned i) {
#if defined(__CUDA_ARCH__)
    return __ldg(reinterpret_cast<const unsigned long long*>(&kExpTabDev[i]));
#else
    return kExpTabHost[i];
#endif
}
LFDG_HD uint64_t expf_tab(unsigned i) {
#if defined(__CUDA_ARCH__)
    return __ldg(reinterpret_cast<const unsigned long long*>(&kExpfTabDev[i]));
#else
    return kExpfTabHost[i];
#endif
}

LFDG_HD uint64_t as_u64(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    union {
        double d;
        uint64_t u;
    } v;
    v.d = x;
    return v.u;
#endif
}
LFDG_HD double as_f64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)x);
#else
    union {
        double d;
        uint64_t u;
    } v;
    v.u = x;
    return v.d;
#endif
}
LFDG_HD uint32_t as_u32(float x) {
#if defined(__CUDA_ARCH__)
    return (uint32_t)__float_as_uint(x);
#else
    union {
        float f;
        uint32_t u;
    } v;
    v.f = x;
    return v.u;
#endif
}

LFDG_HD double fma_(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

// __exp_fma (glibc sysdeps/ieee754/dbl-64/e_exp.c, x86-64 FMA build).  `tab` (nullable) is a
// copy of the 256-entry table, e.g. staged in shared memory by a hot kernel.
LFDG_HD double exp_with(double x, const uint64_t* tab) {
    const double kInvLn2N = 0x1.71547652b82fep+7;
    const double kShift = 0x1.8p+52;
    const double kNegLn2hiN = -0x1.62e42fefa0000p-8;
    const double kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    // exp(x) < 2^-1076 for x <= -746: glibc's specialcase rounds it to +0 (checked against libm
    // over [-1100, -700], tests/test_libm_port.py).  Early out: frequent in the visibility term.
    if (x <= -746.0) return 0.0;
    const uint64_t ux = as_u64(x);
    uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ff;
    if (abstop - 0x3c9u > 0x3eu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x;  // |x| < 2^-54
        if (abstop > 0x408u) {                                 // |x| >= 1024
            if (ux == 0xfff0000000000000ull) return 0.0;
            if (abstop == 0x7ffu) return 1.0 + x;
            if (ux >> 63) return 0.0;       // __math_uflow: 0x1p-767 * 0x1p-767
            return as_f64(0x7ff0000000000000ull);  // __math_oflow
        }
        abstop = 0;  // 512 <= |x| < 1024: specialcase below
    }
    double kd = fma_(x, kInvLn2N, kShift);  // z = InvLn2N * x; kd = z + Shift (contracted)
    const uint64_t ki = as_u64(kd);
    kd = kd - kShift;
    const double r = fma_(kd, kNegLn2loN, fma_(kd, kNegLn2hiN, x));
    const unsigned idx = 2u * (unsigned)(ki & 127u);
    const uint64_t top = ki << 45;
    const double tail = as_f64(tab ? tab[idx] : exp_tab(idx));
    uint64_t sbits = (tab ? tab[idx + 1] : exp_tab(idx + 1)) + top;
    const double r2 = r * r;
    const double tmp = fma_(r2 * r2, fma_(r, C5, C4), fma_(fma_(r, C3, C2), r2, r + tail));
    if (abstop == 0) {
        if ((ki & 0x80000000ull) == 0) {
            sbits -= 1009ull << 52;
            const double scale = as_f64(sbits);
            return 0x1p1009 * fma_(scale, tmp, scale);
        }
        sbits += 1022ull << 52;
        const double scale = as_f64(sbits);
        const double t = scale * tmp;
        double y = scale + t;
        if (y < 1.0) {
            const double hi = y + 1.0;
            double lo = (scale - y) + t;
            lo = ((1.0 - hi) + y) + lo;
            y = (lo + hi) - 1.0;
            if (y == 0.0) y = 0.0;
        }
        return 0x1p-1022 * y;
    }
    const double scale = as_f64(sbits);
    return fma_(scale, tmp, scale);
}

LFDG_HD double exp(double x) { return exp_with(x, nullptr); }

// The same function restricted to !(x > 0) (every exp argument of the energy is minus a
// square, refine.hpp:36/149/158): identical results (checked against libm on CPU and GPU),
// with the branch structure reduced to the cases that can occur and the polynomial constants
// read from constant memory, so the hot loop does not rematerialise them per call.
#if defined(__CUDACC__)
static __constant__ double kExpC[8] = {0x1.71547652b82fep+7, 0x1.8p+52, -0x1.62e42fefa0000p-8,
                                       -0x1.cf79abc9e3b3ap-47, 0x1.ffffffffffdbdp-2, 0x1.555555555543cp-3,
                                       0x1.55555cf172b91p-5, 0x1.1111167a4d017p-7};
#endif
static const double kExpCHost[8] = {0x1.71547652b82fep+7, 0x1.8p+52, -0x1.62e42fefa0000p-8,
                                    -0x1.cf79abc9e3b3ap-47, 0x1.ffffffffffdbdp-2, 0x1.555555555543cp-3,
                                    0x1.55555cf172b91p-5, 0x1.1111167a4d017p-7};
#if defined(__CUDA_ARCH__)
#define LFDG_EXPC(i) kExpC[i]
#else
#define LFDG_EXPC(i) kExpCHost[i]
#endif

LFDG_HD double exp_nonpos(double x) {
    if (x <= -746.0) return 0.0;              // < 2^-1076: glibc rounds to +0
    if (!(x <= -0x1p-54)) return 1.0 + x;     // |x| < 2^-54 (abstop < 0x3c9), -0.0, NaN
    double kd = fma_(x, LFDG_EXPC(0), LFDG_EXPC(1));
    const uint64_t ki = as_u64(kd);
    kd = kd - LFDG_EXPC(1);
    const double r = fma_(kd, LFDG_EXPC(3), fma_(kd, LFDG_EXPC(2), x));
    const unsigned idx = 2u * (unsigned)(ki & 127u);
#if defined(__CUDA_ARCH__)
    const ulonglong2 te = __ldg(reinterpret_cast<const ulonglong2*>(&kExpTabDev[idx]));  // (tail, sbits) pair
    const double tail = as_f64(te.x);
    uint64_t sbits = te.y + (ki << 45);
#else
    const double tail = as_f64(exp_tab(idx));
    uint64_t sbits = exp_tab(idx + 1) + (ki << 45);
#endif
    const double r2 = r * r;
    const double tmp = fma_(r2 * r2, fma_(r, LFDG_EXPC(7), LFDG_EXPC(6)), fma_(fma_(r, LFDG_EXPC(5), LFDG_EXPC(4)), r2, r + tail));
    if (x <= -512.0) {  // specialcase, k < 0 (abstop == 0 for 512 <= |x| < 1024)
        sbits += 1022ull << 52;
        const double scale = as_f64(sbits);
        const double t = scale * tmp;
        double y = scale + t;
        if (y < 1.0) {
            const double hi = y + 1.0;
            double lo = (scale - y) + t;
            lo = ((1.0 - hi) + y) + lo;
            y = (lo + hi) - 1.0;
            if (y == 0.0) y = 0.0;
        }
        return 0x1p-1022 * y;
    }
    const double scale = as_f64(sbits);
    return fma_(scale, tmp, scale);
}


#if defined(__CUDACC__)
// exp_nonpos split for the refinement's hot loop: exp_nonpos_in_core(x) tells, from the high
// word alone (integer pipe), whether x lies in (-512, -2^-54] where exp_nonpos takes neither
// early exit nor the specialcase; exp_nonpos_core(x) is exp_nonpos's main path for that
// range (the same operations and constants, so the same result).  Other x go to exp_nonpos.
__device__ __forceinline__ bool exp_nonpos_in_core(double x) {
    return (unsigned)__double2hiint(x) - 0xBC900000u < 0x03F00000u;  // hi in [hi(-2^-54), hi(-512))
}
__device__ __forceinline__ double exp_nonpos_core_kd(double x) { return fma_(x, LFDG_EXPC(0), LFDG_EXPC(1)); }
// the main path from kd = exp_nonpos_core_kd(x); the result is < 2^((n >> 7) + 1) for
// n = (int)lo(kd) = round(x 128 / ln 2) (table scale 2^(n/128) < 2^((n >> 7) + 1) / 1.0054, times
// 1 + tmp with |tmp| < 0.0028)
__device__ __forceinline__ double exp_nonpos_core_from(double kd, double x) {
    const uint64_t ki = as_u64(kd);
    kd = kd - LFDG_EXPC(1);
    const double r = fma_(kd, LFDG_EXPC(3), fma_(kd, LFDG_EXPC(2), x));
    const unsigned idx = 2u * (unsigned)(ki & 127u);
    const ulonglong2 te = __ldg(reinterpret_cast<const ulonglong2*>(&kExpTabDev[idx]));  // (tail, sbits)
    const double tail = as_f64(te.x);
    const uint64_t sbits = te.y + (ki << 45);
    const double r2 = r * r;
    const double tmp = fma_(r2 * r2, fma_(r, LFDG_EXPC(7), LFDG_EXPC(6)), fma_(fma_(r, LFDG_EXPC(5), LFDG_EXPC(4)), r2, r + tail));
    const double scale = as_f64(sbits);
    return fma_(scale, tmp, scale);
}
__device__ __forceinline__ double exp_nonpos_core(double x) { return exp_nonpos_core_from(exp_nonpos_core_kd(x), x); }
// the same with the (tail, sbits) table in shared memory (a copy of kExpTabDev)
__device__ __forceinline__ double exp_nonpos_core_tab(double x, const ulonglong2* tab) {
    double kd = exp_nonpos_core_kd(x);
    const uint64_t ki = as_u64(kd);
    kd = kd - LFDG_EXPC(1);
    const double r = fma_(kd, LFDG_EXPC(3), fma_(kd, LFDG_EXPC(2), x));
    const ulonglong2 te = tab[ki & 127u];
    const double tail = as_f64(te.x);
    const uint64_t sbits = te.y + (ki << 45);
    const double r2 = r * r;
    const double tmp = fma_(r2 * r2, fma_(r, LFDG_EXPC(7), LFDG_EXPC(6)), fma_(fma_(r, LFDG_EXPC(5), LFDG_EXPC(4)), r2, r + tail));
    const double scale = as_f64(sbits);
    return fma_(scale, tmp, scale);
}
#endif

// __expf_fma (glibc sysdeps/ieee754/flt-32/e_expf.c, x86-64 FMA build).
LFDG_HD float expf(float x) {
    const double kShift = 0x1.8p+52;
    const double kInvLn2N = 0x1.71547652b82fep+5;
    const double C0 = 0x1.c6af84b912394p-20, C1 = 0x1.ebfce50fac4f3p-13, C2 = 0x1.62e42ff0c52d6p-6;
    const uint32_t ux = as_u32(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    const double xd = (double)x;
    if (abstop > 0x42au) {
        if (ux == 0xff800000u) return 0.0f;
        if (abstop > 0x7f7u) return x + x;
        if (x > 0x1.62e42ep6f) return (float)as_f64(0x7ff0000000000000ull);  // __math_oflowf
        if (x < -0x1.9fe368p6f) return 0.0f;                                // __math_uflowf
        if (x < -0x1.9d1d9ep6f) return 0x1p-149f;  // __math_may_uflowf: 0x1.4p-75f * 0x1.4p-75f
    }
    double kd = fma_(kInvLn2N, xd, kShift);
    const uint64_t ki = as_u64(kd);
    kd = kd - kShift;
    const double r = fma_(kInvLn2N, xd, -kd);
    const uint64_t t = expf_tab((unsigned)(ki & 31u)) + (ki << 47);
    const double s = as_f64(t);
    const double z = fma_(r, C0, C1);
    const double r2 = r * r;
    double y = fma_(r, C2, 1.0);
    y = fma_(z, r2, y);
    y = y * s;
    return (float)y;
}

// ---- powf / cbrtf for rgb_to_scaled_lab (image.hpp:70-95) -----------------------------------
// __powf_fma: glibc 2.39 sysdeps/ieee754/flt-32/e_powf.c (the ARM optimized-routines powf) as
// built for x86-64 with FMA (the IFUNC variant both hosts run).  FMA placement read off
// `objdump -d libm.so.6` (0x7df50); log2 table (16 x {invc, logc}) and polynomial constants
// copied from .rodata 0xb7f80 / 0xb8080; exp2 uses __exp2f_data (the expf table above).
#define LFDG_POWF_LOG2_TAB_INIT                                                                         \
    {0x1.661ec79f8f3bep+0, -0x1.efec65b963019p-2, 0x1.571ed4aaf883dp+0, -0x1.b0b6832d4fca4p-2,            \
     0x1.49539f0f010b0p+0, -0x1.7418b0a1fb77bp-2, 0x1.3c995b0b80385p+0, -0x1.39de91a6dcf7bp-2,            \
     0x1.30d190c8864a5p+0, -0x1.01d9bf3f2b631p-2, 0x1.25e227b0b8ea0p+0, -0x1.97c1d1b3b7af0p-3,            \
     0x1.1bb4a4a1a343fp+0, -0x1.2f9e393af3c9fp-3, 0x1.12358f08ae5bap+0, -0x1.960cbbf788d5cp-4,            \
     0x1.0953f419900a7p+0, -0x1.a6f9db6475fcep-5, 0x1.0000000000000p+0, 0x0.0p+0,                         \
     0x1.e608cfd9a47acp-1, 0x1.338ca9f24f53dp-4,  0x1.ca4b31f026aa0p-1, 0x1.476a9543891bap-3,             \
     0x1.b2036576afce6p-1, 0x1.e840b4ac4e4d2p-3,  0x1.9c2d163a1aa2dp-1, 0x1.40645f0c6651cp-2,             \
     0x1.886e6037841edp-1, 0x1.88e9c2c1b9ff8p-2,  0x1.767dcf5534862p-1, 0x1.ce0a44eb17bccp-2}
#define LFDG_CBRTF_FACTOR_INIT \
    {0x1.428a2f98d728ap-1, 0x1.965fea53d6e3cp-1, 0x1.0p+0, 0x1.428a2f98d728bp+0, 0x1.965fea53d6e3dp+0}
#if defined(__CUDACC__)
__device__ const __align__(16) double kPowfLog2Dev[32] = LFDG_POWF_LOG2_TAB_INIT;  // {invc, logc} x 16
__device__ const double kCbrtfFactorDev[5] = LFDG_CBRTF_FACTOR_INIT;
#endif
static const double kPowfLog2Host[32] = LFDG_POWF_LOG2_TAB_INIT;
static const double kCbrtfFactorHost[5] = LFDG_CBRTF_FACTOR_INIT;
LFDG_HD double powf_log2_tab(int i) {  // .rodata 0xb7f80: invc at 2i, logc at 2i + 1
#if defined(__CUDA_ARCH__)
    return __ldg(&kPowfLog2Dev[i]);
#else
    return kPowfLog2Host[i];
#endif
}
LFDG_HD double cbrtf_factor(int i) {  // .rodata 0xab1c0
#if defined(__CUDA_ARCH__)
    return __ldg(&kCbrtfFactorDev[i]);
#else
    return kCbrtfFactorHost[i];
#endif
}

// powf(x, y) for x > 0 (normal, subnormal, +inf) or NaN, and y finite and nonzero — the only
// operands rgb_to_scaled_lab produces ((v + 0.055) / 1.055 with v > 0.04045, y = 2.4).
LFDG_HD float powf_pos(float x, float y) {
    uint32_t ix = as_u32(x);
    if (ix >= 0x7f800000u) return x + y;  // +inf -> +inf for y > 0, NaN -> NaN
    if (ix < 0x00800000u) {               // subnormal x: normalise (e_powf.c)
        ix = as_u32(x * 0x1p23f) & 0x7fffffffu;
        ix -= 23u << 23;
    }
    // log2_inline
    const uint32_t tmp = ix - 0x3f330000u;
    const int i = (int)((tmp >> 19) & 15u);
    const uint32_t top = tmp & 0xff800000u;
    const uint32_t iz = ix - top;
    const int k = (int32_t)top >> 23;
    union {
        uint32_t u;
        float f;
    } zu;
    zu.u = iz;
    const double z = (double)zu.f;
    const double r = fma_(z, powf_log2_tab(2 * i), -1.0);
    const double y0 = (double)k + powf_log2_tab(2 * i + 1);
    double yl = fma_(r, 0x1.27616c9496e0bp-2, -0x1.71969a075c67ap-2);
    const double p = fma_(r, 0x1.ec70a6ca7baddp-2, -0x1.7154748bef6c8p-1);
    const double r2 = r * r;
    double q = fma_(r, 0x1.71547652ab82bp+0, y0);
    const double r4 = r2 * r2;
    q = fma_(r2, p, q);
    yl = fma_(yl, r4, q);
    const double ylogx = (double)y * yl;
    if (((as_u64(ylogx) >> 47) & 0xffffu) > 0x80beu) {  // |y log2 x| >= 126
        if (ylogx > 0x1.fffffffd1d571p+6) return (float)as_f64(0x7ff0000000000000ull);  // __math_oflowf
        if (ylogx <= -150.0) return 0.0f;                                               // __math_uflowf
        if (ylogx < -149.0) return 0x1p-149f;  // __math_may_uflowf: 0x1.4p-75f * 0x1.4p-75f
    }
    // exp2_inline (sign_bias 0)
    double kd = ylogx + 0x1.8p+47;
    const uint64_t ki = as_u64(kd);
    kd = kd - 0x1.8p+47;
    const double rr = ylogx - kd;
    const uint64_t t = expf_tab((unsigned)(ki & 31u)) + (ki << 47);
    const double sc = as_f64(t);
    const double zz = fma_(rr, 0x1.c6af84b912394p-5, 0x1.ebfce50fac4f3p-3);
    const double rr2 = rr * rr;
    double yy = fma_(rr, 0x1.62e42ff0c52d6p-1, 1.0);
    yy = fma_(zz, rr2, yy);
    return (float)(yy * sc);
}

// cbrtf: glibc 2.39 sysdeps/ieee754/flt-32/s_cbrtf.c (double arithmetic, no FMA; constants and
// the factor table from .rodata 0x99f40 / 0xab1c0, operation order read off the disassembly).
LFDG_HD float cbrtf_(float x) {
    const uint32_t ux = as_u32(x) & 0x7fffffffu;
    if (ux == 0u || ux >= 0x7f800000u) return x + x;  // zero, inf, NaN
    // frexpf(|x|)
    int xe;
    union {
        uint32_t u;
        float f;
    } m;
    if (ux < 0x00800000u) {  // subnormal
        m.u = ux;
        m.f *= 0x1p25f;
        xe = (int)(m.u >> 23) - 126 - 25;
    } else {
        xe = (int)(ux >> 23) - 126;
        m.u = ux;
    }
    m.u = (m.u & 0x807fffffu) | (126u << 23);
    const double xm = (double)m.f;
    const float u = (float)(((0x1.6527f4927f555p-1 - 0x1.8832490c2feddp-3 * xm) * xm) + 0x1.f87bc378ed415p-2);
    const float t2 = (u * u) * u;
    const double ud = (double)u, t2d = (double)t2;
    const double ym = (((xm + xm) + t2d) * ud) / ((t2d + t2d) + xm) * cbrtf_factor(2 + xe % 3);
    const float r = (float)ym;
    // ldexpf(+-ym, xe / 3): ym in (0.5, 1.6], the scaled result is a normal float for every
    // finite x (|cbrt(x)| >= 2^-50)
    union {
        uint32_t u;
        float f;
    } o;
    o.f = r;
    o.u += (uint32_t)(xe / 3) << 23;
    return (as_u32(x) >> 31) ? -o.f : o.f;
}

// rgb_to_scaled_lab (image.hpp:70-95), float arithmetic in the reference's order.
LFDG_HD float srgb_to_linear(float v) { return v <= 0.04045f ? v / 12.92f : powf_pos((v + 0.055f) / 1.055f, 2.4f); }
LFDG_HD float lab_f(float t) {
    const float kEps = 216.f / 24389.f;
    const float kKappa = 24389.f / 27.f;
    return t > kEps ? cbrtf_(t) : (kKappa * t + 16.f) / 116.f;
}
LFDG_HD void rgb_to_scaled_lab(float r0, float g0, float b0, float& L, float& A, float& B) {
    const float r = srgb_to_linear(r0);
    const float g = srgb_to_linear(g0);
    const float b = srgb_to_linear(b0);
    const float xr = (0.4124564f * r + 0.3575761f * g + 0.1804375f * b) / 0.95047f;
    const float yr = (0.2126729f * r + 0.7151522f * g + 0.0721750f * b);
    const float zr = (0.0193339f * r + 0.1191920f * g + 0.9503041f * b) / 1.08883f;
    const float fx = lab_f(xr);
    const float fy = lab_f(yr);
    const float fz = lab_f(zr);
    L = (116.f * fy - 16.f) / 100.f;
    A = (500.f * (fx - fy)) / 100.f;
    B = (200.f * (fy - fz)) / 100.f;
}

}  // namespace libm
}  // namespace lfdg
