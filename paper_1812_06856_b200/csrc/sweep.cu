// Plane-sweep initialisation and rasterization on sm_100a.
//
//   k_sweep      sweep_view (sweep.hpp:112-139) + sweep_cost (sweep.hpp:85-107): one CTA per
//                (view, superpixel).  Phase A: one thread per depth hypothesis runs the cost
//                chain over the first target (member rays and colours staged in shared memory);
//                phase B completes the chain of the best partial hypothesis (its cost B);
//                phase C continues the others target by target, member-parallel, dropping a
//                hypothesis as soon as its partial cost exceeds B (exact: partial sums of
//                non-negative terms never exceed the final sum).  Every chain adds in exactly
//                the reference's (target, member-pixel) order, so costs are bit-identical; the
//                (cost, depth) argmin is a block reduction on a total order, which reproduces
//                "ties -> smaller depth" (sweep.hpp:130).  See the comment above k_sweep.
//   k_rasterize  rasterize (sweep.hpp:44-63): one thread per pixel.
//
// FP64 geometry follows geometry.hpp:70-111 operation by operation.  Two template switches
// drop operations that are exact identities for the camera set at hand (checked on the host,
// DESIGN.md "sweep"): kIdR when every rotation is exactly I (then R^T a = a and R w = w up to
// the sign of a zero, which cannot reach the cost: contains() treats -0 as 0 and the bilinear
// residual is squared), kCanonK when every K has K01 = K10 = K20 = K21 = 0 and K22 = 1 (then
// h.z = z whenever z > 0, which is the only case that is sampled).
#include <algorithm>
#include <cmath>

#include "context.h"

namespace lfdg {
namespace {

// Sample addressing (A/B switches): 32-bit texel indices, and the target image's base pointer
// made opaque to the compiler so that it stays in registers — it was rematerialised from
// (target id, W*H) with a 64-bit multiply chain on every sample (sweep 126 -> 116 ms at C3,
// 236 -> 217 ms at C5, 250 -> 243 ms on the converging rig).
#ifndef LFDG_SWEEP_ADDR32
#define LFDG_SWEEP_ADDR32 1
#endif
#ifndef LFDG_SWEEP_OPAQUE
#define LFDG_SWEEP_OPAQUE 1
#endif
#ifndef LFDG_SWEEP_PACK
#define LFDG_SWEEP_PACK 1
#endif

constexpr int kSweepCap = 1024;  // member pixels staged per chunk

// Packed f32x2 arithmetic (two colour channels per instruction).  Products go through
// fma.rn.f32x2(a, b, +0.0) and are added by a separate add.rn.f32x2: ptxas does not fuse that
// pair (it does fuse a plain mul.rn.f32x2 + add.rn.f32x2, even with --fmad=false), so every
// operation rounds as in the reference's SSE code.  fma(a, b, +0) equals the rounded product
// except that an exact zero product is +0: values can differ only in the sign of a zero, which
// cannot change a squared distance.
__device__ __forceinline__ unsigned long long f2pack(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 f2unpack(unsigned long long r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ unsigned long long f2sub(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2add(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2mul(unsigned long long a, unsigned long long b) {  // fma(a, b, +0)
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(0ull));
    return r;
}

// The row half of ImageBuffer::contains / bilinear (image.hpp:42-55) for sample row v: whether
// 0 <= v <= H - 1, the clamped y0 and fy = (float)(v - y0).
struct SampleRow {
    bool ok;
    int y0;
    float fy;
};
__device__ __forceinline__ SampleRow sample_row(int H, double v) {
    SampleRow r;
    r.ok = v >= 0.0 && v <= H - 1.0;
    int y0 = r.ok ? (int)floor(v) : 0;
    if (y0 >= H - 1) y0 = H - 2;
    if (y0 < 0) y0 = 0;
    r.y0 = y0;
    r.fy = (float)(v - y0);
    return r;
}

// Bilinear TSSD of one mapped sample (image.hpp:42-67, sweep.hpp:32-34, :99-103) given its row
// half: channels L, a packed, b scalar, each lerp `top = p00 + fx (p10 - p00)` etc. in the
// reference's order.
__device__ __forceinline__ float tssd_row(const float4* __restrict__ timg, int W, double u, const SampleRow& row,
                                          float4 ref, float T) {
    if (!(u >= 0.0 && row.ok && u <= W - 1.0)) return T;
    int x0 = (int)floor(u);
    if (x0 >= W - 1) x0 = W - 2;
    if (x0 < 0) x0 = 0;
    const int y0 = row.y0;
    const float fx = (float)(u - x0);
    const float fy = row.fy;
#if LFDG_SWEEP_ADDR32
    // 32-bit texel indices (a view has < 2^31 pixels, checked by set_views): two address
    // computations instead of a 64-bit multiply-add chain per sample
    const unsigned i0 = (unsigned)(y0 * W + x0);
    const float4* r0 = timg + i0;
    const float4* r1 = timg + (i0 + (unsigned)W);
#else
    const float4* r0 = timg + ((size_t)y0 * W + x0);
    const float4* r1 = r0 + W;
#endif
    const float4 p00 = __ldg(r0), p10 = __ldg(r0 + 1);
    const float4 p01 = __ldg(r1), p11 = __ldg(r1 + 1);
    const unsigned long long FX = f2pack(fx, fx), FY = f2pack(fy, fy);
    const unsigned long long a00 = f2pack(p00.x, p00.y), a10 = f2pack(p10.x, p10.y);
    const unsigned long long a01 = f2pack(p01.x, p01.y), a11 = f2pack(p11.x, p11.y);
    const unsigned long long top = f2add(a00, f2mul(FX, f2sub(a10, a00)));
    const unsigned long long bot = f2add(a01, f2mul(FX, f2sub(a11, a01)));
    const unsigned long long o01 = f2add(top, f2mul(FY, f2sub(bot, top)));
    const float t2 = p00.z + fx * (p10.z - p00.z), b2 = p01.z + fx * (p11.z - p01.z);
    const float o2 = t2 + fy * (b2 - t2);
    // color_dist2 (image.hpp:13-16): (d0 d0 + d1 d1) + d2 d2, d = ref - sample
    const unsigned long long d01 = f2sub(f2pack(ref.x, ref.y), o01);
    const float2 sq = f2unpack(f2mul(d01, d01));
    const float d2c = ref.z - o2;
    const float dist = (sq.x + sq.y) + d2c * d2c;
    return dist < T ? dist : T;
}

__device__ __forceinline__ float tssd_at(const float4* __restrict__ timg, int W, int H, double u, double v, float4 ref,
                                         float T) {
    return tssd_row(timg, W, u, sample_row(H, v), ref, T);
}

template <bool kIdR, bool kCanonK>
__device__ __forceinline__ float sweep_sample(const Cam& rc, const Cam& tc, const float4* __restrict__ timg, int W,
                                              int H, double d, double vx, double vy, float4 ref, float T) {
    // backproject (geometry.hpp:70-73): world = R^T (d * ray - t)
    const double a0 = d * vx - rc.t[0];
    const double a1 = d * vy - rc.t[1];
    const double a2 = d - rc.t[2];
    double w0, w1, w2;
    if (kIdR) {
        w0 = a0;
        w1 = a1;
        w2 = a2;
    } else {
        w0 = (rc.R[0] * a0 + rc.R[3] * a1) + rc.R[6] * a2;
        w1 = (rc.R[1] * a0 + rc.R[4] * a1) + rc.R[7] * a2;
        w2 = (rc.R[2] * a0 + rc.R[5] * a1) + rc.R[8] * a2;
    }
    // project (geometry.hpp:76-80): x = R X + t, h = K x
    double c0, c1, c2;
    if (kIdR) {
        c0 = w0 + tc.t[0];
        c1 = w1 + tc.t[1];
        c2 = w2 + tc.t[2];
    } else {
        c0 = ((tc.R[0] * w0 + tc.R[1] * w1) + tc.R[2] * w2) + tc.t[0];
        c1 = ((tc.R[3] * w0 + tc.R[4] * w1) + tc.R[5] * w2) + tc.t[1];
        c2 = ((tc.R[6] * w0 + tc.R[7] * w1) + tc.R[8] * w2) + tc.t[2];
    }
    if (c2 <= 0) return T;  // behind the target camera (geometry.hpp:109)
    double hx, hy, hz;
    if (kCanonK) {
        hx = tc.K[0] * c0 + tc.K[2] * c2;
        hy = tc.K[4] * c1 + tc.K[5] * c2;
        hz = c2;
    } else {
        hx = (tc.K[0] * c0 + tc.K[1] * c1) + tc.K[2] * c2;
        hy = (tc.K[3] * c0 + tc.K[4] * c1) + tc.K[5] * c2;
        hz = (tc.K[6] * c0 + tc.K[7] * c1) + tc.K[8] * c2;
    }
    // u = hx / hz, v = hy / hz: one correctly rounded reciprocal and a Markstein correction per
    // quotient, which yields the correctly rounded quotient (as in sweep_chunk_fast)
    const double rz = 1.0 / hz;
    const double qx = hx * rz, qy = hy * rz;
    const double u = __fma_rn(__fma_rn(-qx, hz, hx), rz, qx);
    const double v = __fma_rn(__fma_rn(-qy, hz, hy), rz, qy);
    return tssd_at(timg, W, H, u, v, ref, T);
}

// The kIdR && kCanonK inner loop over a staged chunk, for one (hypothesis, target).  With every
// rotation exactly I, the target-frame z = (d - t_ref.z) + t_t.z is the same for every member
// pixel, so h.z = z and K02 z, K12 z are hoisted, and u = hx / z, v = hy / z use z's correctly
// rounded reciprocal plus one Markstein correction (q = hx rz; r = fma(-q, z, hx) exact;
// q' = fma(r, rz, q)), which is the correctly rounded quotient for operands away from
// overflow/underflow.  The cost chain is the reference's, sample by sample.
__device__ __forceinline__ double sweep_chunk_fast(double cost, const double2* __restrict__ s_ray,
                                                   const float4* __restrict__ s_ref, int cn,
                                                   const float4* __restrict__ timg, int W, int H, double d,
                                                   const Cam& rc, const Cam& tc, float T) {
    const double rt0 = rc.t[0], rt1 = rc.t[1];
    const double z = (d - rc.t[2]) + tc.t[2];
    if (!(z > 0)) {
        for (int i = 0; i < cn; ++i) cost += (double)T;
        return cost;
    }
    const double tt0 = tc.t[0], tt1 = tc.t[1];
    const double K00 = tc.K[0], K11 = tc.K[4];
    const double Kz0 = tc.K[2] * z, Kz1 = tc.K[5] * z;
    const double rz = 1.0 / z;
    // v depends on the member's row only (ray.y; K01 = 0 under kCanonK): members are in row-major
    // order, so the row half of the sample is recomputed only when the row changes (the branch is
    // uniform: every thread of the CTA reads the same member)
    double prev_ry = NAN;
    SampleRow row{false, 0, 0.f};
    for (int i = 0; i < cn; ++i) {
        const double2 ray = s_ray[i];
        if (!(ray.y == prev_ry)) {
            prev_ry = ray.y;
            const double hy = K11 * ((d * ray.y - rt1) + tt1) + Kz1;
            const double qy = hy * rz;
            row = sample_row(H, __fma_rn(__fma_rn(-qy, z, hy), rz, qy));
        }
        const double hx = K00 * ((d * ray.x - rt0) + tt0) + Kz0;
        const double qx = hx * rz;
        const double u = __fma_rn(__fma_rn(-qx, z, hx), rz, qx);
        cost += (double)tssd_row(timg, W, u, row, s_ref[i], T);
    }
    return cost;
}

// One member-parallel sample for hypothesis depth d (fast path: the per-(hypothesis, target)
// z, 1/z, K02 z, K12 z precomputed), bit-identical to sweep_chunk_fast's.
__device__ __forceinline__ float sample_fast(const Cam& rc, const Cam& tc, const float4* __restrict__ timg, int W, int H,
                                             double d, double z, double rz, double kz0, double kz1, double rx,
                                             double ry, float4 ref, float T) {
    if (!(z > 0)) return T;
    const double hx = tc.K[0] * ((d * rx - rc.t[0]) + tc.t[0]) + kz0;
    const double hy = tc.K[4] * ((d * ry - rc.t[1]) + tc.t[1]) + kz1;
    const double qx = hx * rz, qy = hy * rz;
    const double u = __fma_rn(__fma_rn(-qx, z, hx), rz, qx);
    const double v = __fma_rn(__fma_rn(-qy, z, hy), rz, qy);
    return tssd_at(timg, W, H, u, v, ref, T);
}

// sample_fast with its operands packed in shared memory: the target's (K00, t_ref.x), (t_t.x,
// K11), (t_ref.y, t_t.y) and the hypothesis' (d, z), (1/z, K02 z), (K12 z, -) — 16-byte loads
// per sample instead of ten 8-byte ones; same operations in the same order (sweep -6 / -3.5 / -5.7 %
// at C3 / C5 / C4).
__device__ __forceinline__ float sample_fast_packed(const double2* __restrict__ tcc, const double2* __restrict__ hp,
                                                    const float4* __restrict__ timg, int W, int H, double rx, double ry,
                                                    float4 ref, float T) {
    const double2 dz = hp[0];
    if (!(dz.y > 0)) return T;
    const double2 rk = hp[1], k1 = hp[2];
    const double2 c0 = tcc[0], c1 = tcc[1], c2 = tcc[2];
    const double hx = c0.x * ((dz.x * rx - c0.y) + c1.x) + rk.y;
    const double hy = c1.y * ((dz.x * ry - c2.x) + c2.y) + k1.x;
    const double qx = hx * rk.x, qy = hy * rk.x;
    const double u = __fma_rn(__fma_rn(-qx, dz.y, hx), rk.x, qx);
    const double v = __fma_rn(__fma_rn(-qy, dz.y, hy), rk.x, qy);
    return tssd_at(timg, W, H, u, v, ref, T);
}

constexpr int kGroup = 32;       // hypotheses per member-parallel pass
constexpr int kTilePitch = 260;  // floats per tile row: 16-byte rows, conflict-free float4 folds

// Block-wide argmin of (cost, depth) over the hypotheses in list[0, cnt) (or all `levels` when
// list == nullptr), the reference's "ties -> smaller depth" order (sweep.hpp:128-133).
__device__ int block_argmin(const double* s_P, const double* s_d, const int* list, int cnt, double* red_c,
                            double* red_d, int* red_k) {
    double bc = INFINITY, bd = INFINITY;
    int bk = -1;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        const int k = list ? list[q] : q;
        const double c = s_P[k], d = s_d[k];
        if (bk < 0 || c < bc || (c == bc && d < bd)) {
            bc = c;
            bd = d;
            bk = k;
        }
    }
    for (int off = 16; off; off >>= 1) {
        const double oc = __shfl_xor_sync(LFDG_FULL_MASK, bc, off);
        const double od = __shfl_xor_sync(LFDG_FULL_MASK, bd, off);
        const int ok = __shfl_xor_sync(LFDG_FULL_MASK, bk, off);
        if (ok >= 0 && (bk < 0 || oc < bc || (oc == bc && od < bd))) {
            bc = oc;
            bd = od;
            bk = ok;
        }
    }
    const int warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        red_c[warp] = bc;
        red_d[warp] = bd;
        red_k[warp] = bk;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nwarps; ++w)
            if (red_k[w] >= 0 && (bk < 0 || red_c[w] < bc || (red_c[w] == bc && red_d[w] < bd))) {
                bc = red_c[w];
                bd = red_d[w];
                bk = red_k[w];
            }
        red_k[0] = bk;
    }
    __syncthreads();
    const int r = red_k[0];
    __syncthreads();
    return r;
}

// Ordered block compaction: list <- the k in [0, levels) with keep(k); returns the count.
template <typename Pred>
__device__ int block_compact(int levels, int* list, int* s_cnt, Pred keep) {
    int base = 0;
    for (int k0 = 0; k0 < levels; k0 += blockDim.x) {
        const int k = k0 + threadIdx.x;
        const bool f = k < levels && keep(k);
        const unsigned m = __ballot_sync(LFDG_FULL_MASK, f);
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) s_cnt[warp] = __popc(m);
        __syncthreads();
        int off = base;
        for (int w = 0; w < warp; ++w) off += s_cnt[w];
        int tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += s_cnt[w];
        if (f) list[off + __popc(m & ((1u << lane) - 1u))] = k;
        __syncthreads();
        base += tot;
    }
    return base;
}

// sweep_view (sweep.hpp:112-139) for one (view, superpixel): one CTA, the depth hypotheses of
// sample_inverse_depths in shared memory.  Exact pruning, same winner as the dense argmin:
//   A  every hypothesis runs the reference's cost chain over the first target (one thread per
//      hypothesis, rays / colours staged in shared memory);
//   B  the hypothesis h* with the smallest partial cost completes its chain: B = cost(h*);
//   C  the others continue target by target while their partial cost is <= B.  The chain adds
//      non-negative terms, so with round-to-nearest each partial cost is <= the final one
//      (fl(a + x) >= a for x >= 0, monotone in a): a partial cost > B proves cost > B >= the
//      minimum, so that hypothesis can neither win nor tie.
// B and C run member-parallel: each thread samples one member pixel for up to kGroup
// hypotheses into a shared tile, then one thread per hypothesis folds the tile row in member
// order — the same sequential FP64 chain, sample by sample, as sweep_cost (sweep.hpp:85-107).
// Tuning switches (A/B builds only): resident CTAs per SM, the sample counter, the CTA order.
#ifndef LFDG_SWEEP_MINB
#define LFDG_SWEEP_MINB 4
#endif
#ifndef LFDG_SWEEP_COUNT
#define LFDG_SWEEP_COUNT 1
#endif
#ifndef LFDG_SWEEP_ROWMAJOR
#define LFDG_SWEEP_ROWMAJOR 1
#endif
template <bool kIdR, bool kCanonK, bool kScratch>
__global__ void __launch_bounds__(256, LFDG_SWEEP_MINB) k_sweep(const float4* __restrict__ lab, int W, int H, int nsp, int v0,
                                               const Cam* __restrict__ cams, const int* __restrict__ targets,
                                               int n_targets, const int32_t* __restrict__ moff,
                                               const int32_t* __restrict__ mpix, int levels, double inv_lo,
                                               double inv_hi, double step, float T, uint64_t seed, int gw,
                                               int n_views, double4* planes, unsigned long long* samples,
                                               unsigned char* __restrict__ gscr, size_t slot_bytes, int cta0) {
    extern __shared__ __align__(16) unsigned char smem[];
    // [staging / tile union][cams][s_d][s_P][list]
    constexpr size_t kUnion = kSweepCap * (sizeof(double2) + sizeof(float4)) > kGroup * kTilePitch * sizeof(float)
                                  ? kSweepCap * (sizeof(double2) + sizeof(float4))
                                  : kGroup * kTilePitch * sizeof(float);
    double2* s_ray = reinterpret_cast<double2*>(smem);
    float4* s_ref = reinterpret_cast<float4*>(smem + kSweepCap * sizeof(double2));
    float* s_tile = reinterpret_cast<float*>(smem);
    Cam* s_cam = reinterpret_cast<Cam*>(smem + kUnion);
    // the per-hypothesis arrays: in shared memory, or (levels beyond the shared-memory budget) in
    // this CTA's slot of a global scratch buffer, the launch then covering CTAs [cta0, cta0 + grid)
    double* s_d;
    int* s_tmp;  // prune-list staging: the (then free) sample tile, or the scratch slot
    if (kScratch) {
        s_d = reinterpret_cast<double*>(gscr + (size_t)blockIdx.x * slot_bytes);
        s_tmp = reinterpret_cast<int*>(s_d + 2 * (size_t)levels) + levels;
    } else {
        s_d = reinterpret_cast<double*>(smem + kUnion + (size_t)(n_targets + 1) * sizeof(Cam));
        s_tmp = reinterpret_cast<int*>(smem);
    }
    double* s_P = s_d + levels;
    int* s_list = reinterpret_cast<int*>(s_P + levels);
    __shared__ double red_c[32], red_d[32];
    __shared__ int red_k[32];
    __shared__ double g_d[kGroup], g_z[kGroup], g_rz[kGroup], g_kz0[kGroup], g_kz1[kGroup];
    __shared__ int g_h[kGroup];
    __shared__ __align__(16) double2 g_pk[kGroup][3];  // LFDG_SWEEP_PACK: (d, z), (1/z, K02 z), (K12 z, -)
    __shared__ __align__(16) double2 s_tcc[3];         // LFDG_SWEEP_PACK: the target's constants

    // CTA order (superpixel row, view, superpixel column): the CTAs resident at any time sweep the
    // same band of image rows in every view, so the target-image rows they gather (the epipolar
    // band of a rectified rig) stay L2-resident across source views instead of every view
    // re-streaming its targets from HBM.
    int sp, view;
    if (LFDG_SWEEP_ROWMAJOR) {
        const int row_tasks = n_views * gw;
        const int cta = (kScratch ? cta0 : 0) + (int)blockIdx.x;
        const int grow = cta / row_tasks;
        const int rem = cta - grow * row_tasks;
        sp = grow * gw + rem % gw;
        view = v0 + rem / gw;
    } else {
        const int cta = (kScratch ? cta0 : 0) + (int)blockIdx.x;
        sp = cta % nsp;
        view = v0 + cta / nsp;
    }
    const size_t hw = (size_t)W * H;
    const int* tg = targets + (size_t)view * n_targets;
    for (int i = threadIdx.x; i < n_targets + 1; i += blockDim.x) s_cam[i] = cams[i == 0 ? view : tg[i - 1]];
    const int32_t m0 = moff[(size_t)view * (nsp + 1) + sp];
    const int n = moff[(size_t)view * (nsp + 1) + sp + 1] - m0;
    const int32_t* mem = mpix + (size_t)view * hw + m0;
    const float4* rimg = lab + (size_t)view * hw;
    __syncthreads();
    const Cam& rc = s_cam[0];

    // ---- A: hypotheses (sample_inverse_depths, geometry.hpp:116-130) and the first target
    const uint64_t s0 = derive_stream_state(seed, (uint64_t)view, (uint64_t)sp);
    const int per = (levels + blockDim.x - 1) / blockDim.x;
    for (int r = 0; r < per; ++r) {
        const int k = r * blockDim.x + threadIdx.x;
        const bool active = k < levels;
        double d = 0;
        if (active) {
            double inv = inv_lo + step * k + u64_to_unit(splitmix_at(s0, (uint64_t)k)) * step;
            if (inv > inv_hi) inv = inv_hi;
            d = 1.0 / inv;
        }
        double cost = 0;
        if (n_targets > 0) {
            const Cam& tc = s_cam[1];
            const float4* timg = lab + (size_t)tg[0] * hw;
            if (LFDG_SWEEP_OPAQUE) asm volatile("mov.b64 %0, %0;" : "+l"(timg));  // kept, not recomputed per sample
            for (int c0 = 0; c0 < n; c0 += kSweepCap) {
                if (n > kSweepCap || (c0 == 0 && r == 0)) {
                    __syncthreads();
                    const int cn = min(kSweepCap, n - c0);
                    for (int i = threadIdx.x; i < cn; i += blockDim.x) {
                        const int p = mem[c0 + i];
                        double rx, ry;
                        cam_ray(rc, (double)(p % W), (double)(p / W), rx, ry);
                        s_ray[i] = make_double2(rx, ry);
                        s_ref[i] = rimg[p];
                    }
                    __syncthreads();
                }
                if (!active) continue;
                const int cn = min(kSweepCap, n - c0);
                if (kIdR && kCanonK) {
                    cost = sweep_chunk_fast(cost, s_ray, s_ref, cn, timg, W, H, d, rc, tc, T);
                } else {
                    for (int i = 0; i < cn; ++i) {
                        const double2 ray = s_ray[i];
                        cost += (double)sweep_sample<kIdR, kCanonK>(rc, tc, timg, W, H, d, ray.x, ray.y, s_ref[i], T);
                    }
                }
            }
        }
        if (active) {
            s_d[k] = d;
            s_P[k] = cost;
        }
    }
    __syncthreads();

    // Continue the chains of list[0, cnt) over targets [t_begin, n_targets), pruning after
    // each target (prune: keep only partial cost <= B).  Returns the surviving count.
    // work counter: samples of this superpixel's sweep, kept in shared memory by thread 0 (a
    // register live across the whole kernel measurably slowed it)
    __shared__ unsigned long long s_samples;
    if (threadIdx.x == 0) s_samples = n_targets > 0 ? (unsigned long long)levels * n : 0;  // phase A
    auto advance = [&](int cnt, int t_begin, bool prune, double B) -> int {
        for (int ti = t_begin; ti < n_targets && cnt > 0; ++ti) {
            if (LFDG_SWEEP_COUNT && threadIdx.x == 0) s_samples += (unsigned long long)cnt * n;
            const Cam& tc = s_cam[ti + 1];
            const float4* timg = lab + (size_t)tg[ti] * hw;
            if (LFDG_SWEEP_OPAQUE) asm volatile("mov.b64 %0, %0;" : "+l"(timg));  // kept, not recomputed per sample
            if (LFDG_SWEEP_PACK && threadIdx.x == 0) {  // read after the chunk loop's first barrier
                s_tcc[0] = make_double2(tc.K[0], rc.t[0]);
                s_tcc[1] = make_double2(tc.t[0], tc.K[4]);
                s_tcc[2] = make_double2(rc.t[1], tc.t[1]);
            }
            for (int g0 = 0; g0 < cnt; g0 += kGroup) {
                const int gn = min(kGroup, cnt - g0);
                if (threadIdx.x < gn) {
                    const int h = s_list[g0 + threadIdx.x];
                    const double d = s_d[h];
                    const double z = (d - rc.t[2]) + tc.t[2];
                    g_h[threadIdx.x] = h;
                    g_d[threadIdx.x] = d;
                    g_z[threadIdx.x] = z;
                    g_rz[threadIdx.x] = 1.0 / z;
                    g_kz0[threadIdx.x] = tc.K[2] * z;
                    g_kz1[threadIdx.x] = tc.K[5] * z;
                    if (LFDG_SWEEP_PACK) {
                        g_pk[threadIdx.x][0] = make_double2(d, z);
                        g_pk[threadIdx.x][1] = make_double2(1.0 / z, tc.K[2] * z);
                        g_pk[threadIdx.x][2] = make_double2(tc.K[5] * z, 0.0);
                    }
                }
                double acc = threadIdx.x < gn ? s_P[s_list[g0 + threadIdx.x]] : 0.0;
                for (int c0 = 0; c0 < n; c0 += blockDim.x) {
                    const int cn = min((int)blockDim.x, n - c0);
                    __syncthreads();
                    if ((int)threadIdx.x < cn) {
                        const int p = mem[c0 + threadIdx.x];
                        double rx, ry;
                        cam_ray(rc, (double)(p % W), (double)(p / W), rx, ry);
                        const float4 ref = rimg[p];
                        for (int gi = 0; gi < gn; ++gi) {
                            float val;
                            if (kIdR && kCanonK)
                                val = LFDG_SWEEP_PACK
                                          ? sample_fast_packed(s_tcc, g_pk[gi], timg, W, H, rx, ry, ref, T)
                                          : sample_fast(rc, tc, timg, W, H, g_d[gi], g_z[gi], g_rz[gi], g_kz0[gi], g_kz1[gi],
                                                  rx, ry, ref, T);
                            else
                                val = sweep_sample<kIdR, kCanonK>(rc, tc, timg, W, H, g_d[gi], rx, ry, ref, T);
                            s_tile[gi * kTilePitch + threadIdx.x] = val;
                        }
                    }
                    __syncthreads();
                    if ((int)threadIdx.x < gn) {
                        const float* row = s_tile + threadIdx.x * kTilePitch;
                        int jj = 0;
                        for (; jj + 4 <= cn; jj += 4) {
                            const float4 q = *reinterpret_cast<const float4*>(row + jj);
                            acc += (double)q.x;
                            acc += (double)q.y;
                            acc += (double)q.z;
                            acc += (double)q.w;
                        }
                        for (; jj < cn; ++jj) acc += (double)row[jj];
                    }
                }
                if ((int)threadIdx.x < gn) s_P[g_h[threadIdx.x]] = acc;
                __syncthreads();
            }
            if (prune) {
                // keep list members whose partial cost is still <= B (ordered, in place)
                int* tmp = s_tmp;
                for (int q = threadIdx.x; q < cnt; q += blockDim.x) tmp[q] = s_list[q];
                __syncthreads();
                cnt = block_compact(cnt, s_list, red_k, [&](int q) { return s_P[tmp[q]] <= B; });
                for (int q = threadIdx.x; q < cnt; q += blockDim.x) s_list[q] = tmp[s_list[q]];
                __syncthreads();
            }
        }
        return cnt;
    };

    int best;
    if (n_targets <= 1) {
        best = block_argmin(s_P, s_d, nullptr, levels, red_c, red_d, red_k);
    } else {
        // ---- B: complete the chain of the best partial hypothesis
        const int hs = block_argmin(s_P, s_d, nullptr, levels, red_c, red_d, red_k);
        if (threadIdx.x == 0) s_list[0] = hs;
        __syncthreads();
        advance(1, 1, false, 0.0);
        const double B = s_P[hs];
        // ---- C: the others, pruned against B after every target
        int cnt = block_compact(levels, s_list, red_k, [&](int k) { return k != hs && s_P[k] <= B; });
        cnt = advance(cnt, 1, true, B);
        if (threadIdx.x == 0) s_list[cnt] = hs;
        __syncthreads();
        best = block_argmin(s_P, s_d, s_list, cnt + 1, red_c, red_d, red_k);
    }
    if (threadIdx.x == 0) {
        planes[(size_t)view * nsp + sp] = make_double4(s_d[best], 0.0, 0.0, -1.0);
        if (LFDG_SWEEP_COUNT) atomicAdd(samples, s_samples);  // work counter [5]
    }
}

// rasterize (sweep.hpp:44-63), one thread per pixel of views [v0, v0+n).
__global__ void k_rasterize(const int32_t* __restrict__ labels, const double4* __restrict__ planes,
                            const double2* __restrict__ cray, const Cam* __restrict__ cams, int W, int H, int nsp,
                            int v0, float* depth) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const int v = v0 + blockIdx.y;
    const int l = labels[(size_t)v * hw + i];
    const double4 pl = planes[(size_t)v * nsp + l];
    const double2 cr = cray[(size_t)v * nsp + l];
    const double ax = pl.x * cr.x, ay = pl.x * cr.y, az = pl.x;
    const double num = (pl.y * ax + pl.z * ay) + pl.w * az;
    const int x = (int)(i % W), y = (int)(i / W);
    double rx, ry;
    cam_ray(cams[v], (double)x, (double)y, rx, ry);
    const double denom = (pl.y * rx + pl.z * ry) + pl.w;
    depth[(size_t)v * hw + i] = fabs(denom) <= 1e-9 ? 0.f : (float)(num / denom);
}

inline unsigned ceil_div(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace

// matching_views (sweep.hpp:67-80), on the host with Eigen's operation order.
std::vector<int> matching_views(const Ctx& c, int view, int max_neighbors) {
    std::vector<int> others;
    for (int i = 0; i < c.V; ++i)
        if (i != view) others.push_back(i);
    if (max_neighbors > 0 && static_cast<int>(others.size()) > max_neighbors) {
        auto center = [&](int v, double out[3]) {
            const lfdg_camera& k = c.cams[v];
            for (int i = 0; i < 3; ++i)
                out[i] = ((-k.R[0 * 3 + i]) * k.t[0] + (-k.R[1 * 3 + i]) * k.t[1]) + (-k.R[2 * 3 + i]) * k.t[2];
        };
        double cv[3];
        center(view, cv);
        auto d2 = [&](int v) {
            double cc[3];
            center(v, cc);
            const double a = cc[0] - cv[0], b = cc[1] - cv[1], e = cc[2] - cv[2];
            return (a * a + b * b) + e * e;
        };
        std::stable_sort(others.begin(), others.end(), [&](int a, int b) { return d2(a) < d2(b); });
        others.resize(max_neighbors);
        std::sort(others.begin(), others.end());
    }
    return others;
}

void sweep_views(Ctx& c, int v0, int n, const lfdg_sweep_params& p, uint64_t seed) {
    if (p.levels < 2) throw Error(LFDG_INVALID_PARAMS, "sweep levels must be >= 2");
    if (!(p.tssd_threshold > 0)) throw Error(LFDG_INVALID_PARAMS, "tssd threshold must be > 0");
    if (!(0 < c.d_min && c.d_min < c.d_max)) throw Error(LFDG_INVARIANT, "depth range requires 0 < d_min < d_max");
    if (v0 < 0 || n < 0 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    for (int v = 0; v < c.V; ++v) c.require_grid(v);  // sweep_cost reads only the own grid, but
    // matching_views needs V and the rasterize that follows needs every grid.
    if (n == 0) return;
    const int nt = c.V - 1 > 0 && p.max_neighbors > 0 ? std::min(p.max_neighbors, c.V - 1) : c.V - 1;
    std::vector<int> tg((size_t)c.V * std::max(nt, 1), 0);
    for (int v = 0; v < c.V; ++v) {
        const std::vector<int> t = matching_views(c, v, p.max_neighbors);
        for (int i = 0; i < nt; ++i) tg[(size_t)v * nt + i] = t[i];
    }
    DevBuf<int>& d_tg = c.sweep_targets;
    d_tg.alloc(tg.size());
    LFDG_CUDA_CHECK(cudaMemcpyAsync(d_tg.p, tg.data(), tg.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    const double inv_lo = 1.0 / c.d_max;
    const double inv_hi = 1.0 / c.d_min;
    const double step = (inv_hi - inv_lo) / (p.levels - 1);
    const int threads = 256;
    // The hypotheses of a superpixel (depth, partial cost, list: 20 B each) live in shared memory
    // while they fit beside the tile — with the prune list staged in the tile (kGroup * kTilePitch
    // ints) — and otherwise in global scratch slots, one per resident CTA, the grid then launched
    // in waves of that many CTAs (the reference accepts any L >= 2).
    const size_t fixed = std::max(kSweepCap * (sizeof(double2) + sizeof(float4)), kGroup * kTilePitch * sizeof(float)) +
                         (size_t)(nt + 1) * sizeof(Cam);
    const size_t in_smem = fixed + (size_t)p.levels * (2 * sizeof(double) + sizeof(int));
    const bool scratch = p.levels > kGroup * kTilePitch || in_smem > (size_t)(227 * 1024);
    const size_t smem = scratch ? fixed : in_smem;
    if (smem > (size_t)(227 * 1024))
        throw Error(LFDG_INVALID_PARAMS, "too many matching views for the sweep's shared-memory camera table");
    const unsigned grid = (unsigned)c.nsp * (unsigned)n;
    const size_t slot_bytes = ((size_t)p.levels * (2 * sizeof(double) + 2 * sizeof(int)) + 255) & ~(size_t)255;
    auto launch = [&](auto kernel, auto kernel_scratch) {
        if (!scratch) {
            LFDG_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            kernel<<<grid, threads, smem, c.stream>>>(c.lab.p, c.W, c.H, c.nsp, v0, c.d_cams.p, d_tg.p, nt, c.moff.p,
                                                      c.mpix.p, p.levels, inv_lo, inv_hi, step, p.tssd_threshold, seed,
                                                      c.gw, n, c.planes.p, c.counters.p + 5, nullptr, 0, 0);
            LFDG_LAUNCHED(&c);
            return;
        }
        LFDG_CUDA_CHECK(cudaFuncSetAttribute(kernel_scratch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        LFDG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_scratch, threads, smem));
        const unsigned wave = std::min<unsigned>(grid, (unsigned)std::max(per_sm, 1) * (unsigned)c.sm_count);
        c.sweep_scratch.alloc(wave * slot_bytes);
        for (unsigned off = 0; off < grid; off += wave) {
            kernel_scratch<<<std::min(wave, grid - off), threads, smem, c.stream>>>(
                c.lab.p, c.W, c.H, c.nsp, v0, c.d_cams.p, d_tg.p, nt, c.moff.p, c.mpix.p, p.levels, inv_lo, inv_hi,
                step, p.tssd_threshold, seed, c.gw, n, c.planes.p, c.counters.p + 5, c.sweep_scratch.p, slot_bytes,
                (int)off);
            LFDG_LAUNCHED(&c);
        }
    };
    if (c.identity_rot && c.canonical_k)
        launch(k_sweep<true, true, false>, k_sweep<true, true, true>);
    else if (c.identity_rot)
        launch(k_sweep<true, false, false>, k_sweep<true, false, true>);
    else if (c.canonical_k)
        launch(k_sweep<false, true, false>, k_sweep<false, true, true>);
    else
        launch(k_sweep<false, false, false>, k_sweep<false, false, true>);
    for (int b = 0; b < n; ++b) c.planes_ready[v0 + b] = 1;
}

void rasterize_views(Ctx& c, int v0, int n) {
    if (v0 < 0 || n < 0 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    for (int v = v0; v < v0 + n; ++v) {
        c.require_grid(v);
        if (!c.planes_ready[v]) throw Error(LFDG_STATE, "view has no planes: sweep or set them first");
    }
    if (n == 0) return;
    if (!c.depth.p) c.depth.alloc((size_t)c.V * c.hw());
    k_rasterize<<<dim3(ceil_div(c.hw(), 256), n), 256, 0, c.stream>>>(c.labels.p, c.planes.p, c.cray.p, c.d_cams.p,
                                                                      c.W, c.H, c.nsp, v0, c.depth.p);
    LFDG_LAUNCHED(&c);
}

}  // namespace lfdg
