// Jacobi refinement on sm_100a: make_refine_context (refine.hpp:53-79) and refine_iteration
// (refine.hpp:253-323) with the full energy E = E_s * E_c (smoothness_term :84, pair_stats
// :111, consistency_term :189, energy :201, normal_candidates :213).
//
// Persistent kernel, one warp per (view, superpixel) task at a time (tasks pulled from a global
// counter in (superpixel row, view, column) order for L2 locality).  The reference's per-task
// control flow is a sequential greedy over an ordered candidate list (propagation candidates in
// grid_neighbors(Kernel) order, then the triangle normals at the current depth) that accepts a
// candidate iff its energy is strictly above the running best, skipping candidates whose bound
// E_s (1 + eta) cannot beat it.  The warp reproduces it exactly:
//   * the candidate list is built in the reference order; E_s of every candidate is computed up
//     front (8 lanes per candidate); bitwise repeats of earlier planes are marked (they cannot
//     be accepted) and the task bound m_task <= 1 + eta prunes what the reference's bound prunes
//     and more, never an acceptable candidate;
//   * E_c is evaluated lane-per-target (pair_stats, refine.hpp:111-172): each lane walks the
//     member pixels in the reference's order and keeps photo_sum / vis_sum / x_count in
//     registers, so every FP64 sum is bit-identical; the per-pixel geometry is computed once per
//     pixel and broadcast through shared memory; the target's (label, depth, 1/depth) comes from
//     one gather of the rasterised target (k_build_raster); photo weights are cached per lane;
//   * with G = 8 or 16 lanes per candidate, 32 / G consecutive surviving candidates are
//     evaluated at once (speculatively); decisions are still taken in index order with exact
//     energies, re-testing the later ones after an acceptance.
// The accepted planes and the accepted count are therefore the reference's.  kFlat selects the
// rectified / grid-rig specialisations (R = I, t.z = 0, one K).  exp/expf are the glibc ports
// (glibc_math.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "context.h"
#include "glibc_math.cuh"

namespace lfdg {
namespace {


struct RefineArgs {
    // geometry / images
    int W, H, nsp, gw, gh, V;
    int rv0;  // first refined view
    const Cam* cams;
    const int32_t* labels;  // [V][HW]
    const float4* color;    // [V][nsp]
    const double2* cray;    // [V][nsp]
    const int32_t* moff;    // [V][nsp+1]
    const double2* mray;    // [V][HW] member rays in CSR order
    const double4* planes;  // snapshot [V][nsp]
    const float* depth;     // snapshot [V][HW]
    const int4* ras;        // [V][HW] gather raster (label word, depth, 1/depth), k_build_raster
    double4* out;           // [V][nsp]
    // context tables
    const int* targets;     // [V][N]
    const double* rel;      // [V][N][12]
    const float* min_nb_sim;  // [V][nsp]
    const float* ring_w;      // [V][nsp][8]
    int N;
    double d_min, d_max;
    double sigma, two_sigma2, inv_two_sigma2, inv_two_alpha2;
    double eta;  // (double)eta
    double max_consistency;
    int use_s, use_c, use_o;
    int kernel_px, kernel_step, radius_sp, per_dir, n_slots;
    double uK00, uK02, uK11, uK12;  // the shared K of a kFlat view set
    int row_inv;                    // kFlat and every rel_trans.y == 0: target rows are view-invariant
                                    // (selects kFlat == 2)
    unsigned long long* counters;
};

// many-target mode (kFlat == 3): the 8-byte gather raster (1 / depth computed per visible sample)
// or the 16-byte one
#ifndef LFDG_MANY_RAS8
#define LFDG_MANY_RAS8 0
#endif
constexpr bool kRas8 = LFDG_MANY_RAS8;

__constant__ int kDir[8][2] = {{1, 0}, {1, -1}, {0, -1}, {-1, -1}, {-1, 0}, {-1, 1}, {0, 1}, {1, 1}};

// glibc lround (dbl-64 s_lround.c on x86-64) followed by static_cast<int>: |x| >= 2^63 and
// NaN go through (long)x = LONG_MIN, whose low 32 bits are 0.
__device__ __forceinline__ int lround_int(double x) {
    long long r;
    if (fabs(x) < 0x1p63) {
        r = llround(x);
    } else {
        r = (long long)0x8000000000000000ull;
    }
    return (int)(unsigned)(unsigned long long)r;
}

// lround(h / z) the slow way (division, then lround), out of line: fast_lround's rare fallback.
// z = NaN marks an invisible pixel of the flat-rig modes 1 / 3 (pixel_geo): -1, outside any image.
__device__ __noinline__ int lround_div(double h, double z) { return z == z ? lround_int(h / z) : -1; }

// exp of the visibility term (refine.hpp:158): glibc's main path inline when the argument is in
// its range (integer test on the high word), the full glibc path (early exits, specialcase) out of
// line otherwise — the same function as libm::exp_nonpos.
__device__ __noinline__ double exp_vis_slow(double x) { return libm::exp_nonpos(x); }
__device__ __forceinline__ double exp_vis(double x) {
    return libm::exp_nonpos_in_core(x) ? libm::exp_nonpos_core(x) : exp_vis_slow(x);
}

// vis_sum += exp(x) (refine.hpp:158, x <= 0): glibc's main path inline when x is in its range
// (integer test on the high word), exp(x) = +0 for x <= -746 (glibc rounds it to zero; vis_sum + 0
// = vis_sum for vis_sum >= +0) without a call, the rest of glibc's path out of line.
__device__ __forceinline__ void accumulate_vis(double& vis_sum, double x) {
    if (libm::exp_nonpos_in_core(x))
        vis_sum += libm::exp_nonpos_core(x);
    else if (!(x <= -746.0))
        vis_sum += exp_vis_slow(x);
}

// The linear-rig mode's copy of glibc's exp table in shared memory (LFDG_EXP_SMEM): the table
// lookup of the visibility exp is one shared load at a link-time address (C3 refine -2.5 %; not
// for 8-lane candidate slots, where it measured +0.7 % at C5).
#ifndef LFDG_EXP_SMEM
#define LFDG_EXP_SMEM 1
#endif
__shared__ __align__(16) ulonglong2 s_exptab[128];
__device__ __forceinline__ void accumulate_vis_smem(double& vis_sum, double x) {
    if (libm::exp_nonpos_in_core(x))
        vis_sum += libm::exp_nonpos_core_tab(x, s_exptab);
    else if (!(x <= -746.0))
        vis_sum += exp_vis_slow(x);
}

// depth_consistency (refine.hpp:34-37)
__device__ __forceinline__ double depth_consistency(double d1, double d2, double two_sigma2) {
    const double r = 1.0 / d1 - 1.0 / d2;
    return libm::exp_nonpos(-(r * r) / two_sigma2);
}

// ---- smoothness_term (refine.hpp:84-100), warp-parallel: lanes = (candidate, ring slot k)
// groups of 8.  Each lane evaluates one ring neighbour; every lane of a group then folds the
// group's 8 slots in ring order with width-8 shuffles, so wsum / acc are the reference's
// sequential sums.  Returns the smoothness of the lane's group candidate.
__device__ __forceinline__ double smoothness_group(const RefineArgs& a, int v, int sp, double4 p, bool active) {
    const int k = threadIdx.x & 7;
    const int gx = sp % a.gw, gy = sp / a.gw;
    bool present = false, has_c = false;
    double w = 0, c = 0;
    if (active) {
        const int nx = gx + kDir[k][0], ny = gy + kDir[k][1];
        if (nx >= 0 && ny >= 0 && nx < a.gw && ny < a.gh) {
            present = true;
            const int nb = ny * a.gw + nx;
            w = (double)a.ring_w[((size_t)v * a.nsp + sp) * 8 + k];
            const double2 cr = a.cray[(size_t)v * a.nsp + sp];
            const double ax = p.x * cr.x, ay = p.x * cr.y, az = p.x;
            const double num = (p.y * ax + p.z * ay) + p.w * az;
            const double2 nr = a.cray[(size_t)v * a.nsp + nb];
            const double denom = (p.y * nr.x + p.z * nr.y) + p.w;
            if (!(fabs(denom) <= 1e-9)) {
                const double ext = num / denom;
                if (ext > 0) {
                    has_c = true;
                    c = w * depth_consistency(a.planes[(size_t)v * a.nsp + nb].x, ext, a.two_sigma2);
                }
            }
        }
    }
    double wsum = 0, acc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const double wj = __shfl_sync(LFDG_FULL_MASK, w, j, 8);
        const double cj = __shfl_sync(LFDG_FULL_MASK, c, j, 8);
        const int pj = __shfl_sync(LFDG_FULL_MASK, (int)present, j, 8);
        const int hj = __shfl_sync(LFDG_FULL_MASK, (int)has_c, j, 8);
        if (pj) wsum += wj;
        if (hj) acc += cj;
    }
    if (wsum <= 1e-30) return 1.0;
    return acc / wsum;
}

// lround(u) for u = hx / z from q = hx * (1/z).  |q - u| <= 1.5 * 2^-52 |u| (two roundings), i.e.
// <= 2^-31 for |q| < 2^20, so when q is farther than 2^-28 from a half-integer, u rounds to the
// same integer as q; the nearest integer is read off the low word of q + 1.5*2^52
// (round-to-nearest, no F2I).  Otherwise it returns false and the caller divides exactly.
__device__ __forceinline__ bool fast_lround(double q, int& out) {
    if (!(fabs(q) < 0x1p20)) return false;
    const double t = q + 0x1.8p52;
    const double d = q - (t - 0x1.8p52);  // exact, in [-0.5, 0.5]
    if (!(fabs(d) < 0.5 - 0x1p-28)) return false;
    out = __double2loint(t);
    return true;
}

// fast_lround for the kFlat hot loop: the integer is read off q + 1.5 * 2^52 when that sum lies in
// [2^52 * 1.5, 2^52 * 1.5 + 2^32) (hi word 0x43380000: 0 <= lround(q) < 2^32), else -1 (outside any
// image: q < -0.5 or q >= 2^32); within 2^-28 of a half-integer it returns false and the caller
// divides exactly.  |q| < 2^20 whenever the result can be inside an image (W, H <= 2^20, checked
// on the host), so the error bound of fast_lround applies.
__device__ __forceinline__ bool fast_lround_img(double q, int& out) {
    const double t = q + 0x1.8p52;
    const double d = q - (t - 0x1.8p52);
    out = __double2hiint(t) == 0x43380000 ? __double2loint(t) : -1;
    return fabs(d) < 0.5 - 0x1p-28;
}

// Per-warp shared-memory slice.  Candidate planes / upper bounds live in a per-warp global
// scratch row (L1-resident); the per-task target table, the per-pixel geometry of the current
// pixel chunk, the photo-weight cache and the per-target results are shared memory.
struct TargetRow {   // one matching view of the task (refine.hpp:116-118, 46-47)
    double R[9];
    double T[3];
    double K00, K01, K02, K11, K12;
    const int4* ras;     // this target's gather raster (see k_build_raster)
};
struct TargetFlat {  // kFlat: R = I, t.z = 0 and the shared K make everything but T.x, T.y implicit
    double T0, T1;
    const int4* ras;
    const void* pad;
};
// Target-independent part of pair_stats' transfer for one member pixel (refine.hpp:131-137):
// s v, and for kFlat (every R = I, every t.z = 0, one shared K) z = s, 1/z, K02 z, K12 z and,
// for a linear rig, the rounded target row.
// 56 bytes (a 16-byte-aligned 64-byte layout for paired loads cost the many-target mode (C4) its
// 7th CTA per SM: +17 % refine time there)
struct PixGeo {
    double sv0, sv1, sv2;
    double f_inv, f_kz0, f_kz1;
    int f_py;
    int ok;
};
struct WarpSmem {
    double4* cand;  // [cap]   (global scratch)
    double* es;     // [cap]   (global scratch)
    int2* acc;      // [cap]   (global scratch) accepted (previous, new) candidate pairs of the task (recheck)
    void* tg;       // [N] TargetRow, or TargetFlat for kFlat
    PixGeo* geo;    // [32] geometry of the current pixel chunk (one entry per lane)
    double2* pc;    // [cw][ways + 1] lane-private photo-weight cache rows: (weight, raster word); the
                    // pad entry staggers the rows over the banks
    double* res;    // [2][N] V + O per target, per candidate slot
    double m_task;  // upper bound of V_t + O_t for the current task
    int cw;         // photo-cache rows: one per (candidate slot, target lane of a round)
};
// photo-cache slots per (lane, target): 4, or 2 in the 8-byte-raster mode (kFlat == 3: many
// targets, where the L1 capacity the cache would take matters more than the cache hits)
#ifndef LFDG_MANY_WAYS
#define LFDG_MANY_WAYS 2
#endif
__host__ __device__ constexpr int cache_ways(int flat_mode) { return flat_mode == 3 ? LFDG_MANY_WAYS : 4; }

// lanes per candidate slot G (8, 16 or 32; 32 / G candidates share a warp): the smallest power
// of two >= N with at least 8 lanes, except in the many-target mode (flat_mode 3) for 17..24
// targets, where 8 lanes over three target rounds keep every lane busy (one 32-lane group would
// leave a quarter or more of them idle: C4, N = 24: 100.1 -> 91.0 ms/view)
__host__ __device__ inline int lanes_per_candidate(int N, int flat_mode) {
    return N <= 8 ? 8 : N <= 16 ? 16 : flat_mode == 3 && N <= 24 ? 8 : 32;
}
// rows of the photo cache: one per (candidate slot, target rounded up to whole rounds of G);
// except in flat_mode 3 this is lane + t0 (N <= G, or G = 32)
__host__ __device__ inline int cache_width(int N, int flat_mode) {
    const int G = lanes_per_candidate(N, flat_mode);
    return 32 / G * ((N + G - 1) / G * G);
}
__host__ __device__ inline size_t target_row_bytes(bool flat) { return flat ? sizeof(TargetFlat) : sizeof(TargetRow); }
__host__ __device__ inline size_t warp_smem_bytes(int N, int flat_mode) {
    const size_t b = (size_t)(cache_ways(flat_mode) + 1) * cache_width(N, flat_mode) * sizeof(double2) +
                     (size_t)N * target_row_bytes(flat_mode != 0) +
                     32 * sizeof(PixGeo) + (size_t)(32 / lanes_per_candidate(N, flat_mode)) * N * sizeof(double);
    return (b + 127) & ~(size_t)127;
}

// The cache-miss path of the photo weight, out of line so that its registers do not weigh on the
// hot loop; the operands are re-read from memory (L1) instead of being kept live.
__device__ __noinline__ double photo_miss(const int* target, const float4* ref, const float4* color, int nsp, int label,
                                          double inv_two_alpha2) {
    const float4 rc = *ref;
    const float4 c = __ldg(&color[(size_t)(*target) * nsp + label]);
    return libm::exp_nonpos(-(double)color_dist2(rc.x, rc.y, rc.z, c.x, c.y, c.z) * inv_two_alpha2);
}

// The photo-cache row of a lane addressed by its 32-bit shared-window offset, made opaque to the
// compiler (LFDG_PC_S32 = 2) so that it stays in one register: the generic row pointer was
// rematerialised from the lane id on every cache probe (8 instructions; refine -3.6 / -1.5 /
// -3.2 % at C3 / C4 / C5).  0: plain pointer (A/B builds only).
// LFDG_SKIP_OK: the gather skips the per-pixel ok test — 1: kFlat 2 (refine -3.5 / -3.3 % at C3 /
// C5), 2: also kFlat 1 / 3 (C4 -3.0 %), 3: also the general kernels (converging rig -3.2 %).
#ifndef LFDG_SKIP_OK
#define LFDG_SKIP_OK 3
#endif
#ifndef LFDG_PC_S32
#define LFDG_PC_S32 2
#endif
__device__ __forceinline__ double2 pc_load(const double2* base, unsigned base_s, int way) {
    if (LFDG_PC_S32) {
        double2 v;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(base_s + 16u * way));
        return v;
    }
    return base[way];
}
__device__ __forceinline__ void pc_store(double2* base, unsigned base_s, int way, double2 v) {
    if (LFDG_PC_S32)
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(base_s + 16u * way), "d"(v.x), "d"(v.y) : "memory");
    else
        base[way] = v;
}

// Per-pixel geometry of member pixel i for plane p (refine.hpp:131-137).
template <int kFlat>
__device__ __forceinline__ PixGeo pixel_geo(const RefineArgs& a, const double2* mr, int i, int n, double4 p,
                                            double plane_num) {
    PixGeo q;
    q.ok = 0;
    q.sv0 = q.sv1 = q.sv2 = 0;
    q.f_inv = q.f_kz0 = q.f_kz1 = 0;
    q.f_py = -1;
    if (i < n) {
        const double2 r = mr[i];
        const double denom = (p.y * r.x + p.z * r.y) + p.w;
        if (!(fabs(denom) <= 1e-9)) {  // degenerate ray: invisible
            const double s = plane_num / denom;
            if (s > 0) {
                q.ok = 1;
                q.sv0 = s * r.x;
                q.sv1 = s * r.y;
                q.sv2 = s;
            }
        }
    }
    if (kFlat == 0 && LFDG_SKIP_OK > 2 && !q.ok) q.sv0 = q.sv1 = q.sv2 = __longlong_as_double(0x7ff8000000000000ll);
    if ((kFlat == 1 || kFlat == 3) && LFDG_SKIP_OK > 1 && !q.ok) {
        // invisible: z = 1 / z = NaN sends both lrounds of every target to lround_div, which
        // returns -1 (outside the image) for it, so the gather needs no ok test
        q.sv2 = q.f_inv = __longlong_as_double(0x7ff8000000000000ll);
    }
    if (kFlat && q.ok) {
        q.f_inv = 1.0 / q.sv2;
        q.f_kz0 = a.uK02 * q.sv2;
        q.f_kz1 = a.uK12 * q.sv2;
        if (kFlat == 2) {  // every T.y = 0 (linear rig): the target row is the same for all targets
            const double hy = a.uK11 * q.sv1 + q.f_kz1;
            if (!fast_lround(hy * q.f_inv, q.f_py)) q.f_py = lround_int(hy / q.sv2);
        }
    }
    return q;
}

// consistency_term (refine.hpp:189-199) of up to two candidate planes of task (v, sp) at once.
// Lanes are (candidate slot, target): with N <= 16 targets each half-warp evaluates its own
// candidate (G = 16 lanes, lane = target), otherwise the whole warp evaluates one (G = 32, lanes
// stride over the targets).  Each lane runs pair_stats (refine.hpp:111-172) for its target
// exactly as the reference does — the member pixels in order, photo_sum / vis_sum / x_count /
// y_nonempty accumulated sequentially in registers, the same one-entry label cache — so every
// sum is bit-identical.  The target-independent geometry of each pixel chunk is computed once
// per pixel (one lane per pixel) and broadcast through shared memory.  The label cache is backed
// by a small lane-private cache of photo weights, which are pure functions of (task colour,
// target, label) and so stay valid for the whole task.  V + O are summed in target order.
template <bool kIdR, bool kCanonK, int kFlat, int kG>
__device__ __forceinline__ double consistency_pair(const RefineArgs& a, const WarpSmem& w, int v, int sp, double4 p,
                                                   int m0, int n) {
    const int lane = threadIdx.x & 31;
    const int N = a.N;
    if (N == 0) return 1.0;
    const int G = kG ? kG : lanes_per_candidate(N, kFlat);  // lanes per candidate slot
    const int cs = lane / G;  // candidate slot
    const int tl = lane % G;  // target lane
    const size_t hw = (size_t)a.W * a.H;
    const double2 cr = a.cray[(size_t)v * a.nsp + sp];
    const double ax = p.x * cr.x, ay = p.x * cr.y, az = p.x;
    const double plane_num = (p.y * ax + p.z * ay) + p.w * az;  // plane.normal.dot(anchor)
    const double2* mr = a.mray + (size_t)v * hw + m0;
    const double occ = a.use_o ? a.eta * (1.0 - (double)a.min_nb_sim[(size_t)v * a.nsp + sp]) : 0.0;
    const PixGeo* geo = w.geo + cs * G;
    double* res = w.res + cs * N;
    for (int t0 = 0; t0 < N; t0 += G) {
        const int t = t0 + tl;
        const bool act = t < N;
        double2* const pcl =  // this lane's cache row
            w.pc + (kFlat == 3 ? cs * ((N + G - 1) / G * G) + t : lane + t0) * (cache_ways(kFlat) + 1);
        unsigned pcl_s = (unsigned)__cvta_generic_to_shared(pcl);
        if (LFDG_PC_S32 > 1) asm volatile("mov.u32 %0, %0;" : "+r"(pcl_s));  // opaque: kept, not recomputed
        double T0 = 0, T1 = 0;
        const int4* ras = nullptr;
        if (kFlat && act) {
            const TargetFlat& g = static_cast<const TargetFlat*>(w.tg)[t];
            T0 = g.T0;
            T1 = g.T1;
            ras = g.ras;
        }
        double photo_sum = 0, vis_sum = 0;
        int x_count = 0;
        bool y_nonempty = false;
        int cached_word = -1;
        double cached_w = 0;
        for (int b = 0; b < n; b += G) {
            w.geo[lane] = pixel_geo<kFlat>(a, mr, b + tl, n, p, plane_num);
            __syncwarp();
            const int cnt = min(G, n - b);
            if (act && kFlat) {
                // Software-pipelined by one pixel: the raster record of pixel jj + 1 is requested
                // before pixel jj is consumed, so the gather's latency overlaps the exp.
                auto issue = [&](const PixGeo* qq, int4& rr) -> bool {
                    // kFlat == 2: an invisible pixel has f_py = -1, so the bounds test below rejects
                    // it without the ok test (its column is computed from zeros and discarded)
                    // kFlat 1 / 3: its z is NaN, and lround_div returns -1 for it
                    if (!(LFDG_SKIP_OK > (kFlat == 2 ? 0 : 1)) && !qq->ok) return false;
                    int px, py;
                    const double hx = a.uK00 * (qq->sv0 + T0) + qq->f_kz0;
                    if (!fast_lround_img(hx * qq->f_inv, px)) px = lround_div(hx, qq->sv2);
                    if (kFlat == 2) {
                        py = qq->f_py;
                    } else {
                        const double hy = a.uK11 * (qq->sv1 + T1) + qq->f_kz1;
                        if (!fast_lround_img(hy * qq->f_inv, py)) py = lround_div(hy, qq->sv2);
                    }
                    if ((unsigned)px >= (unsigned)a.W || (unsigned)py >= (unsigned)a.H) return false;
                    // tgrid.label(px, py) and snapshot.depth[t](px, py) (refine.hpp:146-152) in one
                    // 16-byte gather: (label word, depth, 1 / (double)depth); kFlat == 3: the
                    // 8-byte raster (label word, depth), 1 / depth is computed when it is needed
                    if (kFlat == 3 && kRas8) {
                        const int2 r2 = __ldg(reinterpret_cast<const int2*>(ras) + (unsigned)(py * a.W + px));
                        rr = make_int4(r2.x, r2.y, 0, 0);
                    } else {
                        rr = __ldg(ras + (unsigned)(py * a.W + px));
                    }
                    return true;
                };
                const PixGeo* qp = geo;  // walked as a pointer: a loop-carried register, never recomputed
                int4 rn = make_int4(0, 0, 0, 0);
                bool vn = issue(qp, rn);
                for (int jj = 0; jj < cnt; ++jj) {
                    const int4 r = rn;
                    const bool valid = vn;
                    const PixGeo* qc = qp++;
                    if (jj + 1 < cnt) vn = issue(qp, rn);
                    if (!valid) continue;
                    const double zt = qc->sv2, inv_z = qc->f_inv;
                    if (r.x != cached_word) {  // refine.hpp:147-150
                        const int way = (((unsigned)r.x >> 28) + 2 * ((unsigned)r.x >> 30)) & (cache_ways(kFlat) - 1);
                        const double2 c = pc_load(pcl, pcl_s, way);
                        if (__double2loint(c.y) == r.x) {
                            cached_w = c.x;
                        } else {
                            cached_w = photo_miss(a.targets + (size_t)v * N + t, a.color + (size_t)v * a.nsp + sp,
                                                  a.color, a.nsp, r.x & 0x0FFFFFFF, a.inv_two_alpha2);
                            pc_store(pcl, pcl_s, way, make_double2(cached_w, __hiloint2double(-1, r.x)));
                        }
                        cached_word = r.x;
                    }
                    photo_sum += cached_w;
                    const float td = __int_as_float(r.y);
                    if (td <= 0) continue;  // no target depth: not in X or Y
                    if (zt <= (double)td * (1.0 + 1e-6)) {
                        const double rr = inv_z - (kFlat == 3 && kRas8 ? 1.0 / (double)td : __hiloint2double(r.w, r.z));
                        if (kFlat == 2 && kG != 8 && LFDG_EXP_SMEM)
                            accumulate_vis_smem(vis_sum, -rr * rr * a.inv_two_sigma2);
                        else
                            accumulate_vis(vis_sum, -rr * rr * a.inv_two_sigma2);
                        ++x_count;
                    } else {
                        y_nonempty = true;
                    }
                }
            } else if (act) {
                const PixGeo* qp = geo;  // walked as a pointer: a loop-carried register, never recomputed
                for (int jj = 0; jj < cnt; ++jj, ++qp) {
                    const PixGeo& q = *qp;
                    // general rigs: an invisible pixel's s v is NaN, so x2 > 0 below rejects it
                    if (!(LFDG_SKIP_OK > 2) && !q.ok) continue;
                    int px, py;
                    double zt, inv_z;
                    const TargetRow& g = static_cast<const TargetRow*>(w.tg)[t];
                    double x0, x1, x2;
                    if (kIdR) {
                        x0 = q.sv0 + g.T[0];
                        x1 = q.sv1 + g.T[1];
                        x2 = q.sv2 + g.T[2];
                    } else {
                        x0 = ((g.R[0] * q.sv0 + g.R[1] * q.sv1) + g.R[2] * q.sv2) + g.T[0];
                        x1 = ((g.R[3] * q.sv0 + g.R[4] * q.sv1) + g.R[5] * q.sv2) + g.T[1];
                        x2 = ((g.R[6] * q.sv0 + g.R[7] * q.sv1) + g.R[8] * q.sv2) + g.T[2];
                    }
                    if (!(x2 > 0)) continue;  // behind the target camera
                    const double hx = kCanonK ? g.K00 * x0 + g.K02 * x2 : (g.K00 * x0 + g.K01 * x1) + g.K02 * x2;
                    const double hy = g.K11 * x1 + g.K12 * x2;
                    inv_z = 1.0 / x2;
                    if (!fast_lround(hx * inv_z, px)) px = lround_div(hx, x2);
                    if (!fast_lround(hy * inv_z, py)) py = lround_div(hy, x2);
                    zt = x2;
                    if ((unsigned)px >= (unsigned)a.W || (unsigned)py >= (unsigned)a.H) continue;
                    const int4 r = __ldg(g.ras + (unsigned)(py * a.W + px));
                    if (r.x != cached_word) {  // refine.hpp:147-150
                        const int way = (((unsigned)r.x >> 28) + 2 * ((unsigned)r.x >> 30)) & (cache_ways(kFlat) - 1);
                        const double2 c = pc_load(pcl, pcl_s, way);
                        if (__double2loint(c.y) == r.x) {
                            cached_w = c.x;
                        } else {
                            cached_w = photo_miss(a.targets + (size_t)v * N + t, a.color + (size_t)v * a.nsp + sp,
                                                  a.color, a.nsp, r.x & 0x0FFFFFFF, a.inv_two_alpha2);
                            pc_store(pcl, pcl_s, way, make_double2(cached_w, __hiloint2double(-1, r.x)));
                        }
                        cached_word = r.x;
                    }
                    photo_sum += cached_w;
                    const float td = __int_as_float(r.y);
                    if (td <= 0) continue;  // no target depth: not in X or Y
                    if (zt <= (double)td * (1.0 + 1e-6)) {
                        const double rr = inv_z - __hiloint2double(r.w, r.z);
                        accumulate_vis(vis_sum, -rr * rr * a.inv_two_sigma2);
                        ++x_count;
                    } else {
                        y_nonempty = true;
                    }
                }
            }
            __syncwarp();
        }
        if (act) {
            const double photo = photo_sum / (double)n;
            const double vis = x_count > 0 ? photo * (vis_sum / x_count) : 0.0;
            res[t] = vis + (y_nonempty ? occ : 0.0);
        }
    }
    __syncwarp();
    double acc = 0;
    for (int t = 0; t < N; ++t) acc += res[t];
    __syncwarp();
    return acc / (double)N;
}

// The reference's sequential greedy over cand[base, base + n) (refine.hpp:279-303) with the
// running prune E_s (1 + eta) <= e_cur.  A warp evaluates up to 32 / G consecutive surviving
// candidates at once (one per lane group, G = lanes_per_candidate): the later ones
// speculatively, against the running best before the earlier ones are decided.  Decisions are
// still taken in index order with exact energies — after an acceptance the later candidates are
// re-tested against the new best and dropped if the prune now rejects them (they can then not be
// accepted either) — so the accepted planes and the count are the reference's.
// init: cand[0] is the current plane and its energy initialises e_cur (refine.hpp:277).
// current: index in cand of the running plane.
template <bool kIdR, bool kCanonK, int kFlat, bool kRecheck, int kG>
__device__ __forceinline__ void greedy(const RefineArgs& a, const WarpSmem& w, int base, int n, int v, int sp, int m0,
                                       int n_members, bool init, double& e_cur, int& current, unsigned& accepted,
                                       unsigned long long& pix_evals, unsigned& cand_evals,
                                       unsigned long long& idle_evals) {
    // (accepted also indexes w.acc: the recheck list of this task's acceptances)
    const int lane = threadIdx.x & 31;
    const bool prune = a.use_s && a.use_c;
    const int G = kG ? kG : lanes_per_candidate(a.N, kFlat);
    const int slots = init ? 1 : 32 / G;
    int next = base;
    n += base;
    // The reference prunes with E_s (1 + eta) <= e_cur (refine.hpp:297).  Here the task's own bound
    // m_task = 1 + eta (1 - min_nb_sim) >= every V_t + O_t (photo, visibility ratio <= 1, O_t =
    // eta (1 - min_nb_sim) or 0), padded by 2^-30 against rounding, also prunes: a candidate with
    // E_s m_task <= e_cur has E <= e_cur and is never accepted, so the winner and the accepted
    // count are the reference's; only non-accepted evaluations are skipped.  es = -inf marks a
    // repeat of an earlier plane of this task (mark_repeats).
    auto passes = [&](int idx) {
        return w.es[idx] != -INFINITY && (init || !prune || w.es[idx] * w.m_task > e_cur);
    };
    while (next < n) {
        // the next `slots` surviving candidates in index order (lane group k evaluates the k-th),
        // gathered over as many 32-candidate windows as it takes
        int cnt = 0, first = -1, mine = -1;
        while (cnt < slots && next < n) {
            const int idx = next + lane;
            unsigned m = __ballot_sync(LFDG_FULL_MASK, idx < n && passes(idx));
            int last = -1;
            while (m && cnt < slots) {
                const int ck = next + __ffs(m) - 1;
                m &= m - 1;
                if (lane / G == cnt) mine = ck;
                if (cnt == 0) first = ck;
                last = ck;
                ++cnt;
            }
            next = cnt == slots && last >= 0 ? last + 1 : next + 32;
        }
        if (cnt == 0) continue;
        if (mine < 0) mine = first;  // idle groups repeat the first candidate
        idle_evals += (unsigned long long)(slots - cnt) * a.N * n_members;
        double ec = 0;
        if (a.use_c) {
            ec = consistency_pair<kIdR, kCanonK, kFlat, kG>(a, w, v, sp, w.cand[mine], m0, n_members);
            pix_evals += (unsigned long long)a.N * n_members * cnt;
        }
        cand_evals += cnt;
        for (int k = 0; k < cnt; ++k) {
            const int c = __shfl_sync(LFDG_FULL_MASK, mine, k * G);
            const double eck = __shfl_sync(LFDG_FULL_MASK, ec, k * G);
            double e;
            if (a.use_c)
                e = prune ? w.es[c] * eck : (a.use_s ? 1.0 * w.es[c] : 1.0) * eck;
            else
                e = a.use_s ? 1.0 * w.es[c] : 1.0;
            if (init) {
                e_cur = e;
            } else if ((k == 0 || passes(c)) && e > e_cur) {
                if (kRecheck && lane == 0) w.acc[accepted] = make_int2(current, c);
                e_cur = e;
                current = c;
                accepted++;
            }
        }
    }
    __syncwarp();
}

// A candidate bit-identical to a plane met earlier in this task (the initial plane cand[0], or
// any earlier candidate, evaluated or pruned) has that plane's energy, which is <= the running
// best at that point and hence <= e_cur now: it can never be accepted (this subsumes the
// reference's skip of the current plane, refine.hpp:292).  Marks cand[lo, hi) repeats with
// es = -inf; the others get es = 0 when there is no smoothness term.
__device__ void mark_repeats(const RefineArgs& a, const WarpSmem& w, int lo, int hi) {
    const int lane = threadIdx.x & 31;
    for (int c = lo + lane; c < hi; c += 32) {
        const double4 p = w.cand[c];
        bool rep = false;
        for (int c2 = 0; c2 < c && !rep; ++c2) {
            const double4 q = w.cand[c2];
            rep = __double_as_longlong(p.x) == __double_as_longlong(q.x) &&
                  __double_as_longlong(p.y) == __double_as_longlong(q.y) &&
                  __double_as_longlong(p.z) == __double_as_longlong(q.z) &&
                  __double_as_longlong(p.w) == __double_as_longlong(q.w);
        }
        if (rep)
            w.es[c] = -INFINITY;
        else if (!a.use_s)
            w.es[c] = 0.0;
    }
    __syncwarp();
}

// es of cand[base, base + n): 4 candidates per warp step (8 ring lanes each).
__device__ void smoothness_all(const RefineArgs& a, const WarpSmem& w, int base, int n, int v, int sp) {
    const int lane = threadIdx.x & 31;
    n += base;
    for (int b = base; b < n; b += 4) {
        const int ci = b + (lane >> 3);
        const bool active = ci < n;
        const double4 p = active ? w.cand[ci] : make_double4(1, 0, 0, -1);
        const double es = smoothness_group(a, v, sp, p, active);
        if (active && (lane & 7) == 0) w.es[ci] = es;
    }
    __syncwarp();
}

// RefineStats' independent re-check (refine.hpp:281-286): for every acceptance of the task,
// energy(candidate) and energy(previous plane) are evaluated again from scratch against the
// snapshot — smoothness_term and consistency_term recomputed, multiplied in energy()'s order
// (refine.hpp:201-207) — and an acceptance whose candidate does not strictly beat its
// predecessor counts as a violation.  Only in stats mode (the reference pays the same price).
template <bool kIdR, bool kCanonK, int kFlat, int kG>
__device__ __forceinline__ unsigned recheck_acceptances(const RefineArgs& a, const WarpSmem& w, int v, int sp, int m0, int n_members,
                                        unsigned n_acc) {
    const int lane = threadIdx.x & 31;
    const int G = kG ? kG : lanes_per_candidate(a.N, kFlat);
    const int slots = 32 / G;
    unsigned violations = 0;
    for (unsigned k = 0; k < n_acc; ++k) {
        const int2 pr = w.acc[k];  // (previous, candidate)
        double e[2];
        for (int j = 0; j < 2; ++j) {
            const int idx = j == 0 ? pr.x : pr.y;
            double es = 1.0;
            if (a.use_s) {
                const double4 p = w.cand[idx];
                es = smoothness_group(a, v, sp, p, true);  // every 8-lane group computes the same value
            }
            e[j] = es;
        }
        double ec[2] = {1.0, 1.0};
        if (a.use_c) {
            if (slots >= 2) {
                const int mine = lane / G == 0 ? pr.x : pr.y;
                const double r = consistency_pair<kIdR, kCanonK, kFlat, kG>(a, w, v, sp, w.cand[mine], m0, n_members);
                ec[0] = __shfl_sync(LFDG_FULL_MASK, r, 0);
                ec[1] = __shfl_sync(LFDG_FULL_MASK, r, G);
            } else {
                ec[0] = consistency_pair<kIdR, kCanonK, kFlat, kG>(a, w, v, sp, w.cand[pr.x], m0, n_members);
                ec[1] = consistency_pair<kIdR, kCanonK, kFlat, kG>(a, w, v, sp, w.cand[pr.y], m0, n_members);
            }
        }
        double en[2];
        for (int j = 0; j < 2; ++j) {  // energy(): e = 1; e *= E_s; e *= E_c
            double x = 1.0;
            if (a.use_s) x *= e[j];
            if (a.use_c) x *= ec[j];
            en[j] = x;
        }
        if (!(en[1] > en[0])) ++violations;
    }
    return violations;
}

// Persistent kernel: each warp pulls (view, superpixel) tasks from a global counter and runs
// refine_iteration's task body (refine.hpp:269-320) for it.
// Resident CTAs per SM (register budget): 8 (64 registers), or 7 in the many-target mode,
// whose latency-bound gathers gain more from the registers and the L1 than from an 8th CTA
// (C4: 111 -> 100 ms/view; C3 prefers 8: 104.7 vs 106.8 ms per refine launch).
#ifndef LFDG_REFINE_MINB
#define LFDG_REFINE_MINB 8
#endif
#ifndef LFDG_MANY_MINB
#define LFDG_MANY_MINB 7
#endif
#ifndef LFDG_REFINE_MINB_GENERAL
#define LFDG_REFINE_MINB_GENERAL 8
#endif
__host__ __device__ constexpr int refine_min_blocks(int flat_mode) {
    return flat_mode == 3 ? LFDG_MANY_MINB : flat_mode == 0 ? LFDG_REFINE_MINB_GENERAL : LFDG_REFINE_MINB;
}
template <bool kIdR, bool kCanonK, int kFlat, bool kRecheck, int kG>
__global__ void __launch_bounds__(128, refine_min_blocks(kFlat))
    k_refine(RefineArgs a, int n_tasks, int* task_counter, int cap, double4* g_cand, double* g_es, int2* g_acc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if constexpr (kFlat == 2 && kG != 8 && LFDG_EXP_SMEM) {
        for (int i = threadIdx.x; i < 128; i += blockDim.x)
            s_exptab[i] = reinterpret_cast<const ulonglong2*>(libm::kExpTabDev)[i];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gwarp = blockIdx.x * (blockDim.x >> 5) + warp;
    unsigned char* base = smem_raw + warp * warp_smem_bytes(a.N, kFlat);
    WarpSmem w;
    w.cw = cache_width(a.N, kFlat);
    w.pc = reinterpret_cast<double2*>(base);
    w.tg = base + (size_t)(cache_ways(kFlat) + 1) * w.cw * sizeof(double2);
    w.geo = reinterpret_cast<PixGeo*>(static_cast<unsigned char*>(w.tg) + (size_t)a.N * target_row_bytes(kFlat));
    w.res = reinterpret_cast<double*>(w.geo + 32);
    w.cand = g_cand + (size_t)gwarp * cap;
    w.es = g_es + (size_t)gwarp * cap;
    w.acc = g_acc + (size_t)gwarp * cap;

    unsigned long long pix_evals = 0;
    unsigned cand_evals = 0;
    unsigned long long accepted_total = 0, violations_total = 0, idle_evals = 0;
    while (true) {
        int task = 0;
        if (lane == 0) task = atomicAdd(task_counter, 1);
        task = __shfl_sync(LFDG_FULL_MASK, task, 0);
        if (task >= n_tasks) break;

        // Task order (superpixel row, view, superpixel column): warps running concurrently work on
        // the same band of image rows in every view, so the target gathers of all in-flight
        // tasks share one L2-resident band instead of streaming whole views (L2 locality).
        const int rn = n_tasks / a.nsp;
        const int row = task / (rn * a.gw);
        const int rem = task - row * rn * a.gw;
        const int v = a.rv0 + rem / a.gw;
        const int sp = row * a.gw + rem % a.gw;
        const size_t vs = (size_t)v * a.nsp;
        const double4 cur0 = a.planes[vs + sp];
        const int m0 = a.moff[(size_t)v * (a.nsp + 1) + sp];
        const int n_members = a.moff[(size_t)v * (a.nsp + 1) + sp + 1] - m0;
        int current = 0;  // index in w.cand of the running plane (cand[0] = cur0)
        double e_cur = 0;
        unsigned accepted = 0;
        w.m_task = (a.use_o ? 1.0 + a.eta * (1.0 - (double)a.min_nb_sim[vs + sp]) : 1.0) * (1.0 + 0x1p-30);
        for (int ti = lane; ti < a.N; ti += 32) {  // the task's matching views (refine.hpp:116-118)
            const int t = a.targets[(size_t)v * a.N + ti];
            const double* rel = a.rel + ((size_t)v * a.N + ti) * 12;
            if (kFlat) {
                TargetFlat& g = static_cast<TargetFlat*>(w.tg)[ti];
                g.T0 = rel[9];
                g.T1 = rel[10];
                g.ras = kFlat == 3 && kRas8 ? reinterpret_cast<const int4*>(reinterpret_cast<const int2*>(a.ras) +
                                                                   (size_t)t * a.W * a.H)
                                   : a.ras + (size_t)t * a.W * a.H;
            } else {
                TargetRow& g = static_cast<TargetRow*>(w.tg)[ti];
                for (int k = 0; k < 9; ++k) g.R[k] = rel[k];
                for (int k = 0; k < 3; ++k) g.T[k] = rel[9 + k];
                const Cam& tc = a.cams[t];
                g.K00 = tc.K[0];
                g.K01 = tc.K[1];
                g.K02 = tc.K[2];
                g.K11 = tc.K[4];
                g.K12 = tc.K[5];
                g.ras = a.ras + (size_t)t * a.W * a.H;
            }
        }
        for (int k = lane; k < (cache_ways(kFlat) + 1) * w.cw; k += 32)  // new reference colour: empty photo cache
            w.pc[k] = make_double2(0.0, __hiloint2double(-1, -1));
        __syncwarp();

        // ---- e_cur = energy(current) (refine.hpp:277)
        if (lane == 0) w.cand[0] = cur0;
        __syncwarp();
        if (a.use_s) smoothness_all(a, w, 0, 1, v, sp);
        mark_repeats(a, w, 0, 1);
        greedy<kIdR, kCanonK, kFlat, kRecheck, kG>(a, w, 0, 1, v, sp, m0, n_members, true, e_cur, current, accepted, pix_evals,
                                     cand_evals, idle_evals);

        // ---- phase A: grid_neighbors(Kernel) order (superpixel.hpp:318-343), re-anchored
        const int gx = sp % a.gw, gy = sp / a.gw;
        const double2 crs = a.cray[vs + sp];
        int n_cand = 0;
        for (int s0 = 0; s0 < a.n_slots; s0 += 32) {
            const int slot = s0 + lane;
            bool ok = false;
            double4 cand = make_double4(0, 0, 0, 0);
            if (slot < a.n_slots) {
                int dx, dy;
                if (slot < 8) {
                    dx = kDir[slot][0];
                    dy = kDir[slot][1];
                } else {
                    const int k = (slot - 8) / a.per_dir;
                    const int r = a.kernel_step * ((slot - 8) % a.per_dir + 1);
                    dx = kDir[k][0] * r;
                    dy = kDir[k][1] * r;
                    if (abs(dx) <= 1 && abs(dy) <= 1) dx = 1 << 20;  // already in the ring
                }
                const int nx = gx + dx, ny = gy + dy;
                if (nx >= 0 && ny >= 0 && nx < a.gw && ny < a.gh) {
                    const int nb = ny * a.gw + nx;
                    const double4 np = a.planes[vs + nb];
                    const double2 nr = a.cray[vs + nb];
                    // plane_depth_at(cam, nb_plane, nb_centroid, centroid) (geometry.hpp:85-92)
                    const double ax = np.x * nr.x, ay = np.x * nr.y, az = np.x;
                    const double denom = (np.y * crs.x + np.z * crs.y) + np.w;
                    if (!(fabs(denom) <= 1e-9)) {
                        const double d = ((np.y * ax + np.z * ay) + np.w * az) / denom;
                        if (d > 0 && !(d < a.d_min || d > a.d_max)) {
                            ok = true;
                            cand = make_double4(d, np.y, np.z, np.w);
                        }
                    }
                }
            }
            const unsigned m = __ballot_sync(LFDG_FULL_MASK, ok);
            if (ok) w.cand[1 + n_cand + __popc(m & ((1u << lane) - 1u))] = cand;
            n_cand += __popc(m);
        }
        __syncwarp();
        if (a.use_s) smoothness_all(a, w, 1, n_cand, v, sp);
        mark_repeats(a, w, 1, 1 + n_cand);
        greedy<kIdR, kCanonK, kFlat, kRecheck, kG>(a, w, 1, n_cand, v, sp, m0, n_members, false, e_cur, current, accepted, pix_evals,
                                     cand_evals, idle_evals);

        // ---- phase B: normal_candidates (refine.hpp:213-242) at the phase-A depth
        {
            bool okn = false;
            double4 nc = make_double4(0, 0, 0, 0);
            const double cur_depth = w.cand[current].x;
            if (lane < 8) {
                const int k = lane;
                const int ax_ = gx + kDir[k][0], ay_ = gy + kDir[k][1];
                const int bx_ = gx + kDir[(k + 1) & 7][0], by_ = gy + kDir[(k + 1) & 7][1];
                const bool ina = ax_ >= 0 && ay_ >= 0 && ax_ < a.gw && ay_ < a.gh;
                const bool inb = bx_ >= 0 && by_ >= 0 && bx_ < a.gw && by_ < a.gh;
                if (ina && inb) {
                    const int ia = ay_ * a.gw + ax_, ib = by_ * a.gw + bx_;
                    const double dr = cur0.x;  // snapshot depth of this superpixel
                    const double rx = dr * crs.x, ry = dr * crs.y, rz = dr;
                    const double da = a.planes[vs + ia].x, db = a.planes[vs + ib].x;
                    const double2 ra = a.cray[vs + ia], rb = a.cray[vs + ib];
                    const double A0 = da * ra.x - rx, A1 = da * ra.y - ry, A2 = da - rz;
                    const double B0 = db * rb.x - rx, B1 = db * rb.y - ry, B2 = db - rz;
                    double n0 = A1 * B2 - A2 * B1, n1 = A2 * B0 - A0 * B2, n2 = A0 * B1 - A1 * B0;
                    const double len = sqrt((n0 * n0 + n1 * n1) + n2 * n2);
                    if (!(len <= 1e-12)) {
                        n0 = n0 / len;
                        n1 = n1 / len;
                        n2 = n2 / len;
                        if ((n0 * crs.x + n1 * crs.y) + n2 > 0) {
                            n0 = -n0;
                            n1 = -n1;
                            n2 = -n2;
                        }
                        if (!((n0 * crs.x + n1 * crs.y) + n2 >= 0) && !(cur_depth < a.d_min || cur_depth > a.d_max)) {
                            okn = true;
                            nc = make_double4(cur_depth, n0, n1, n2);
                        }
                    }
                }
            }
            const unsigned m = __ballot_sync(LFDG_FULL_MASK, okn);
            if (okn) w.cand[1 + n_cand + __popc(m & ((1u << lane) - 1u))] = nc;
            __syncwarp();
            const int nn = __popc(m);
            if (a.use_s) smoothness_all(a, w, 1 + n_cand, nn, v, sp);
            mark_repeats(a, w, 1 + n_cand, 1 + n_cand + nn);
            greedy<kIdR, kCanonK, kFlat, kRecheck, kG>(a, w, 1 + n_cand, nn, v, sp, m0, n_members, false, e_cur, current, accepted,
                                         pix_evals, cand_evals, idle_evals);
        }
        if (lane == 0) a.out[vs + sp] = w.cand[current];
        accepted_total += accepted;
        if (kRecheck && accepted) {
            __syncwarp();
            violations_total += recheck_acceptances<kIdR, kCanonK, kFlat, kG>(a, w, v, sp, m0, n_members, accepted);
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (accepted_total) atomicAdd(&a.counters[0], accepted_total);
        if (violations_total) atomicAdd(&a.counters[1], violations_total);
        atomicAdd(&a.counters[2], pix_evals);
        atomicAdd(&a.counters[3], (unsigned long long)cand_evals);
        atomicAdd(&a.counters[4], idle_evals);
    }
}

// min_neighbor_similarity (superpixel.hpp:352-357) and the ring colour weights of
// smoothness_term (refine.hpp:92), one thread per superpixel.
__global__ void k_color_tables(const float4* __restrict__ color, int nsp, int gw, int gh, float alpha,
                               float* min_nb_sim, float* ring_w) {
    const int sp = blockIdx.x * blockDim.x + threadIdx.x;
    if (sp >= nsp) return;
    const int v = blockIdx.y;
    const float4 c = color[(size_t)v * nsp + sp];
    const int gx = sp % gw, gy = sp / gw;
    const float denom = 2.f * alpha * alpha;
    float m = 1.f;
    for (int k = 0; k < 8; ++k) {
        const int nx = gx + kDir[k][0], ny = gy + kDir[k][1];
        float w = -1.f;
        if (nx >= 0 && ny >= 0 && nx < gw && ny < gh) {
            const float4 o = color[(size_t)v * nsp + ny * gw + nx];
            w = libm::expf(-color_dist2(c.x, c.y, c.z, o.x, o.y, o.z) / denom);
            m = w < m ? w : m;  // std::min(m, w)
        }
        ring_w[((size_t)v * nsp + sp) * 8 + k] = w;
    }
    min_nb_sim[(size_t)v * nsp + sp] = m;
}

// Refine gather raster for every view, rebuilt from the snapshot each iteration: the target-side
// operands of pair_stats (refine.hpp:146-155) in one 16-byte record per pixel —
//   .x  label | ((gx & 3) | (gy & 1) << 2) << 28   (photo-cache key and slot of the label)
//   .y  snapshot depth (float bits)
//   .zw 1.0 / (double)depth, the operand of depth_consistency's 1/td (refine.hpp:158)
__global__ void k_build_raster(const int32_t* __restrict__ labels, const float* __restrict__ depth, int W, int H,
                               int gw, int4* ras) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const int v = blockIdx.y;
    const int lab = labels[(size_t)v * hw + i];
    const float td = depth[(size_t)v * hw + i];
    const int gx = lab % gw, gy = lab / gw;
    const int word = lab | (((gx & 3) | ((gy & 1) << 2)) << 28);
    const double inv = 1.0 / (double)td;
    ras[(size_t)v * hw + i] = make_int4(word, __float_as_int(td), __double2loint(inv), __double2hiint(inv));
}

// Member rays in CSR order: mray[v][k] = ray(pixel mpix[v][k]) (geometry.hpp:45).
__global__ void k_member_rays(const int32_t* __restrict__ mpix, const Cam* cams, int W, int H, double2* mray) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const int v = blockIdx.y;
    const int p = mpix[(size_t)v * hw + i];
    double rx, ry;
    cam_ray(cams[v], (double)(p % W), (double)(p / W), rx, ry);
    mray[(size_t)v * hw + i] = make_double2(rx, ry);
}

// The 8-byte raster of kFlat == 3 (many matching views: half the gather footprint in L2):
// (label word, depth); 1 / depth is computed at the sample.
__global__ void k_build_raster8(const int32_t* __restrict__ labels, const float* __restrict__ depth, int W, int H,
                                int gw, int2* ras) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const int v = blockIdx.y;
    const int lab = labels[(size_t)v * hw + i];
    const int gx = lab % gw, gy = lab / gw;
    ras[(size_t)v * hw + i] = make_int2(lab | (((gx & 3) | ((gy & 1) << 2)) << 28),
                                        __float_as_int(depth[(size_t)v * hw + i]));
}

inline unsigned ceil_div(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace

void make_refine_tables(Ctx& c, const lfdg_energy_params& p, int sweep_levels) {
    if (p.sigma < 0 || !(p.alpha > 0) || p.eta < 0 || p.eta > 1) throw Error(LFDG_INVALID_PARAMS, "bad energy params");
    if (p.steps_init <= 0 || p.size_init < 0 || p.iterations < 0) throw Error(LFDG_INVALID_PARAMS, "bad kernel params");
    c.require_views();
    for (int v = 0; v < c.V; ++v) c.require_grid(v);
    RefineTables& t = c.refine;
    t.params = p;
    if (t.params.sigma == 0) {
        const double step = (1.0 / c.d_min - 1.0 / c.d_max) / (sweep_levels - 1);  // sweep.hpp:38-40
        t.params.sigma = 1.5 * step;
    }
    if (t.params.size_init == 0) t.params.size_init = std::min(c.W, c.H);
    const int nt = p.max_neighbors > 0 ? std::min(p.max_neighbors, c.V - 1) : c.V - 1;
    t.n_targets = nt;
    t.targets_host.assign((size_t)c.V * std::max(nt, 1), 0);
    std::vector<double> rel((size_t)c.V * std::max(nt, 1) * 12, 0.0);
    for (int v = 0; v < c.V; ++v) {
        const std::vector<int> tv = matching_views(c, v, p.max_neighbors);
        const lfdg_camera& cv = c.cams[v];
        for (int i = 0; i < nt; ++i) {
            const int tt = tv[i];
            t.targets_host[(size_t)v * nt + i] = tt;
            const lfdg_camera& ct = c.cams[tt];
            double* r = &rel[((size_t)v * nt + i) * 12];
            // rel_rot = R_t * R_v^T (refine.hpp:74): (i,j) = (Rt_i0 Rv_j0 + Rt_i1 Rv_j1) + Rt_i2 Rv_j2
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    r[a * 3 + b] = (ct.R[a * 3 + 0] * cv.R[b * 3 + 0] + ct.R[a * 3 + 1] * cv.R[b * 3 + 1]) +
                                   ct.R[a * 3 + 2] * cv.R[b * 3 + 2];
            // rel_trans = t_t - rel_rot * t_v (refine.hpp:75)
            for (int a = 0; a < 3; ++a)
                r[9 + a] = ct.t[a] - ((r[a * 3 + 0] * cv.t[0] + r[a * 3 + 1] * cv.t[1]) + r[a * 3 + 2] * cv.t[2]);
        }
    }
    cudaStream_t st = c.stream;
    t.targets.alloc(t.targets_host.size());
    LFDG_CUDA_CHECK(cudaMemcpyAsync(t.targets.p, t.targets_host.data(), t.targets_host.size() * sizeof(int),
                                    cudaMemcpyHostToDevice, st));
    t.rel.alloc(rel.size());
    LFDG_CUDA_CHECK(cudaMemcpyAsync(t.rel.p, rel.data(), rel.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    t.min_nb_sim.alloc((size_t)c.V * c.nsp);
    t.ring_w.alloc((size_t)c.V * c.nsp * 8);
    k_color_tables<<<dim3(ceil_div(c.nsp, 128), c.V), 128, 0, st>>>(c.color.p, c.nsp, c.gw, c.gh, p.alpha,
                                                                   t.min_nb_sim.p, t.ring_w.p);
    LFDG_LAUNCHED(&c);
    RefineScratch& rd = c.refine_s;
    rd.mray.alloc((size_t)c.V * c.hw());
    k_member_rays<<<dim3(ceil_div(c.hw(), 256), c.V), 256, 0, st>>>(c.mpix.p, c.d_cams.p, c.W, c.H, rd.mray.p);
    LFDG_LAUNCHED(&c);
    if ((size_t)c.nsp >= (1u << 28)) throw Error(LFDG_INVALID_PARAMS, "too many superpixels per view");
    c.ras.alloc((size_t)c.V * c.hw());
    t.ready = true;
}

void refine_iteration(Ctx& c, int l, bool recheck) {
    RefineTables& t = c.refine;
    const lfdg_energy_params& p = t.params;
    for (int v = 0; v < c.V; ++v)
        if (!c.planes_ready[v]) throw Error(LFDG_STATE, "every view needs planes before refinement");
    const int rv0 = c.refine_v0;
    const int rn = c.refine_n < 0 ? c.V : c.refine_n;
    RefineArgs a{};
    a.W = c.W;
    a.H = c.H;
    a.nsp = c.nsp;
    a.gw = c.gw;
    a.gh = c.gh;
    a.V = c.V;
    a.rv0 = rv0;
    a.cams = c.d_cams.p;
    a.labels = c.labels.p;
    a.color = c.color.p;
    a.cray = c.cray.p;
    a.moff = c.moff.p;
    a.mray = c.refine_s.mray.p;
    a.planes = c.planes.p;
    a.depth = c.depth.p;
    a.ras = c.ras.p;
    a.out = c.planes_next.p;
    a.targets = t.targets.p;
    a.rel = t.rel.p;
    a.min_nb_sim = t.min_nb_sim.p;
    a.ring_w = t.ring_w.p;
    a.N = t.n_targets;
    a.d_min = c.d_min;
    a.d_max = c.d_max;
    a.sigma = p.sigma;
    a.two_sigma2 = 2.0 * p.sigma * p.sigma;
    a.inv_two_sigma2 = 1.0 / (2.0 * p.sigma * p.sigma);
    a.inv_two_alpha2 = 1.0 / (2.0 * static_cast<double>(p.alpha) * p.alpha);
    a.eta = static_cast<double>(p.eta);
    a.use_s = p.use_smoothness;
    a.use_c = p.use_consistency;
    a.use_o = p.use_occlusion;
    a.max_consistency = p.use_occlusion ? 1.0 + p.eta : 1.0;
    // refine.hpp:256-257
    a.kernel_px = static_cast<int>(p.size_init / static_cast<double>(l));
    a.kernel_step = std::max(1, static_cast<int>(std::lround(p.steps_init / static_cast<double>(l))));
    a.radius_sp = a.kernel_px / std::max(1, c.S);  // superpixel.hpp:330
    a.per_dir = a.radius_sp >= a.kernel_step ? a.radius_sp / a.kernel_step : 0;
    a.n_slots = 8 + 8 * a.per_dir;
    a.counters = c.counters.p;
    const int cap = 1 + a.n_slots + 8;  // cand[0] = the task's plane, then phase A, then phase B
    bool flat = c.identity_rot && c.canonical_k;
    for (const lfdg_camera& k : c.cams)
        flat = flat && k.t[2] == 0.0 && k.K[0] == c.cams[0].K[0] && k.K[2] == c.cams[0].K[2] &&
               k.K[4] == c.cams[0].K[4] && k.K[5] == c.cams[0].K[5];
    // the flat-rig kernels' fast lround needs image sides <= 2^20; wider images take the general
    // kernels (exact for any rig)
    if (c.W > (1 << 20) || c.H > (1 << 20)) flat = false;
    if (flat) {
        a.row_inv = 1;
        for (int vv = 0; vv < c.V; ++vv)
            for (int i = 0; i < t.n_targets; ++i) {
                const lfdg_camera& cv = c.cams[vv];
                const lfdg_camera& ct = c.cams[t.targets_host[(size_t)vv * t.n_targets + i]];
                // rel_trans.y = t_t.y - (R_rel t_v).y with R_rel = I (kFlat)
                if (ct.t[1] - ((0.0 * cv.t[0] + 1.0 * cv.t[1]) + 0.0 * cv.t[2]) != 0.0) a.row_inv = 0;
            }
    }
    // kFlat mode: 2 linear rig (row-invariant targets), 3 many targets with the 8-byte raster,
    // 1 other flat rigs, 0 general
    const int flat_mode = !flat ? 0 : a.row_inv ? 2 : a.N > 16 ? 3 : 1;
    // four warps per CTA; fewer when the per-warp tables (which grow with the number of matching
    // views) would not fit the 227 KB of shared memory of a CTA — one warp holds ~1000 targets
    const size_t wbytes = warp_smem_bytes(a.N, flat_mode);
    const size_t budget = 227 * 1024 - sizeof(s_exptab);  // less the static exp table
    const int warps = 4 * wbytes <= budget ? 4 : 2 * wbytes <= budget ? 2 : 1;
    const size_t smem = warps * wbytes;
    if (smem > budget) throw Error(LFDG_INVALID_PARAMS, "too many matching views for the refinement kernel");
    if (rn > 0) {
        // the refine gather raster from the current snapshot (labels, depth)
        // many matching views on a non-linear flat rig: the 8-byte raster (kFlat == 3) halves the
        // gather working set (C4: 24 targets x a wide vertical disparity band)
        const bool ras8 = flat_mode == 3 && kRas8;
        if (ras8)
            k_build_raster8<<<dim3(ceil_div(c.hw(), 256), c.V), 256, 0, c.stream>>>(
                c.labels.p, c.depth.p, c.W, c.H, c.gw, reinterpret_cast<int2*>(c.ras.p));
        else
            k_build_raster<<<dim3(ceil_div(c.hw(), 256), c.V), 256, 0, c.stream>>>(c.labels.p, c.depth.p, c.W, c.H,
                                                                                    c.gw, c.ras.p);
        LFDG_LAUNCHED(&c);
        auto launch = [&](auto kernel) {
            LFDG_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int per_sm = 0;
            LFDG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 32 * warps, smem));
            const int n_tasks = rn * c.nsp;
            const int blocks = std::max(1, std::min(per_sm * c.sm_count, (n_tasks + warps - 1) / warps));
            RefineScratch& rd = c.refine_s;
            rd.task_counter.alloc(1);
            rd.cand.alloc((size_t)blocks * warps * cap);
            rd.es.alloc((size_t)blocks * warps * cap);
            rd.acc.alloc((size_t)blocks * warps * cap);
            LFDG_CUDA_CHECK(cudaMemsetAsync(rd.task_counter.p, 0, sizeof(int), c.stream));
            kernel<<<blocks, 32 * warps, smem, c.stream>>>(a, n_tasks, rd.task_counter.p, cap, rd.cand.p, rd.es.p,
                                                          rd.acc.p);
        };
        // kFlat (flat above): every rotation I, canonical and identical K, every camera centre at
        // z = 0 (then every rel_trans.z = 0): the rectified / grid rigs of the fixtures.
        // kRecheck (stats mode): a separate instantiation carries the re-check, so the hot
        // variant's register allocation is untouched by it
        // kG: lanes per candidate slot as a compile-time constant for the hot (non-stats) variants
        // (the slot / target-lane arithmetic then folds to shifts and masks)
        auto pick = [&](auto rc, auto gc) {
            constexpr bool R = decltype(rc)::value;
            constexpr int KG = decltype(gc)::value;
            if (flat) {
                if (a.row_inv)
                    launch(k_refine<true, true, 2, R, KG>);
                else if (flat_mode == 3)
                    launch(k_refine<true, true, 3, R, KG>);
                else
                    launch(k_refine<true, true, 1, R, KG>);
            } else if (c.identity_rot && c.canonical_k) {
                launch(k_refine<true, true, 0, R, KG>);
            } else if (c.identity_rot) {
                launch(k_refine<true, false, 0, R, KG>);
            } else if (c.canonical_k) {
                launch(k_refine<false, true, 0, R, KG>);
            } else {
                launch(k_refine<false, false, 0, R, KG>);
            }
        };
        if (flat) {
            a.uK00 = c.cams[0].K[0];
            a.uK02 = c.cams[0].K[2];
            a.uK11 = c.cams[0].K[4];
            a.uK12 = c.cams[0].K[5];
        }
        const int G = lanes_per_candidate(a.N, flat_mode);
        if (recheck)
            pick(std::true_type{}, std::integral_constant<int, 0>{});
        else if (G == 8)
            pick(std::false_type{}, std::integral_constant<int, 8>{});
        else if (G == 16)
            pick(std::false_type{}, std::integral_constant<int, 16>{});
        else
            pick(std::false_type{}, std::integral_constant<int, 32>{});
        LFDG_LAUNCHED(&c);
        LFDG_CUDA_CHECK(cudaMemcpyAsync(c.planes.p + (size_t)rv0 * c.nsp, c.planes_next.p + (size_t)rv0 * c.nsp,
                                        (size_t)rn * c.nsp * sizeof(double4), cudaMemcpyDeviceToDevice, c.stream));
    }
}

}  // namespace lfdg
