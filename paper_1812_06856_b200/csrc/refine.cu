// Jacobi refinement on sm_100a: make_refine_context (refine.hpp:53-79) and refine_iteration
// (refine.hpp:253-323) with the full energy E = E_s * E_c (smoothness_term :84, pair_stats
// :111, consistency_term :189, energy :201, normal_candidates :213).
//
// One CTA per (view, superpixel) task.  The reference's per-task control flow is a sequential
// greedy over an ordered candidate list (propagation candidates in grid_neighbors(Kernel) order,
// then the triangle normals at the phase-A depth) that accepts a candidate iff its energy is
// strictly above the running best, pruning candidates whose upper bound E_s * (1 + eta) cannot
// beat it.  The CTA reproduces it exactly:
//   * the candidate list is enumerated in the reference order (ordered block compaction);
//   * E_s of every candidate is computed in parallel (one thread per candidate);
//   * candidates are evaluated in chunks, in order, against the running best at chunk
//     formation (a lower bound of the reference's running best, so every candidate the
//     reference evaluates is evaluated here); within a chunk one thread per (candidate,
//     target) pair runs pair_stats' member loop in the reference's pixel order, so every
//     FP64 sum is bit-identical; the chunk is then folded sequentially in index order.
// The winner is therefore the reference's plane and `accepted` its exact count.  A candidate
// identical to the running plane has e == e_cur exactly and is never accepted, so the
// reference's identity skip (refine.hpp:292) needs no special case.  exp/expf are the glibc
// ports (glibc_math.cuh).
#include <algorithm>
#include <cmath>

#include "context.h"
#include "glibc_math.cuh"

namespace lfdg {
namespace {

constexpr int kThreads = 128;
constexpr int kMaxCand = 512;  // propagation slots + 8 normals per task (checked on the host)

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
    unsigned long long* counters;
};

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

// depth_consistency (refine.hpp:34-37)
__device__ __forceinline__ double depth_consistency(double d1, double d2, double two_sigma2) {
    const double r = 1.0 / d1 - 1.0 / d2;
    return libm::exp(-(r * r) / two_sigma2);
}

// smoothness_term (refine.hpp:84-100) for candidate plane p of task (v, sp).
__device__ double smoothness(const RefineArgs& a, int v, int sp, double4 p) {
    const int gx = sp % a.gw, gy = sp / a.gw;
    const double2 cr = a.cray[(size_t)v * a.nsp + sp];
    const double ax = p.x * cr.x, ay = p.x * cr.y, az = p.x;
    const double num = (p.y * ax + p.z * ay) + p.w * az;
    const float* rw = a.ring_w + ((size_t)v * a.nsp + sp) * 8;
    double wsum = 0, acc = 0;
    for (int k = 0; k < 8; ++k) {
        const int nx = gx + kDir[k][0], ny = gy + kDir[k][1];
        if (nx < 0 || ny < 0 || nx >= a.gw || ny >= a.gh) continue;
        const int nb = ny * a.gw + nx;
        const double w = (double)rw[k];
        wsum += w;
        const double2 nr = a.cray[(size_t)v * a.nsp + nb];
        const double denom = (p.y * nr.x + p.z * nr.y) + p.w;
        if (fabs(denom) <= 1e-9) continue;
        const double ext = num / denom;
        if (ext <= 0) continue;
        acc += w * depth_consistency(a.planes[(size_t)v * a.nsp + nb].x, ext, a.two_sigma2);
    }
    if (wsum <= 1e-30) return 1.0;
    return acc / wsum;
}

// pair_stats (refine.hpp:111-172) -> visibility + occlusion, for one (candidate, target).
__device__ double pair_contrib(const RefineArgs& a, int v, int sp, double4 p, int ti) {
    const int t = a.targets[(size_t)v * a.N + ti];
    const double* rel = a.rel + ((size_t)v * a.N + ti) * 12;
    const double R0 = rel[0], R1 = rel[1], R2 = rel[2], R3 = rel[3], R4 = rel[4], R5 = rel[5];
    const double R6 = rel[6], R7 = rel[7], R8 = rel[8], T0 = rel[9], T1 = rel[10], T2 = rel[11];
    const Cam& tc = a.cams[t];
    const double K00 = tc.K[0], K01 = tc.K[1], K02 = tc.K[2], K11 = tc.K[4], K12 = tc.K[5];
    const size_t hw = (size_t)a.W * a.H;
    const int32_t* tl = a.labels + (size_t)t * hw;
    const float* tdep = a.depth + (size_t)t * hw;
    const float4* tcol = a.color + (size_t)t * a.nsp;
    const float4 rc = a.color[(size_t)v * a.nsp + sp];
    const double2 cr = a.cray[(size_t)v * a.nsp + sp];
    const double ax = p.x * cr.x, ay = p.x * cr.y, az = p.x;
    const double plane_num = (p.y * ax + p.z * ay) + p.w * az;
    const int m0 = a.moff[(size_t)v * (a.nsp + 1) + sp];
    const int n = a.moff[(size_t)v * (a.nsp + 1) + sp + 1] - m0;
    const double2* mr = a.mray + (size_t)v * hw + m0;

    double photo_sum = 0, vis_sum = 0;
    int x_count = 0;
    bool y_nonempty = false;
    int cached_label = -1;
    double cached_w = 0;
    for (int i = 0; i < n; ++i) {
        const double2 r = mr[i];
        const double denom = (p.y * r.x + p.z * r.y) + p.w;
        if (fabs(denom) <= 1e-9) continue;
        const double s = plane_num / denom;
        if (s <= 0) continue;
        const double sv0 = s * r.x, sv1 = s * r.y, sv2 = s;
        const double x0 = ((R0 * sv0 + R1 * sv1) + R2 * sv2) + T0;
        const double x1 = ((R3 * sv0 + R4 * sv1) + R5 * sv2) + T1;
        const double x2 = ((R6 * sv0 + R7 * sv1) + R8 * sv2) + T2;
        if (x2 <= 0) continue;
        const double u = ((K00 * x0 + K01 * x1) + K02 * x2) / x2;
        const double w = (K11 * x1 + K12 * x2) / x2;
        const int px = lround_int(u);
        const int py = lround_int(w);
        if (px < 0 || py < 0 || px >= a.W || py >= a.H) continue;
        const size_t q = (size_t)py * a.W + px;
        const int tlab = tl[q];
        if (tlab != cached_label) {
            cached_label = tlab;
            const float4 c = tcol[tlab];
            cached_w = libm::exp(-(double)color_dist2(rc.x, rc.y, rc.z, c.x, c.y, c.z) * a.inv_two_alpha2);
        }
        photo_sum += cached_w;
        const float td = tdep[q];
        if (td <= 0) continue;
        if (x2 <= (double)td * (1.0 + 1e-6)) {
            const double rr = 1.0 / x2 - 1.0 / (double)td;
            vis_sum += libm::exp(-rr * rr * a.inv_two_sigma2);
            ++x_count;
        } else {
            y_nonempty = true;
        }
    }
    const double photo = photo_sum / (double)n;
    const double vis = x_count > 0 ? photo * (vis_sum / x_count) : 0.0;
    double occ = 0.0;
    if (a.use_o && y_nonempty) occ = a.eta * (1.0 - (double)a.min_nb_sim[(size_t)v * a.nsp + sp]);
    return vis + occ;
}

struct Shared {
    double4 cand[kMaxCand];
    double es[kMaxCand];
    int sel[kThreads];
    double res[kThreads];  // per (chunk candidate, target) contribution
    double e_chunk[kThreads];
    int scan[kThreads];
    double4 current;
    double e_cur;
    int n_cand;
    int nsel;
    int next;
    unsigned accepted;
};

// Evaluate candidates [0, n_cand) of s.cand in chunks (see file comment).  Thread 0 owns
// s.current / s.e_cur.  `first_is_current`: s.cand[0] is the current plane and its energy
// initialises e_cur (refine.hpp:277) without an acceptance test.
__device__ void run_candidates(const RefineArgs& a, Shared& s, int v, int sp, bool init_pass) {
    const int tid = threadIdx.x;
    const int N = a.N;
    const int K = N > 0 ? max(1, kThreads / N) : kThreads;
    const bool prune = a.use_s && a.use_c;
    if (tid == 0) s.next = 0;
    __syncthreads();
    while (true) {
        if (tid == 0) {
            int k = 0, nx = s.next;
            while (nx < s.n_cand && k < K) {
                if (init_pass || !prune || s.es[nx] * a.max_consistency > s.e_cur) s.sel[k++] = nx;
                ++nx;
            }
            s.next = nx;
            s.nsel = k;
        }
        __syncthreads();
        const int nsel = s.nsel;
        if (nsel == 0) break;
        if (a.use_c && N > 0) {
            if (tid < nsel * N) {
                const int ci = tid / N, ti = tid % N;
                s.res[tid] = pair_contrib(a, v, sp, s.cand[s.sel[ci]], ti);
            }
            __syncthreads();
        }
        if (tid < nsel) {
            const int c = s.sel[tid];
            double e;
            if (a.use_c) {
                double ec = 1.0;
                if (N > 0) {
                    double acc = 0;
                    for (int ti = 0; ti < N; ++ti) acc += s.res[tid * N + ti];
                    ec = acc / (double)N;
                }
                e = prune ? s.es[c] * ec : (a.use_s ? 1.0 * s.es[c] : 1.0) * ec;
            } else {
                e = a.use_s ? 1.0 * s.es[c] : 1.0;
            }
            s.e_chunk[tid] = e;
        }
        __syncthreads();
        if (tid == 0) {
            for (int ci = 0; ci < nsel; ++ci) {
                const double e = s.e_chunk[ci];
                if (init_pass) {
                    s.e_cur = e;
                } else if (e > s.e_cur) {
                    s.e_cur = e;
                    s.current = s.cand[s.sel[ci]];
                    s.accepted++;
                }
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) k_refine(RefineArgs a) {
    __shared__ Shared s;
    const int tid = threadIdx.x;
    const int task = blockIdx.x;
    const int v = a.rv0 + task / a.nsp;
    const int sp = task % a.nsp;
    const size_t vs = (size_t)v * a.nsp;
    const double4 cur0 = a.planes[vs + sp];
    if (tid == 0) {
        s.current = cur0;
        s.accepted = 0;
        s.n_cand = 1;
        s.cand[0] = cur0;
    }
    __syncthreads();
    // ---- e_cur = energy(current) (refine.hpp:277)
    if (tid == 0 && a.use_s) s.es[0] = smoothness(a, v, sp, cur0);
    __syncthreads();
    run_candidates(a, s, v, sp, true);

    // ---- phase A: propagation candidates in grid_neighbors(Kernel) order (superpixel.hpp:318-343)
    const int gx = sp % a.gw, gy = sp / a.gw;
    const double2 crs = a.cray[vs + sp];
    int base = 0;
    for (int s0 = 0; s0 < a.n_slots; s0 += kThreads) {
        const int slot = s0 + tid;
        bool ok = false;
        double4 cand = make_double4(0, 0, 0, 0);
        if (slot < a.n_slots) {
            int dx, dy;
            if (slot < 8) {
                dx = kDir[slot][0];
                dy = kDir[slot][1];
            } else {
                const int k = (slot - 8) / a.per_dir;   // direction (kDir order)
                const int ri = (slot - 8) % a.per_dir;  // radius-minor: r = step, 2 step, ... <= radius_sp
                const int r = a.kernel_step * (ri + 1);
                dx = kDir[k][0] * r;
                dy = kDir[k][1] * r;
                if (abs(dx) <= 1 && abs(dy) <= 1) dx = 1 << 20;  // already in the ring (superpixel.hpp:334)
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
        // ordered block compaction
        s.scan[tid] = ok ? 1 : 0;
        __syncthreads();
        for (int off = 1; off < kThreads; off <<= 1) {
            const int t = tid >= off ? s.scan[tid - off] : 0;
            __syncthreads();
            s.scan[tid] += t;
            __syncthreads();
        }
        if (ok) s.cand[base + s.scan[tid] - 1] = cand;
        base += s.scan[kThreads - 1];
        __syncthreads();
    }
    if (tid == 0) s.n_cand = base;
    __syncthreads();
    if (a.use_s)
        for (int i = tid; i < base; i += kThreads) s.es[i] = smoothness(a, v, sp, s.cand[i]);
    __syncthreads();
    run_candidates(a, s, v, sp, false);

    // ---- phase B: normal_candidates (refine.hpp:213-242) at the current depth
    bool okn = false;
    double4 nc = make_double4(0, 0, 0, 0);
    const double cur_depth = s.current.x;
    if (tid < 8) {
        const int k = tid;
        const int ax_ = gx + kDir[k][0], ay_ = gy + kDir[k][1];
        const int bx_ = gx + kDir[(k + 1) % 8][0], by_ = gy + kDir[(k + 1) % 8][1];
        const bool ina = ax_ >= 0 && ay_ >= 0 && ax_ < a.gw && ay_ < a.gh;
        const bool inb = bx_ >= 0 && by_ >= 0 && bx_ < a.gw && by_ < a.gh;
        if (ina && inb) {
            const int ia = ay_ * a.gw + ax_, ib = by_ * a.gw + bx_;
            const double dr = cur0.x;  // snapshot depth of the reference superpixel
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
                if (!((n0 * crs.x + n1 * crs.y) + n2 >= 0)) {
                    if (!(cur_depth < a.d_min || cur_depth > a.d_max)) {
                        okn = true;
                        nc = make_double4(cur_depth, n0, n1, n2);
                    }
                }
            }
        }
    }
    s.scan[tid] = okn ? 1 : 0;
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int k = 0; k < 8; ++k) {
            const int t = s.scan[k];
            s.scan[k] = acc;
            acc += t;
        }
        s.n_cand = acc;
    }
    __syncthreads();
    if (okn) s.cand[s.scan[tid]] = nc;
    __syncthreads();
    if (a.use_s && tid < s.n_cand) s.es[tid] = smoothness(a, v, sp, s.cand[tid]);
    __syncthreads();
    run_candidates(a, s, v, sp, false);

    if (tid == 0) {
        a.out[vs + sp] = s.current;
        if (s.accepted) atomicAdd(&a.counters[0], (unsigned long long)s.accepted);
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

inline unsigned ceil_div(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }

struct RefineDev {
    DevBuf<double2> mray;
};
RefineDev& refine_dev() {
    static RefineDev d;
    return d;
}

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
    RefineDev& rd = refine_dev();
    rd.mray.alloc((size_t)c.V * c.hw());
    k_member_rays<<<dim3(ceil_div(c.hw(), 256), c.V), 256, 0, st>>>(c.mpix.p, c.d_cams.p, c.W, c.H, rd.mray.p);
    LFDG_LAUNCHED(&c);
    LFDG_CUDA_CHECK(cudaStreamSynchronize(st));
    t.ready = true;
}

void refine_iteration(Ctx& c, int l) {
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
    a.mray = refine_dev().mray.p;
    a.planes = c.planes.p;
    a.depth = c.depth.p;
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
    if (a.n_slots + 8 > kMaxCand) throw Error(LFDG_INVALID_PARAMS, "propagation kernel too large for the device task");
    if (a.N > kThreads) throw Error(LFDG_INVALID_PARAMS, "too many matching views for one CTA (max 128)");
    if (rn > 0) {
        k_refine<<<(unsigned)(rn * c.nsp), kThreads, 0, c.stream>>>(a);
        LFDG_LAUNCHED(&c);
        LFDG_CUDA_CHECK(cudaMemcpyAsync(c.planes.p + (size_t)rv0 * c.nsp, c.planes_next.p + (size_t)rv0 * c.nsp,
                                        (size_t)rn * c.nsp * sizeof(double4), cudaMemcpyDeviceToDevice, c.stream));
    }
}

}  // namespace lfdg
