// SLIC over-segmentation on sm_100a: slic_segment (superpixel.hpp:179-312).
//
// Pipeline per batch of views (blockIdx.z / blockIdx.y = view within the batch):
//   k_slic_init       centre init at cell mid-points          superpixel.hpp:196-213
//   10 x k_slic_assign  pixel-per-thread argmin over <=25 centres  superpixel.hpp:219-245
//        k_slic_update  warp-per-cluster ordered sums            superpixel.hpp:246-267
//   enforce_connectivity (superpixel.hpp:87-172):
//        k_ccl_*      union-find CCL, root = min pixel index == the reference's DFS component
//                     order (components are discovered in raster order of their first pixel)
//        k_keeper     largest component per label, ties -> smallest root (first encountered)
//        k_tile_*     ordered compaction of orphan roots
//        k_adj_*      orphan -> adjacent component lists
//        k_orphan_merge  one warp per view replays the reference's ordered rounds exactly
//   k_empty_repair    BFS-last-pixel donation, ordered by id   superpixel.hpp:272-308
//   recompute_stats (superpixel.hpp:55-83): k_bbox + scan + k_stats (ordered CSR + sums)
//
// Order-dependent double sums (colour sums) are kept in the reference's row-major order by
// having one lane own each cluster's accumulator while the warp scans the cluster's window
// row-major; integer sums (x, y, count) use warp reductions (exact in any order).
#include <algorithm>
#include <cstring>

#include "context.h"

namespace lfdg {
namespace {

constexpr int kTile = 1024;  // pixels per compaction tile

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------- centres -------------
__global__ void k_slic_init(const float4* __restrict__ lab, int W, int H, int S, int gw, int gh, int v0,
                            double* ccx, double* ccy, float4* ccol) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    const int nsp = gw * gh;
    if (id >= nsp) return;
    const int b = blockIdx.y;
    const size_t hw = (size_t)W * H;
    const int gx = id % gw, gy = id / gw;
    const int x0 = gx * S, x1 = min(W, x0 + S);
    const int y0 = gy * S, y1 = min(H, y0 + S);
    const double cx = 0.5 * (x0 + x1 - 1);
    const double cy = 0.5 * (y0 + y1 - 1);
    ccx[(size_t)b * nsp + id] = cx;
    ccy[(size_t)b * nsp + id] = cy;
    ccol[(size_t)b * nsp + id] = lab[(size_t)(v0 + b) * hw + (size_t)((int)cy) * W + (int)cx];
}

// ---------------------------------------------------------------- assign --------------
// One thread per pixel; candidates scanned gy-major, gx-minor (ids ascending); ties on d go
// to the smaller spatial distance, then to the first id (superpixel.hpp:227-241).
__global__ void __launch_bounds__(128) k_slic_assign(const float4* __restrict__ lab, int W, int H, int S, int gw,
                                                     int gh, float spatial_w, int v0, const double* __restrict__ ccx,
                                                     const double* __restrict__ ccy,
                                                     const float4* __restrict__ ccol, int32_t* labels, int* abox) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int b = blockIdx.z;
    const int nsp = gw * gh;
    const size_t hw = (size_t)W * H;
    // The block's candidate centres (one image row, <= 128 consecutive pixels: cells
    // [gxb0, gxb1] x [gy0, gy1]) staged in shared memory once instead of read per pixel
    extern __shared__ __align__(16) unsigned char smem[];
    const int pgy = y / S;
    const int gy0 = max(0, pgy - 2), gy1 = min(gh - 1, pgy + 2);
    const int xb = blockIdx.x * blockDim.x;
    const int gxb0 = max(0, xb / S - 2), gxb1 = min(gw - 1, min(W - 1, xb + (int)blockDim.x - 1) / S + 2);
    const int wb = gxb1 - gxb0 + 1;
    const int ne = (gy1 - gy0 + 1) * wb;
    double2* s_c = reinterpret_cast<double2*>(smem);
    float4* s_col = reinterpret_cast<float4*>(s_c + ne);
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
        const int id = (gy0 + e / wb) * gw + gxb0 + e % wb;
        s_c[e] = make_double2(ccx[(size_t)b * nsp + id], ccy[(size_t)b * nsp + id]);
        s_col[e] = ccol[(size_t)b * nsp + id];
    }
    __syncthreads();
    if (x >= W) return;
    const float4 pc = lab[(size_t)(v0 + b) * hw + (size_t)y * W + x];
    const int pgx = x / S;
    const float two_s = 2.f * S;
    // ds = (float)sqrt(D) > 2S is decided on D alone outside a +-2^-20 band around (2S)^2: there
    // the float rounding of the square root cannot move ds across 2S (ulp(2S) <= 2^-23 2S), so
    // the double square root is only taken for candidates that can be in range.
    const double d_far = (double)two_s * two_s * (1.0 + 0x1p-20);
    float best_d = 0.f, best_s = 0.f;
    int best = -1;
    const int gx0 = max(0, pgx - 2), gx1 = min(gw - 1, pgx + 2);
    for (int gy = gy0; gy <= gy1; ++gy) {
        for (int gx = gx0; gx <= gx1; ++gx) {
            const int id = gy * gw + gx;
            const int e = (gy - gy0) * wb + (gx - gxb0);
            const double2 cc = s_c[e];
            const double ddx = (double)x - cc.x;
            const double ddy = (double)y - cc.y;
            const double D = ddx * ddx + ddy * ddy;
            if (D > d_far) continue;  // ds > 2S for sure
            const float ds = (float)sqrt(D);
            if (ds > two_s) continue;
            const float4 c = s_col[e];
            const float dc = sqrtf(color_dist2(pc.x, pc.y, pc.z, c.x, c.y, c.z));
            const float d = dc + spatial_w * ds;
            if (best < 0 || d < best_d || (d == best_d && ds < best_s)) {
                best_d = d;
                best_s = ds;
                best = id;
            }
        }
    }
    labels[(size_t)(v0 + b) * hw + (size_t)y * W + x] = best;
    // the cluster's pixel bbox for k_slic_update, as four minima (x, y, -x, -y); the lanes of a
    // warp share y and have consecutive x, so one lane per label of the warp updates it
    const unsigned am = __activemask();
    const unsigned peers = __match_any_sync(am, best);
    const int lane = threadIdx.x & 31;
    if (lane == __ffs(peers) - 1) {
        int* bx = abox + ((size_t)b * nsp + best) * 4;
        atomicMin(bx + 0, x);
        atomicMin(bx + 1, y);
        atomicMin(bx + 2, -(x - lane + (31 - __clz(peers))));
        atomicMin(bx + 3, -y);
    }
}

// ---------------------------------------------------------------- update --------------
// Warp per cluster. A pixel can only take a label whose cell is within +-2 cells of its own
// (k_slic_assign), so cluster (gx, gy)'s members lie in the pixel window of cells
// [gx-2, gx+2] x [gy-2, gy+2]; scanning it row-major visits members in the reference's order.
__global__ void __launch_bounds__(256) k_slic_update(const float4* __restrict__ lab,
                                                     const int32_t* __restrict__ labels, int W, int H, int S,
                                                     int gw, int gh, int v0, double* ccx, double* ccy,
                                                     float4* ccol, const int* __restrict__ abox) {
    const int nsp = gw * gh;
    const int id = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    if (id >= nsp) return;
    const size_t hw = (size_t)W * H;
    const int32_t* lb = labels + (size_t)(v0 + b) * hw;
    const float4* im = lab + (size_t)(v0 + b) * hw;
    // the members lie in the cluster's assignment bbox (k_slic_assign), itself inside the window
    // of cells [gx-2, gx+2] x [gy-2, gy+2]; empty bbox: no members
    const int* bx = abox + ((size_t)b * nsp + id) * 4;
    const int xa = max(0, bx[0]), xb = min(W, 1 - bx[2]);
    const int ya = max(0, bx[1]), yb = min(H, 1 - bx[3]);
    // colour sums: lane k < 3 owns channel k's sequential sum; each step's member colours are
    // converted to double by the member lanes (all 32 at once: the conversion unit is the
    // kernel's bottleneck when three lanes convert member by member), staged in shared memory and
    // added in ascending lane (= row-major pixel) order
    __shared__ double4 s_col[8][32];
    double4* buf = s_col[(threadIdx.x >> 5) & 7];
    const double* bch = reinterpret_cast<const double*>(buf) + (lane < 3 ? lane : 0);
    long long sx = 0, sy = 0;
    int cnt = 0;
    double sc = 0;  // this lane's channel sum (lanes 0-2)
    // (row, 32-wide chunk) steps in row-major order, software-pipelined by one step: the label
    // and colour of the next step are loaded before the current one is consumed
    int ny = ya, nx = xa;  // next step to load
    auto load = [&](int& lv, float4& cv) {
        const int x = nx + lane;
        lv = -1;
        if (x < xb) {
            const size_t o = (size_t)ny * W + x;
            lv = lb[o];
            cv = im[o];
        }
        nx += 32;
        if (nx >= xb) {
            nx = xa;
            ++ny;
        }
    };
    int l_next = -1;
    float4 c_next = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool any = ya < yb && xa < xb;
    if (any) load(l_next, c_next);
    for (int y = ya, xc = xa; any && y < yb;) {
        const int lv = l_next;
        const float4 cv = c_next;
        if (ny < yb) load(l_next, c_next);
        const int x = xc + lane;
        xc += 32;
        const int yc = y;
        if (xc >= xb) {
            xc = xa;
            ++y;
        }
        {
            const int y = yc;
            const bool m = lv == id;
            unsigned mask = __ballot_sync(LFDG_FULL_MASK, m);
            if (!mask) continue;
            if (m) buf[lane] = make_double4((double)cv.x, (double)cv.y, (double)cv.z, 0.0);
            const int n = __popc(mask);
            sx += __reduce_add_sync(LFDG_FULL_MASK, m ? (unsigned)x : 0u);
            sy += (long long)y * n;
            cnt += n;
            __syncwarp();
            if (lane < 3) {
                while (mask) {
                    const int j = __ffs(mask) - 1;
                    mask &= mask - 1;
                    sc += bch[4 * j];
                }
            }
            __syncwarp();
        }
    }
    const double s0 = sc;
    const double s1 = __shfl_sync(LFDG_FULL_MASK, sc, 1);
    const double s2 = __shfl_sync(LFDG_FULL_MASK, sc, 2);
    if (lane == 0 && cnt > 0) {
        const size_t o = (size_t)b * nsp + id;
        ccx[o] = (double)sx / cnt;
        ccy[o] = (double)sy / cnt;
        ccol[o] = make_float4((float)(s0 / cnt), (float)(s1 / cnt), (float)(s2 / cnt), 0.f);
    }
}

// ---------------------------------------------------------------- CCL -----------------
__device__ __forceinline__ int uf_find(const int* P, int a) {
    const volatile int* vp = P;
    int p = vp[a];
    while (p != a) {
        a = p;
        p = vp[a];
    }
    return a;
}

__device__ __forceinline__ void uf_union(int* P, int a, int b) {
    bool done;
    do {
        a = uf_find(P, a);
        b = uf_find(P, b);
        if (a < b) {
            const int old = atomicMin(&P[b], a);
            done = (old == b);
            b = old;
        } else if (b < a) {
            const int old = atomicMin(&P[a], b);
            done = (old == a);
            a = old;
        } else {
            done = true;
        }
    } while (!done);
}

__global__ void k_ccl_init(int W, int H, int* parent, int* csize, int* orphan_idx) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const size_t o = (size_t)blockIdx.y * hw + i;
    parent[o] = (int)i;
    csize[o] = 0;
    orphan_idx[o] = -1;
}

__global__ void k_ccl_merge(const int32_t* __restrict__ labels, int W, int H, int v0, int* parent) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const int b = blockIdx.y;
    const int32_t* lb = labels + (size_t)(v0 + b) * hw;
    int* P = parent + (size_t)b * hw;
    const int x = (int)(i % W), y = (int)(i / W);
    const int32_t l = lb[i];
    if (x + 1 < W && lb[i + 1] == l) uf_union(P, (int)i, (int)i + 1);
    if (y + 1 < H && lb[i + W] == l) uf_union(P, (int)i, (int)(i + W));
}

__global__ void k_ccl_compress(int W, int H, int* parent, int* csize) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    int* P = parent + (size_t)blockIdx.y * hw;
    const int r = uf_find(P, (int)i);
    P[i] = r;
    atomicAdd(&csize[(size_t)blockIdx.y * hw + r], 1);
}

// Keeper of each label: the largest component, ties to the one discovered first (smallest
// root): key = size << 32 | (0xffffffff - root), maximised.
__global__ void k_keeper(const int32_t* __restrict__ labels, int W, int H, int nsp, int v0, const int* parent,
                         const int* csize, unsigned long long* keeper) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const int b = blockIdx.y;
    if (parent[(size_t)b * hw + i] != (int)i) return;
    const int32_t l = labels[(size_t)(v0 + b) * hw + i];
    const unsigned long long key =
        ((unsigned long long)csize[(size_t)b * hw + i] << 32) | (0xffffffffull - (unsigned long long)i);
    atomicMax(&keeper[(size_t)b * nsp + l], key);
}

__device__ __forceinline__ bool is_orphan_root(const int32_t* lb, const int* P, const unsigned long long* keeper,
                                               size_t i) {
    if (P[i] != (int)i) return false;
    const unsigned long long k = keeper[lb[i]];
    const unsigned root = 0xffffffffu - (unsigned)(k & 0xffffffffull);
    return root != (unsigned)i;
}

// Ordered compaction of orphan roots: per-tile counts, scanned, then written in order.
__global__ void k_tile_count(const int32_t* __restrict__ labels, int W, int H, int nsp, int v0, const int* parent,
                             const unsigned long long* keeper, int* tile_cnt, int n_tiles) {
    const size_t hw = (size_t)W * H;
    const int b = blockIdx.y;
    const size_t i = (size_t)blockIdx.x * kTile + threadIdx.x;
    __shared__ int s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    bool f = false;
    if (i < hw)
        f = is_orphan_root(labels + (size_t)(v0 + b) * hw, parent + (size_t)b * hw, keeper + (size_t)b * nsp, i);
    const unsigned m = __ballot_sync(LFDG_FULL_MASK, f);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(&s, __popc(m));
    __syncthreads();
    if (threadIdx.x == 0) tile_cnt[(size_t)b * n_tiles + blockIdx.x] = s;
}

__global__ void k_tile_write(const int32_t* __restrict__ labels, int W, int H, int nsp, int v0, const int* parent,
                             const unsigned long long* keeper, const int* tile_off, int n_tiles, int* orphan_list,
                             int* orphan_idx) {
    const size_t hw = (size_t)W * H;
    const int b = blockIdx.y;
    const size_t i = (size_t)blockIdx.x * kTile + threadIdx.x;
    __shared__ int warp_base[kTile / 32];
    bool f = false;
    if (i < hw)
        f = is_orphan_root(labels + (size_t)(v0 + b) * hw, parent + (size_t)b * hw, keeper + (size_t)b * nsp, i);
    const unsigned m = __ballot_sync(LFDG_FULL_MASK, f);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) warp_base[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int k = 0; k < kTile / 32; ++k) {
            const int t = warp_base[k];
            warp_base[k] = acc;
            acc += t;
        }
    }
    __syncthreads();
    if (f) {
        const int pos = tile_off[(size_t)b * (n_tiles + 1) + blockIdx.x] + warp_base[w] + __popc(m & lanemask_lt());
        orphan_list[(size_t)b * hw + pos] = (int)i;
        orphan_idx[(size_t)b * hw + i] = pos;
    }
}

// Exclusive scan of `len` ints per row (rows = blockIdx.x); out has len+1 entries per row,
// out[len] = total.  len_dev (nullable) gives a per-row length read on the device.
__global__ void __launch_bounds__(1024) k_scan_rows(const int* in, size_t in_stride, int* out, size_t out_stride,
                                                    int len, const int* len_dev) {
    const int row = blockIdx.x;
    const int n = len_dev ? len_dev[row] : len;
    const int* a = in + (size_t)row * in_stride;
    int* o = out + (size_t)row * out_stride;
    __shared__ int sums[1024];
    const int per = (n + 1023) / 1024;
    const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
    int s = 0;
    for (int k = lo; k < hi; ++k) s += a[k];
    sums[threadIdx.x] = s;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const int v = threadIdx.x >= off ? sums[threadIdx.x - off] : 0;
        __syncthreads();
        sums[threadIdx.x] += v;
        __syncthreads();
    }
    int acc = sums[threadIdx.x] - s;
    for (int k = lo; k < hi; ++k) {
        const int t = a[k];
        o[k] = acc;
        acc += t;
    }
    if (threadIdx.x == 1023) o[n] = sums[1023];
}

// Orphan -> adjacent components (4-neighbours in other components).  Entries: >= 0 is an
// orphan index, < 0 is a keeper with label -(entry + 1).
__global__ void k_adj(const int32_t* __restrict__ labels, int W, int H, int v0, const int* parent,
                      const int* orphan_idx, int* adj_cnt, const int* adj_off, int* adj_cur, int* adj) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const int b = blockIdx.y;
    const int* P = parent + (size_t)b * hw;
    const int* oi = orphan_idx + (size_t)b * hw;
    const int r = P[i];
    const int j = oi[r];
    if (j < 0) return;
    const int x = (int)(i % W), y = (int)(i / W);
    const int dx[4] = {1, -1, 0, 0}, dy[4] = {0, 0, 1, -1};
    for (int k = 0; k < 4; ++k) {
        const int nx = x + dx[k], ny = y + dy[k];
        if (nx < 0 || ny < 0 || nx >= W || ny >= H) continue;
        const size_t q = (size_t)ny * W + nx;
        const int rq = P[q];
        if (rq == r) continue;
        if (!adj) {
            atomicAdd(&adj_cnt[(size_t)b * hw + j], 1);
        } else {
            const int jq = oi[rq];
            const int e = jq >= 0 ? jq : -(labels[(size_t)(v0 + b) * hw + rq] + 1);
            const int pos = atomicAdd(&adj_cur[(size_t)b * hw + j], 1);
            adj[(size_t)b * 4 * hw + adj_off[(size_t)b * (hw + 1) + j] + pos] = e;
        }
    }
}

// The reference's merge rounds (superpixel.hpp:139-171), replayed in component order by one
// warp per view: count[] and assigned[] evolve exactly as in the sequential loop.  Lanes
// evaluate an orphan's adjacency list in parallel; the max over the strict total order
// (count desc, label asc) is order-independent, so only the orphan order matters.
__global__ void __launch_bounds__(32) k_orphan_merge(const int32_t* __restrict__ labels, int W, int H, int nsp,
                                                     int v0, const int* parent, const int* csize,
                                                     const unsigned long long* keeper, const int* orphan_list,
                                                     const int* tile_off, int n_tiles, const int* adj_off,
                                                     const int* adj, int* g_count, int* g_merged,
                                                     unsigned char* g_assigned, int smem_cap) {
    extern __shared__ int sm[];
    const int b = blockIdx.x;
    const int lane = threadIdx.x;
    const size_t hw = (size_t)W * H;
    const int n_orph = tile_off[(size_t)b * (n_tiles + 1) + n_tiles];
    if (n_orph == 0) return;
    const bool in_smem = (size_t)nsp * 4 + (size_t)n_orph * 9 <= (size_t)smem_cap;
    int* count = in_smem ? sm : g_count + (size_t)b * nsp;
    int* merged = in_smem ? sm + nsp : g_merged + (size_t)b * hw;
    int* osize = in_smem ? sm + nsp + n_orph : nullptr;
    unsigned char* assigned =
        in_smem ? reinterpret_cast<unsigned char*>(sm + nsp + 2 * n_orph) : g_assigned + (size_t)b * hw;
    const int32_t* lb = labels + (size_t)(v0 + b) * hw;
    const int* cs = csize + (size_t)b * hw;
    const int* ol = orphan_list + (size_t)b * hw;
    const int* aoff = adj_off + (size_t)b * (hw + 1);
    const int* ad = adj + (size_t)b * 4 * hw;
    // count[label] = size of the label's keeper (every label that has pixels has one).
    for (int l = lane; l < nsp; l += 32) {
        const unsigned long long k = keeper[(size_t)b * nsp + l];
        count[l] = (int)(k >> 32);
    }
    for (int j = lane; j < n_orph; j += 32) {
        merged[j] = lb[ol[j]];
        assigned[j] = 0;
        if (osize) osize[j] = cs[ol[j]];
    }
    __syncwarp();
    volatile int* vcount = count;
    volatile int* vmerged = merged;
    volatile unsigned char* vassigned = assigned;
    bool progress = true;
    while (progress) {
        progress = false;
        bool pending = false;
        for (int j = 0; j < n_orph; ++j) {
            if (vassigned[j]) continue;
            const int a0 = aoff[j], a1 = aoff[j + 1];
            unsigned long long best = 0;
            for (int k = a0 + lane; k < a1; k += 32) {
                const int e = ad[k];
                int nl = -1;
                if (e < 0) {
                    nl = -(e + 1);
                } else if (vassigned[e]) {
                    nl = vmerged[e];
                }
                if (nl >= 0) {
                    const unsigned long long key =
                        ((unsigned long long)(unsigned)vcount[nl] << 32) | (0xffffffffull - (unsigned)nl);
                    best = key > best ? key : best;
                }
            }
            for (int off = 16; off; off >>= 1) {
                const unsigned long long o = __shfl_xor_sync(LFDG_FULL_MASK, best, off);
                best = o > best ? o : best;
            }
            if (best == 0) {
                pending = true;
                continue;
            }
            const int bl = (int)(0xffffffffu - (unsigned)(best & 0xffffffffull));
            if (lane == 0) {
                vmerged[j] = bl;
                vassigned[j] = 1;
                vcount[bl] = vcount[bl] + (osize ? osize[j] : cs[ol[j]]);
            }
            __syncwarp();
            progress = true;
        }
        if (!pending) break;
    }
    __syncwarp();
    // Publish the merge result for k_relabel (always in global memory).
    for (int j = lane; j < n_orph; j += 32) {
        g_merged[(size_t)b * hw + j] = vassigned[j] ? vmerged[j] : -1;
    }
}

__global__ void k_relabel(int32_t* labels, int W, int H, int v0, const int* parent, const int* orphan_idx,
                          const int* g_merged) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const int b = blockIdx.y;
    const int r = parent[(size_t)b * hw + i];
    const int j = orphan_idx[(size_t)b * hw + r];
    if (j < 0) return;
    const int m = g_merged[(size_t)b * hw + j];
    if (m >= 0) labels[(size_t)(v0 + b) * hw + i] = m;
}

// ---------------------------------------------------------------- stats ---------------
__global__ void k_fix_bbox_hi(int* bb, size_t m) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        bb[i * 4 + 1] = -1;
        bb[i * 4 + 3] = -1;
    }
}

// Per-view orphan count (the last entry of each view's tile-offset row).
__global__ void k_gather_counts(const int* tile_off, int n_tiles, int n, int* out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < n) out[b] = tile_off[(size_t)b * (n_tiles + 1) + n_tiles];
}

// Pixel count per label (superpixel.hpp:275-276), warp-aggregated.
__global__ void k_label_hist(const int32_t* __restrict__ labels, int W, int H, int nsp, int v0, int* cnt) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    const int l = i < hw ? labels[(size_t)(v0 + b) * hw + i] : -1;
    const unsigned peers = __match_any_sync(LFDG_FULL_MASK, l);
    if (l < 0) return;
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&cnt[(size_t)b * nsp + l], __popc(peers));
}

__global__ void k_fill_int(int* p, size_t n, int v) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// Per-label bounding box + pixel count with warp-aggregated atomics (lanes = 32 consecutive
// pixels of one row).
__global__ void k_bbox(const int32_t* __restrict__ labels, int W, int H, int nsp, int v0, int* bbox, int* cnt) {
    const int b = blockIdx.z;
    const int y = blockIdx.y;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t hw = (size_t)W * H;
    const int l = x < W ? labels[(size_t)(v0 + b) * hw + (size_t)y * W + x] : -1;
    const unsigned peers = __match_any_sync(LFDG_FULL_MASK, l);
    if (l < 0) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    if (lane != leader) return;
    const int last = 31 - __clz(peers);
    int* bb = bbox + ((size_t)b * nsp + l) * 4;
    atomicMin(&bb[0], x);
    atomicMax(&bb[1], x + (last - leader));
    atomicMin(&bb[2], y);
    atomicMax(&bb[3], y);
    atomicAdd(&cnt[(size_t)b * nsp + l], __popc(peers));
}

// recompute_stats (superpixel.hpp:55-83) + grid.pixels CSR, warp per label scanning its
// bounding box row-major.  Also the centroid ray used by rasterize/refine.
__global__ void __launch_bounds__(256) k_stats(const float4* __restrict__ lab, const int32_t* __restrict__ labels,
                                               int W, int H, int nsp, int v0, const int* bbox,
                                               const int* __restrict__ moff_b, const Cam* cams, int32_t* mpix,
                                               double* cx_out, double* cy_out, float4* col_out, int32_t* cnt_out,
                                               double2* cray) {
    const int id = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    if (id >= nsp) return;
    const int v = v0 + b;
    const size_t hw = (size_t)W * H;
    const int32_t* lb = labels + (size_t)v * hw;
    const float4* im = lab + (size_t)v * hw;
    const int* bb = bbox + ((size_t)b * nsp + id) * 4;
    const int xa = bb[0], xb = bb[1] + 1, ya = bb[2], yb = bb[3] + 1;
    const int base = moff_b[(size_t)b * (nsp + 1) + id];
    int32_t* mp = mpix + (size_t)v * hw + base;
    long long sx = 0, sy = 0;
    int cnt = 0;
    double s0 = 0, s1 = 0, s2 = 0;
    for (int y = ya; y < yb; ++y) {
        for (int xc = xa; xc < xb; xc += 32) {
            const int x = xc + lane;
            const bool m = x < xb && lb[(size_t)y * W + x] == id;
            unsigned mask = __ballot_sync(LFDG_FULL_MASK, m);
            if (!mask) continue;
            float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
            if (m) {
                c = im[(size_t)y * W + x];
                mp[cnt + __popc(mask & lanemask_lt())] = y * W + x;
            }
            const int n = __popc(mask);
            sx += __reduce_add_sync(LFDG_FULL_MASK, m ? (unsigned)x : 0u);
            sy += (long long)y * n;
            cnt += n;
            while (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                const float a0 = __shfl_sync(LFDG_FULL_MASK, c.x, j);
                const float a1 = __shfl_sync(LFDG_FULL_MASK, c.y, j);
                const float a2 = __shfl_sync(LFDG_FULL_MASK, c.z, j);
                s0 += (double)a0;
                s1 += (double)a1;
                s2 += (double)a2;
            }
        }
    }
    if (lane == 0) {
        const size_t o = (size_t)v * nsp + id;
        double cx = 0, cy = 0;
        float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
        if (cnt > 0) {
            cx = (double)sx / cnt;
            cy = (double)sy / cnt;
            col = make_float4((float)(s0 / cnt), (float)(s1 / cnt), (float)(s2 / cnt), 0.f);
        }
        cx_out[o] = cx;
        cy_out[o] = cy;
        col_out[o] = col;
        cnt_out[o] = cnt;
        double rx, ry;
        cam_ray(cams[v], cx, cy, rx, ry);
        cray[o] = make_double2(rx, ry);
    }
}

// Empty-cluster repair (superpixel.hpp:272-308), one warp per view: the ordered list of
// empty ids is found with ballots; each is handled by lane 0 with the reference's BFS
// (neighbour order +x, -x, +y, -y) and donates the BFS-last pixel.
__global__ void __launch_bounds__(32) k_empty_repair(int32_t* labels, int W, int H, int S, int gw, int gh, int v0,
                                                     int* cnt, int* queue, int* seen) {
    const int b = blockIdx.x;
    const int lane = threadIdx.x;
    const int nsp = gw * gh;
    const size_t hw = (size_t)W * H;
    int32_t* lb = labels + (size_t)(v0 + b) * hw;
    int* cn = cnt + (size_t)b * nsp;
    int* q = queue + (size_t)b * hw;
    int* sn = seen + (size_t)b * hw;
    int stamp = 0;
    for (int base = 0; base < nsp; base += 32) {
        const int id0 = base + lane;
        unsigned empty = __ballot_sync(LFDG_FULL_MASK, id0 < nsp && cn[id0] == 0);
        while (empty) {
            const int j = __ffs(empty) - 1;
            empty &= empty - 1;
            const int id = base + j;
            if (lane == 0) {
                const int gx = id % gw, gy = id / gw;
                const int x = min(W - 1, gx * S + S / 2);
                const int y = min(H - 1, gy * S + S / 2);
                const int old = lb[(size_t)y * W + x];
                if (cn[old] > 1) {
                    ++stamp;
                    int head = 0, tail = 0;
                    q[tail++] = y * W + x;
                    sn[y * W + x] = stamp;
                    int last = q[0];
                    while (head < tail) {
                        last = q[head++];
                        const int px = last % W, py = last / W;
                        const int nb[4][2] = {{px + 1, py}, {px - 1, py}, {px, py + 1}, {px, py - 1}};
                        for (int k = 0; k < 4; ++k) {
                            const int qx = nb[k][0], qy = nb[k][1];
                            if (qx < 0 || qy < 0 || qx >= W || qy >= H) continue;
                            const int qi = qy * W + qx;
                            if (sn[qi] != stamp && lb[qi] == old) {
                                sn[qi] = stamp;
                                q[tail++] = qi;
                            }
                        }
                    }
                    lb[last] = id;
                    cn[old] -= 1;
                    cn[id] = 1;
                }
            }
            __syncwarp();
        }
    }
}

inline unsigned ceil_div(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }

// Final stats + CSR for views [v0, v0+n) from their label maps.
void recompute_stats(Ctx& c, int v0, int n) {
    SlicScratch& s = c.slic_s;
    const size_t hw = c.hw();
    const int nsp = c.nsp;
    cudaStream_t st = c.stream;
    s.bbox.alloc((size_t)n * nsp * 4);
    s.lcnt.alloc((size_t)n * nsp);
    s.moff_b.alloc((size_t)n * (nsp + 1));
    // bbox init: x0 = INT_MAX, x1 = -1, y0 = INT_MAX, y1 = -1
    {
        const size_t m = (size_t)n * nsp;
        k_fill_int<<<ceil_div(m * 4, 256), 256, 0, st>>>(s.bbox.p, m * 4, 0x7fffffff);
        LFDG_LAUNCHED(&c);
        LFDG_CUDA_CHECK(cudaMemsetAsync(s.lcnt.p, 0, m * sizeof(int), st));
    }
    k_fix_bbox_hi<<<ceil_div((size_t)n * nsp, 256), 256, 0, st>>>(s.bbox.p, (size_t)n * nsp);
    LFDG_LAUNCHED(&c);
    {
        dim3 g(ceil_div(c.W, 128), c.H, n);
        k_bbox<<<g, 128, 0, st>>>(c.labels.p, c.W, c.H, nsp, v0, s.bbox.p, s.lcnt.p);
        LFDG_LAUNCHED(&c);
    }
    k_scan_rows<<<n, 1024, 0, st>>>(s.lcnt.p, nsp, s.moff_b.p, nsp + 1, nsp, nullptr);
    LFDG_LAUNCHED(&c);
    {
        dim3 g(ceil_div((size_t)nsp * 32, 256), n);
        k_stats<<<g, 256, 0, st>>>(c.lab.p, c.labels.p, c.W, c.H, nsp, v0, s.bbox.p, s.moff_b.p, c.d_cams.p,
                                   c.mpix.p, c.cx.p, c.cy.p, c.color.p, c.count.p, c.cray.p);
        LFDG_LAUNCHED(&c);
    }
    for (int b = 0; b < n; ++b)
        LFDG_CUDA_CHECK(cudaMemcpyAsync(c.moff.p + (size_t)(v0 + b) * (nsp + 1), s.moff_b.p + (size_t)b * (nsp + 1),
                                        (nsp + 1) * sizeof(int), cudaMemcpyDeviceToDevice, st));
}

}  // namespace

void ensure_grid_buffers(Ctx& c, int S) {
    c.require_views();
    const int gw = (c.W + S - 1) / S, gh = (c.H + S - 1) / S;
    if (S == c.S && c.labels.p) return;
    c.S = S;
    c.gw = gw;
    c.gh = gh;
    c.nsp = gw * gh;
    const size_t hw = c.hw();
    c.labels.alloc((size_t)c.V * hw);
    c.mpix.alloc((size_t)c.V * hw);
    c.moff.alloc((size_t)c.V * (c.nsp + 1));
    c.count.alloc((size_t)c.V * c.nsp);
    c.cx.alloc((size_t)c.V * c.nsp);
    c.cy.alloc((size_t)c.V * c.nsp);
    c.color.alloc((size_t)c.V * c.nsp);
    c.cray.alloc((size_t)c.V * c.nsp);
    c.planes.alloc((size_t)c.V * c.nsp);
    c.planes_next.alloc((size_t)c.V * c.nsp);
    c.grid_ready.assign(c.V, 0);
    c.planes_ready.assign(c.V, 0);
    c.refine.ready = false;
}

void slic_views(Ctx& c, int v0, int n, const lfdg_slic_params& p) {
    if (p.size < 4) throw Error(LFDG_INVALID_PARAMS, "superpixel size must be >= 4");
    if (!(p.compactness > 0)) throw Error(LFDG_INVALID_PARAMS, "compactness must be > 0");
    if (p.iterations < 1) throw Error(LFDG_INVALID_PARAMS, "iterations must be >= 1");
    c.require_views();
    if (v0 < 0 || n < 0 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    if (c.W < p.size || c.H < p.size) throw Error(LFDG_INVALID_PARAMS, "image smaller than superpixel size");
    if (n == 0) return;
    ensure_grid_buffers(c, p.size);
    SlicScratch& s = c.slic_s;
    const size_t hw = c.hw();
    const int S = p.size, gw = c.gw, gh = c.gh, nsp = c.nsp;
    const int W = c.W, H = c.H;
    cudaStream_t st = c.stream;
    s.ccx.alloc((size_t)n * nsp);
    s.ccy.alloc((size_t)n * nsp);
    s.ccol.alloc((size_t)n * nsp);

    k_slic_init<<<dim3(ceil_div(nsp, 128), n), 128, 0, st>>>(c.lab.p, W, H, S, gw, gh, v0, s.ccx.p, s.ccy.p,
                                                                s.ccol.p);
    LFDG_LAUNCHED(&c);
    const float spatial_w = p.compactness / static_cast<float>(S);
    s.abox.alloc((size_t)n * nsp * 4);
    // staged centres of one assign block: <= 128 / S + 6 cells per row band, 5 band rows
    const size_t assign_smem = (size_t)(128 / S + 6) * 5 * (sizeof(double2) + sizeof(float4));
    if (assign_smem > 48 * 1024)
        LFDG_CUDA_CHECK(cudaFuncSetAttribute(k_slic_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)assign_smem));
    for (int it = 0; it < p.iterations; ++it) {
        LFDG_CUDA_CHECK(cudaMemsetAsync(s.abox.p, 0x7f, (size_t)n * nsp * 4 * sizeof(int), st));  // empty boxes
        k_slic_assign<<<dim3(ceil_div(W, 128), H, n), 128, assign_smem, st>>>(c.lab.p, W, H, S, gw, gh, spatial_w, v0, s.ccx.p,
                                                                     s.ccy.p, s.ccol.p, c.labels.p, s.abox.p);
        LFDG_LAUNCHED(&c);
        k_slic_update<<<dim3(ceil_div((size_t)nsp * 32, 256), n), 256, 0, st>>>(c.lab.p, c.labels.p, W, H, S, gw, gh,
                                                                               v0, s.ccx.p, s.ccy.p, s.ccol.p,
                                                                               s.abox.p);
        LFDG_LAUNCHED(&c);
    }

    // ---- enforce_connectivity
    s.parent.alloc((size_t)n * hw);
    s.csize.alloc((size_t)n * hw);
    s.orphan_idx.alloc((size_t)n * hw);
    s.orphan_list.alloc((size_t)n * hw);
    s.keeper.alloc((size_t)n * nsp);
    const int n_tiles = (int)ceil_div(hw, kTile);
    s.tile_cnt.alloc((size_t)n * n_tiles);
    s.tile_off.alloc((size_t)n * (n_tiles + 1));
    const dim3 gp(ceil_div(hw, 256), n);
    k_ccl_init<<<gp, 256, 0, st>>>(W, H, s.parent.p, s.csize.p, s.orphan_idx.p);
    LFDG_LAUNCHED(&c);
    k_ccl_merge<<<gp, 256, 0, st>>>(c.labels.p, W, H, v0, s.parent.p);
    LFDG_LAUNCHED(&c);
    k_ccl_compress<<<gp, 256, 0, st>>>(W, H, s.parent.p, s.csize.p);
    LFDG_LAUNCHED(&c);
    LFDG_CUDA_CHECK(cudaMemsetAsync(s.keeper.p, 0, (size_t)n * nsp * sizeof(unsigned long long), st));
    k_keeper<<<gp, 256, 0, st>>>(c.labels.p, W, H, nsp, v0, s.parent.p, s.csize.p, s.keeper.p);
    LFDG_LAUNCHED(&c);
    k_tile_count<<<dim3(n_tiles, n), kTile, 0, st>>>(c.labels.p, W, H, nsp, v0, s.parent.p, s.keeper.p,
                                                     s.tile_cnt.p, n_tiles);
    LFDG_LAUNCHED(&c);
    k_scan_rows<<<n, 1024, 0, st>>>(s.tile_cnt.p, n_tiles, s.tile_off.p, n_tiles + 1, n_tiles, nullptr);
    LFDG_LAUNCHED(&c);
    k_tile_write<<<dim3(n_tiles, n), kTile, 0, st>>>(c.labels.p, W, H, nsp, v0, s.parent.p, s.keeper.p, s.tile_off.p,
                                                     n_tiles, s.orphan_list.p, s.orphan_idx.p);
    LFDG_LAUNCHED(&c);
    // adjacency lists (count, scan, fill)
    s.adj_cnt.alloc((size_t)n * hw);
    s.adj_off.alloc((size_t)n * (hw + 1));
    s.adj_cur.alloc((size_t)n * hw);
    s.adj.alloc((size_t)n * 4 * hw);
    LFDG_CUDA_CHECK(cudaMemsetAsync(s.adj_cnt.p, 0, (size_t)n * hw * sizeof(int), st));
    LFDG_CUDA_CHECK(cudaMemsetAsync(s.adj_cur.p, 0, (size_t)n * hw * sizeof(int), st));
    k_adj<<<gp, 256, 0, st>>>(c.labels.p, W, H, v0, s.parent.p, s.orphan_idx.p, s.adj_cnt.p, nullptr, nullptr,
                              nullptr);
    LFDG_LAUNCHED(&c);
    // per-view orphan counts live at tile_off[b*(n_tiles+1) + n_tiles]
    s.lcnt.alloc((size_t)n);
    k_gather_counts<<<ceil_div(n, 128), 128, 0, st>>>(s.tile_off.p, n_tiles, n, s.lcnt.p);
    LFDG_LAUNCHED(&c);
    k_scan_rows<<<n, 1024, 0, st>>>(s.adj_cnt.p, hw, s.adj_off.p, hw + 1, 0, s.lcnt.p);
    LFDG_LAUNCHED(&c);
    k_adj<<<gp, 256, 0, st>>>(c.labels.p, W, H, v0, s.parent.p, s.orphan_idx.p, s.adj_cnt.p, s.adj_off.p,
                              s.adj_cur.p, s.adj.p);
    LFDG_LAUNCHED(&c);
    s.g_count.alloc((size_t)n * nsp);
    s.g_merged.alloc((size_t)n * hw);
    s.g_assigned.alloc((size_t)n * hw);
    int smem_cap = 0;
    LFDG_CUDA_CHECK(cudaDeviceGetAttribute(&smem_cap, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
    smem_cap = std::min(smem_cap, 200 * 1024);
    LFDG_CUDA_CHECK(cudaFuncSetAttribute(k_orphan_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap));
    k_orphan_merge<<<n, 32, smem_cap, st>>>(c.labels.p, W, H, nsp, v0, s.parent.p, s.csize.p, s.keeper.p,
                                            s.orphan_list.p, s.tile_off.p, n_tiles, s.adj_off.p, s.adj.p,
                                            s.g_count.p, s.g_merged.p, s.g_assigned.p, smem_cap);
    LFDG_LAUNCHED(&c);
    k_relabel<<<gp, 256, 0, st>>>(c.labels.p, W, H, v0, s.parent.p, s.orphan_idx.p, s.g_merged.p);
    LFDG_LAUNCHED(&c);

    // ---- empty-cluster repair
    s.lcnt.alloc((size_t)n * nsp);
    LFDG_CUDA_CHECK(cudaMemsetAsync(s.lcnt.p, 0, (size_t)n * nsp * sizeof(int), st));
    k_label_hist<<<gp, 256, 0, st>>>(c.labels.p, W, H, nsp, v0, s.lcnt.p);
    LFDG_LAUNCHED(&c);
    s.queue.alloc((size_t)n * hw);
    s.seen.alloc((size_t)n * hw);
    LFDG_CUDA_CHECK(cudaMemsetAsync(s.seen.p, 0, (size_t)n * hw * sizeof(int), st));
    k_empty_repair<<<n, 32, 0, st>>>(c.labels.p, W, H, S, gw, gh, v0, s.lcnt.p, s.queue.p, s.seen.p);
    LFDG_LAUNCHED(&c);

    recompute_stats(c, v0, n);
    for (int b = 0; b < n; ++b) c.grid_ready[v0 + b] = 1;
}

void grid_from_labels(Ctx& c, int v, int S, const int32_t* host_labels) {
    c.require_view(v);
    if (S < 1) throw Error(LFDG_INVALID_PARAMS, "cell size must be >= 1");
    const int gw = (c.W + S - 1) / S, gh = (c.H + S - 1) / S;
    const size_t hw = c.hw();
    for (size_t i = 0; i < hw; ++i)
        if (host_labels[i] < 0 || host_labels[i] >= gw * gh)
            throw Error(LFDG_INVALID_PARAMS, "label map does not fit the configured grid");
    ensure_grid_buffers(c, S);
    LFDG_CUDA_CHECK(cudaMemcpyAsync(c.labels.p + (size_t)v * hw, host_labels, hw * sizeof(int32_t),
                                    cudaMemcpyHostToDevice, c.stream));
    recompute_stats(c, v, 1);
    LFDG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    c.grid_ready[v] = 1;
}

}  // namespace lfdg
