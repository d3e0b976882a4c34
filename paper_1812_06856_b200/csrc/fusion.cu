// Stability-based fusion on sm_100a: gather_candidates + stability_fuse + fuse_all
// (fusion.hpp:31-100) — SURVEY.md §8(f) "next" row 1.
//
//   k_fuse_project   one thread per (source view, source pixel): plane-free reprojection of the
//                    source depth into the reference view (fusion.hpp:44-53, Eigen order, FP64,
//                    glibc lround semantics); pass 1 counts candidates per reference pixel,
//                    pass 2 fills them (atomic cursor) with their (source view, source pixel) key
//   k_fuse_sort      per reference pixel, order the list by key = the reference's scan order
//                    (only needed when the lists themselves are returned, gather_candidates)
//   k_fuse_stability one thread per reference pixel: O(k^2) stability counting in inverse depth,
//                    winner = min (depth, source view) with stability >= 0 (fusion.hpp:65-92)
//
// The fused value of a pixel is a function of the candidate multiset only (integer counts and a
// total-order minimum), so the unordered fill gives the reference's result bit for bit.
#include <algorithm>
#include <vector>

#include "context.h"

namespace lfdg {
namespace {

struct FuseXf {  // R = R_ref R_src^T, t = t_ref - R t_src (fusion.hpp:42-43), per source view
    double R[9];
    double t[3];
};

__device__ __forceinline__ int lround_to_int(double x) {
    long long r = fabs(x) < 0x1p63 ? llround(x) : (long long)0x8000000000000000ull;
    return (int)(unsigned)(unsigned long long)r;
}

// Returns the reference pixel index (or -1) and the candidate depth.
__device__ __forceinline__ int fuse_project(const Cam& src, const Cam& ref, const FuseXf& xf, int W, int H, int x, int y,
                                            float d, float& zout) {
    if (!(d > 0)) return -1;  // fusion.hpp:47
    double rx, ry;
    cam_ray(src, (double)x, (double)y, rx, ry);
    const double a0 = (double)d * rx, a1 = (double)d * ry, a2 = (double)d;
    const double x0 = ((xf.R[0] * a0 + xf.R[1] * a1) + xf.R[2] * a2) + xf.t[0];
    const double x1 = ((xf.R[3] * a0 + xf.R[4] * a1) + xf.R[5] * a2) + xf.t[1];
    const double x2 = ((xf.R[6] * a0 + xf.R[7] * a1) + xf.R[8] * a2) + xf.t[2];
    if (x2 <= 0) return -1;
    const double h0 = (ref.K[0] * x0 + ref.K[1] * x1) + ref.K[2] * x2;
    const double h1 = (ref.K[3] * x0 + ref.K[4] * x1) + ref.K[5] * x2;
    const double h2 = (ref.K[6] * x0 + ref.K[7] * x1) + ref.K[8] * x2;
    const int px = lround_to_int(h0 / h2);
    const int py = lround_to_int(h1 / h2);
    if (px < 0 || py < 0 || px >= W || py >= H) return -1;
    zout = (float)x2;
    return py * W + px;
}

__global__ void k_fuse_project(const float* __restrict__ depth, const Cam* __restrict__ cams, const FuseXf* xf,
                               int W, int H, int ref_view, int* counts, const int* offsets, int* cursor, float* cdep,
                               long long* ckey) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const int s = blockIdx.y;
    const int x = (int)(i % W), y = (int)(i / W);
    float z;
    const int q = fuse_project(cams[s], cams[ref_view], xf[s], W, H, x, y, depth[(size_t)s * hw + i], z);
    if (q < 0) return;
    if (!cdep) {
        atomicAdd(&counts[q], 1);
        return;
    }
    const int pos = offsets[q] + atomicAdd(&cursor[q], 1);
    cdep[pos] = z;
    ckey[pos] = ((long long)s << 32) | (long long)i;
}

// Insertion-sort each pixel's list by key (the reference's (source view, pixel) scan order).
__global__ void k_fuse_sort(int npx, const int* __restrict__ offsets, float* cdep, long long* ckey) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npx) return;
    const int a = offsets[p], b = offsets[p + 1];
    for (int k = a + 1; k < b; ++k) {
        const long long key = ckey[k];
        const float d = cdep[k];
        int j = k - 1;
        while (j >= a && ckey[j] > key) {
            ckey[j + 1] = ckey[j];
            cdep[j + 1] = cdep[j];
            --j;
        }
        ckey[j + 1] = key;
        cdep[j + 1] = d;
    }
}

// stability_fuse (fusion.hpp:65-92) over CSR lists; view of a candidate = key >> 32.
__global__ void k_fuse_stability(int npx, const int* __restrict__ offsets, const float* __restrict__ cdep,
                                 const long long* __restrict__ ckey, const int* __restrict__ cview, double eps,
                                 float* out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npx) return;
    const int a = offsets[p], b = offsets[p + 1];
    float best_depth = 0.f;
    int best_view = 0;
    bool found = false;
    for (int c = a; c < b; ++c) {
        const float dc = cdep[c];
        const double inv_c = 1.0 / (double)dc;
        int stability = 0;
        for (int j = a; j < b; ++j) {
            if (j == c) continue;
            stability += fabs(1.0 / (double)cdep[j] - inv_c) <= eps ? 1 : -1;
        }
        if (stability < 0) continue;
        const int vc = ckey ? (int)(ckey[c] >> 32) : cview[c];
        if (!found || dc < best_depth || (dc == best_depth && vc < best_view)) {
            best_depth = dc;
            best_view = vc;
            found = true;
        }
    }
    out[p] = found ? best_depth : 0.f;
}

// Exclusive scan of n ints (single block, sequential segments), out[n] = total.
__global__ void __launch_bounds__(1024) k_scan1(const int* in, int* out, int n) {
    __shared__ int sums[1024];
    const int per = (n + 1023) / 1024;
    const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
    int s = 0;
    for (int k = lo; k < hi; ++k) s += in[k];
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
        const int t = in[k];
        out[k] = acc;
        acc += t;
    }
    if (threadIdx.x == 1023) out[n] = sums[1023];
}

inline unsigned ceil_div(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }

// Host transforms in Eigen's order (fusion.hpp:42-43).
std::vector<FuseXf> fuse_transforms(const Ctx& c, int ref) {
    std::vector<FuseXf> out(c.V);
    const lfdg_camera& cr = c.cams[ref];
    for (int s = 0; s < c.V; ++s) {
        const lfdg_camera& cs = c.cams[s];
        FuseXf& x = out[s];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                x.R[a * 3 + b] = (cr.R[a * 3 + 0] * cs.R[b * 3 + 0] + cr.R[a * 3 + 1] * cs.R[b * 3 + 1]) +
                                 cr.R[a * 3 + 2] * cs.R[b * 3 + 2];
        for (int a = 0; a < 3; ++a)
            x.t[a] = cr.t[a] - ((x.R[a * 3 + 0] * cs.t[0] + x.R[a * 3 + 1] * cs.t[1]) + x.R[a * 3 + 2] * cs.t[2]);
    }
    return out;
}

// Candidate lists of reference view `ref` from every view's depth raster; returns the total.
long long build_candidates(Ctx& c, int ref, bool ordered) {
    FuseScratch& s = c.fuse_s;
    const size_t hw = c.hw();
    cudaStream_t st = c.stream;
    const std::vector<FuseXf> xf = fuse_transforms(c, ref);
    s.xf.alloc((size_t)c.V * 12);
    static_assert(sizeof(FuseXf) == 12 * sizeof(double), "FuseXf layout");
    LFDG_CUDA_CHECK(cudaMemcpyAsync(s.xf.p, xf.data(), xf.size() * sizeof(FuseXf), cudaMemcpyHostToDevice, st));
    s.counts.alloc(hw);
    s.offsets.alloc(hw + 1);
    s.cursor.alloc(hw);
    LFDG_CUDA_CHECK(cudaMemsetAsync(s.counts.p, 0, hw * sizeof(int), st));
    LFDG_CUDA_CHECK(cudaMemsetAsync(s.cursor.p, 0, hw * sizeof(int), st));
    const dim3 g(ceil_div(hw, 256), c.V);
    k_fuse_project<<<g, 256, 0, st>>>(c.depth.p, c.d_cams.p, reinterpret_cast<const FuseXf*>(s.xf.p), c.W, c.H, ref, s.counts.p, nullptr, nullptr,
                                      nullptr, nullptr);
    LFDG_LAUNCHED(&c);
    k_scan1<<<1, 1024, 0, st>>>(s.counts.p, s.offsets.p, (int)hw);
    LFDG_LAUNCHED(&c);
    int total = 0;
    LFDG_CUDA_CHECK(cudaMemcpyAsync(&total, s.offsets.p + hw, sizeof(int), cudaMemcpyDeviceToHost, st));
    LFDG_CUDA_CHECK(cudaStreamSynchronize(st));
    s.cdep.alloc(std::max(total, 1));
    s.ckey.alloc(std::max(total, 1));
    k_fuse_project<<<g, 256, 0, st>>>(c.depth.p, c.d_cams.p, reinterpret_cast<const FuseXf*>(s.xf.p), c.W, c.H, ref, nullptr, s.offsets.p, s.cursor.p,
                                      s.cdep.p, s.ckey.p);
    LFDG_LAUNCHED(&c);
    if (ordered) {
        k_fuse_sort<<<ceil_div(hw, 256), 256, 0, st>>>((int)hw, s.offsets.p, s.cdep.p, s.ckey.p);
        LFDG_LAUNCHED(&c);
    }
    return total;
}

}  // namespace

void fuse_views(Ctx& c, int v0, int n, double eps) {
    if (eps <= 0) throw Error(LFDG_INVARIANT, "fusion epsilon must be > 0");
    c.require_views();
    if (v0 < 0 || n < 0 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    c.fused.alloc((size_t)c.V * c.hw());
    for (int r = v0; r < v0 + n; ++r) {
        build_candidates(c, r, false);
        FuseScratch& s = c.fuse_s;
        k_fuse_stability<<<ceil_div(c.hw(), 128), 128, 0, c.stream>>>((int)c.hw(), s.offsets.p, s.cdep.p, s.ckey.p,
                                                                        nullptr, eps, c.fused.p + (size_t)r * c.hw());
        LFDG_LAUNCHED(&c);
    }
}

long long gather_candidates_host(Ctx& c, int ref, int32_t* offsets, float* depths, int32_t* views, long long capacity) {
    c.require_view(ref);
    const long long total = build_candidates(c, ref, true);
    FuseScratch& s = c.fuse_s;
    const size_t hw = c.hw();
    if (offsets)
        LFDG_CUDA_CHECK(cudaMemcpyAsync(offsets, s.offsets.p, (hw + 1) * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    if (depths && views && capacity >= total && total > 0) {
        std::vector<long long> keys(total);
        LFDG_CUDA_CHECK(cudaMemcpyAsync(depths, s.cdep.p, total * sizeof(float), cudaMemcpyDeviceToHost, c.stream));
        LFDG_CUDA_CHECK(cudaMemcpyAsync(keys.data(), s.ckey.p, total * sizeof(long long), cudaMemcpyDeviceToHost,
                                        c.stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
        for (long long k = 0; k < total; ++k) views[k] = (int32_t)(keys[k] >> 32);
    }
    LFDG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    return total;
}

// stability_fuse on caller-supplied lists (any order): offsets [npx+1], depths / views [total].
void stability_fuse_lists(int device, int npx, const int32_t* offsets, const float* depths, const int32_t* views,
                          double eps, float* out) {
    if (eps <= 0) throw Error(LFDG_INVARIANT, "fusion epsilon must be > 0");
    LFDG_CUDA_CHECK(cudaSetDevice(device));
    const long long total = offsets[npx];
    DevBuf<int> doff, dview;
    DevBuf<float> ddep, dout;
    doff.alloc(npx + 1);
    dview.alloc(std::max<long long>(total, 1));
    ddep.alloc(std::max<long long>(total, 1));
    dout.alloc(std::max(npx, 1));
    LFDG_CUDA_CHECK(cudaMemcpy(doff.p, offsets, (npx + 1) * sizeof(int), cudaMemcpyHostToDevice));
    if (total) {
        LFDG_CUDA_CHECK(cudaMemcpy(ddep.p, depths, total * sizeof(float), cudaMemcpyHostToDevice));
        LFDG_CUDA_CHECK(cudaMemcpy(dview.p, views, total * sizeof(int), cudaMemcpyHostToDevice));
    }
    if (npx) {
        k_fuse_stability<<<ceil_div(npx, 128), 128>>>(npx, doff.p, ddep.p, nullptr, dview.p, eps, dout.p);
        LFDG_CUDA_CHECK(cudaGetLastError());
        LFDG_CUDA_CHECK(cudaMemcpy(out, dout.p, npx * sizeof(float), cudaMemcpyDeviceToHost));
    }
}

}  // namespace lfdg
