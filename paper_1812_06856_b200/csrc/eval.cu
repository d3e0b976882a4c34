// Evaluation against ground truth on sm_100a (eval.hpp; SURVEY.md §8(f) "next" row 3), the
// pipeline's per-view report (pipeline.hpp:452-466):
//
//   k_nocc_mask   compute_nocc_mask (eval.hpp:104-135): one thread per reference pixel lifts the
//                 ground-truth depth and tests its visibility in every other view (FP64, Eigen
//                 order, glibc lround semantics)
//   k_to_disp     depth_to_disparity (eval.hpp:61-66)
//   k_disc_edges  mark_disc's jump map (eval.hpp:76-88); k_disc_mark its radius-9 band (:89-97)
//   k_bad_counts  bad_pixel_rate (eval.hpp:45-58) for every region x threshold: integer counts
//                 (exact in any order); the host forms 100 * bad / total
//
// Region labels follow eval.hpp:15: Nocc 0, All 1, Disc 2, Ignore 3.
#include <vector>

#include "context.h"

namespace lfdg {
namespace {

constexpr unsigned char kNocc = 0, kAll = 1, kDisc = 2, kIgnore = 3;

__device__ __forceinline__ int lround_i(double x) {
    long long r = fabs(x) < 0x1p63 ? llround(x) : (long long)0x8000000000000000ull;
    return (int)(unsigned)(unsigned long long)r;
}

__global__ void k_nocc_mask(const float* __restrict__ gt, const Cam* __restrict__ cams, int V, int W, int H, int ref,
                            double tol, unsigned char* mask) {
    const size_t hw = (size_t)W * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hw) return;
    const float d = gt[(size_t)ref * hw + i];
    if (d <= 0) {
        mask[i] = kIgnore;
        return;
    }
    const Cam& rc = cams[ref];
    double rx, ry;
    cam_ray(rc, (double)(i % W), (double)(i / W), rx, ry);
    // backproject (geometry.hpp:70-73): R^T (d ray - t)
    const double a0 = (double)d * rx - rc.t[0], a1 = (double)d * ry - rc.t[1], a2 = (double)d * 1.0 - rc.t[2];
    const double w0 = (rc.R[0] * a0 + rc.R[3] * a1) + rc.R[6] * a2;
    const double w1 = (rc.R[1] * a0 + rc.R[4] * a1) + rc.R[7] * a2;
    const double w2 = (rc.R[2] * a0 + rc.R[5] * a1) + rc.R[8] * a2;
    unsigned char label = kNocc;
    for (int v = 0; v < V; ++v) {
        if (v == ref) continue;
        const Cam& c = cams[v];
        // project (geometry.hpp:76-80)
        const double c0 = ((c.R[0] * w0 + c.R[1] * w1) + c.R[2] * w2) + c.t[0];
        const double c1 = ((c.R[3] * w0 + c.R[4] * w1) + c.R[5] * w2) + c.t[1];
        const double c2 = ((c.R[6] * w0 + c.R[7] * w1) + c.R[8] * w2) + c.t[2];
        const double h0 = (c.K[0] * c0 + c.K[1] * c1) + c.K[2] * c2;
        const double h1 = (c.K[3] * c0 + c.K[4] * c1) + c.K[5] * c2;
        const double h2 = (c.K[6] * c0 + c.K[7] * c1) + c.K[8] * c2;
        const int px = lround_i(h0 / h2);
        const int py = lround_i(h1 / h2);
        bool visible = false;
        if (c2 > 0 && px >= 0 && py >= 0 && px < W && py < H) {
            const float td = gt[(size_t)v * hw + (size_t)py * W + px];
            visible = td > 0 && (1.0 / td - 1.0 / c2) <= tol;
        }
        if (!visible) {
            label = kAll;  // occluded somewhere
            break;
        }
    }
    mask[i] = label;
}

__global__ void k_to_disp(const float* __restrict__ depth, size_t n, double focal, double baseline, float* out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float d = depth[i];
    out[i] = d > 0 ? (float)(focal * baseline / d) : 0.f;
}

__global__ void k_disc_edges(const float* __restrict__ disp, int W, int H, double jump, unsigned char* edge) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)W * H) return;
    const int x = (int)(i % W), y = (int)(i / W);
    const float d = disp[i];
    edge[i] = (x + 1 < W && fabsf(disp[i + 1] - d) > jump) || (y + 1 < H && fabsf(disp[i + W] - d) > jump);
}

__global__ void k_disc_mark(const unsigned char* __restrict__ edge, int W, int H, int radius, unsigned char* mask) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)W * H) return;
    if (mask[i] == kIgnore) return;
    const int x = (int)(i % W), y = (int)(i / W);
    bool near = false;
    for (int dy = -radius; dy <= radius && !near; ++dy) {
        const int ny = y + dy;
        if (ny < 0 || ny >= H) continue;
        for (int dx = -radius; dx <= radius && !near; ++dx) {
            const int nx = x + dx;
            if (nx >= 0 && nx < W && edge[(size_t)ny * W + nx]) near = true;
        }
    }
    if (near) mask[i] = kDisc;
}

// counts[0..2] = pixels in Nocc / All / Disc; counts[3 + 3 t + r] = bad pixels at threshold t.
__global__ void k_bad_counts(const float* __restrict__ est, const float* __restrict__ truth,
                             const unsigned char* __restrict__ mask, size_t n, const double* __restrict__ thr, int nt,
                             unsigned long long* counts) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned char m = i < n ? mask[i] : kIgnore;
    // in_region (eval.hpp:33-41)
    const bool in_nocc = m == kNocc || m == kDisc, in_all = m != kIgnore, in_disc = m == kDisc;
    const bool in[3] = {in_nocc, in_all, in_disc};
    float e = 0.f, g = 0.f;
    if (i < n) {
        e = est[i];
        g = truth[i];
    }
    for (int r = 0; r < 3; ++r) {
        const unsigned b = __ballot_sync(0xffffffffu, in[r]);
        if ((threadIdx.x & 31) == 0 && b) atomicAdd(&counts[r], (unsigned long long)__popc(b));
    }
    for (int t = 0; t < nt; ++t) {
        const bool bad = !isfinite(e) || e == 0.f || fabsf(e - g) > thr[t];
        for (int r = 0; r < 3; ++r) {
            const unsigned b = __ballot_sync(0xffffffffu, in[r] && bad);
            if ((threadIdx.x & 31) == 0 && b) atomicAdd(&counts[3 + 3 * t + r], (unsigned long long)__popc(b));
        }
    }
}

inline unsigned blocks_for(size_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace
}  // namespace lfdg

extern "C" {

// The per-view evaluation of run_pipeline (pipeline.hpp:452-466) on the GPU, host buffers in.
int lfdg_eval_bad_pixel(int device, int n_views, int width, int height, const float* gt_depth, const lfdg_camera* cams,
                        int view, const float* est_depth, double inv_depth_tol, double focal, double baseline,
                        const double* thresholds, int n_thresholds, double* rates, unsigned char* mask_out) {
    using namespace lfdg;
    try {
        if (n_views < 1 || width < 2 || height < 2 || view < 0 || view >= n_views || n_thresholds < 0)
            throw Error(LFDG_INVALID_PARAMS, "bad evaluation arguments");
        LFDG_CUDA_CHECK(cudaSetDevice(device));
        const size_t hw = (size_t)width * height;
        std::vector<Cam> hc(n_views);
        for (int v = 0; v < n_views; ++v) {
            for (int k = 0; k < 9; ++k) {
                hc[v].K[k] = cams[v].K[k];
                hc[v].R[k] = cams[v].R[k];
            }
            for (int k = 0; k < 3; ++k) hc[v].t[k] = cams[v].t[k];
        }
        DevBuf<float> gt, est, gd, ed;
        DevBuf<Cam> dc;
        DevBuf<unsigned char> mask, edge;
        DevBuf<double> thr;
        DevBuf<unsigned long long> cnt;
        gt.alloc((size_t)n_views * hw);
        est.alloc(hw);
        gd.alloc(hw);
        ed.alloc(hw);
        dc.alloc(n_views);
        mask.alloc(hw);
        edge.alloc(hw);
        thr.alloc(n_thresholds > 0 ? n_thresholds : 1);
        cnt.alloc(3 + 3 * (size_t)n_thresholds);
        LFDG_CUDA_CHECK(cudaMemcpy(gt.p, gt_depth, (size_t)n_views * hw * sizeof(float), cudaMemcpyHostToDevice));
        LFDG_CUDA_CHECK(cudaMemcpy(est.p, est_depth, hw * sizeof(float), cudaMemcpyHostToDevice));
        LFDG_CUDA_CHECK(cudaMemcpy(dc.p, hc.data(), n_views * sizeof(Cam), cudaMemcpyHostToDevice));
        if (n_thresholds > 0)
            LFDG_CUDA_CHECK(cudaMemcpy(thr.p, thresholds, n_thresholds * sizeof(double), cudaMemcpyHostToDevice));
        LFDG_CUDA_CHECK(cudaMemset(cnt.p, 0, (3 + 3 * (size_t)n_thresholds) * sizeof(unsigned long long)));
        k_nocc_mask<<<blocks_for(hw), 256>>>(gt.p, dc.p, n_views, width, height, view, inv_depth_tol, mask.p);
        // disparity domain when focal and baseline are known, else inverse depth (pipeline.hpp:455-466)
        const bool disp = focal > 0 && baseline > 0;
        k_to_disp<<<blocks_for(hw), 256>>>(est.p, hw, disp ? focal : 1.0, disp ? baseline : 1.0, ed.p);
        k_to_disp<<<blocks_for(hw), 256>>>(gt.p + (size_t)view * hw, hw, disp ? focal : 1.0, disp ? baseline : 1.0,
                                           gd.p);
        if (disp) {
            k_disc_edges<<<blocks_for(hw), 256>>>(gd.p, width, height, 2.0, edge.p);
            k_disc_mark<<<blocks_for(hw), 256>>>(edge.p, width, height, 9, mask.p);
        }
        k_bad_counts<<<blocks_for(hw), 256>>>(ed.p, gd.p, mask.p, hw, thr.p, n_thresholds, cnt.p);
        LFDG_CUDA_CHECK(cudaGetLastError());
        std::vector<unsigned long long> h(3 + 3 * (size_t)n_thresholds);
        LFDG_CUDA_CHECK(cudaMemcpy(h.data(), cnt.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        if (mask_out) LFDG_CUDA_CHECK(cudaMemcpy(mask_out, mask.p, hw, cudaMemcpyDeviceToHost));
        for (int t = 0; t < n_thresholds; ++t)
            for (int r = 0; r < 3; ++r)  // EmptyRegion (eval.hpp:56) -> -1
                rates[3 * t + r] = h[r] == 0 ? -1.0 : 100.0 * (double)h[3 + 3 * t + r] / (double)h[r];
        return LFDG_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    }
}

}  // extern "C"
