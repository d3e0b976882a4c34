// Host-side context: device-resident copies of the reference's value types.
//
// HBM layout (all views of one context share W x H and the superpixel cell size S):
//   lab      float4 [V][H*W]   scaled-LAB image (image.hpp:83), w = 0 pad -> one 16 B load
//   labels   int32  [V][H*W]   SuperpixelGrid::label_map (superpixel.hpp:43)
//   cx, cy   f64    [V][nsp]   SuperpixelRecord centroid (superpixel.hpp:31)
//   color    float4 [V][nsp]   SuperpixelRecord::mean_color
//   count    int32  [V][nsp]   SuperpixelRecord::pixel_count
//   moff     int32  [V][nsp+1] CSR offsets of SuperpixelGrid::pixels
//   mpix     int32  [V][H*W]   CSR member pixel indices, row-major per superpixel
//   planes   f64x4  [V][nsp]   PlaneMap::planes {depth, nx, ny, nz} (sweep.hpp:28)
//   depth    f32    [V][H*W]   PlaneMap::depth (sweep.hpp:29)
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lfdg.h"
#include "common.cuh"
#include "nvtx3/nvToolsExt.h"

namespace lfdg {

// NVTX range around a C-ABI stage entry (slic, sweep, rasterize, refine, fuse, transfers), so a
// profiler timeline groups the kernels by the reference's stage names.  Header-only NVTX v3: a
// no-op unless a tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define LFDG_CUDA_CHECK(expr)                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw ::lfdg::Error(LFDG_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
    } while (0)

// Kernel launch bookkeeping: checks the launch and counts it.
#define LFDG_LAUNCHED(ctx)                          \
    do {                                            \
        LFDG_CUDA_CHECK(cudaGetLastError());        \
        (ctx)->launches++;                          \
    } while (0)

// Device allocation with optional guard zones (guard.cu).  With LFDG_GUARD=1 in the environment
// every buffer gets 64 KiB of a known byte pattern on both sides and an exact-size allocation,
// and lfdg_debug_check_guards() reports any buffer whose guards were overwritten: an
// out-of-bounds-write detector for runs where compute-sanitizer is unavailable.
bool guard_mode();
void* dev_alloc(size_t bytes);
void dev_free(void* p);

// Grow-only device buffer: re-allocation (which synchronizes the device) happens only when a
// larger size is requested, so steady-state calls never allocate.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;    // requested element count
    size_t cap = 0;  // allocated element count
    void alloc(size_t count) {
        n = count;
        if (count <= cap && p && !(guard_mode() && count != cap)) return;
        if (p) dev_free(p);
        p = nullptr;
        cap = 0;
        if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
        cap = count;
    }
    void release() {
        if (p) dev_free(p);
        p = nullptr;
        n = cap = 0;
    }
    ~DevBuf() { release(); }
};

// Static tables of make_refine_context (refine.hpp:53-79) on the device.
struct RefineTables {
    bool ready = false;
    lfdg_energy_params params{};  // sigma / size_init resolved
    int n_targets = 0;
    std::vector<int> targets_host;  // [V][n_targets]
    DevBuf<int> targets;            // [V][n_targets]
    DevBuf<double> rel;             // [V][n_targets][12]: rel_rot (9, row-major) + rel_trans (3)
    DevBuf<float> min_nb_sim;       // [V][nsp]
    DevBuf<float> ring_w;           // [V][nsp][8] color_similarity to ring neighbour k (or -1: absent)
};

// Per-context scratch (device work buffers of each stage; grow-only, reused across calls).
struct SlicScratch {
    DevBuf<double> ccx, ccy;
    DevBuf<float4> ccol;
    DevBuf<int> parent, csize, orphan_idx, orphan_list, tile_cnt, tile_off;
    DevBuf<unsigned long long> keeper;
    DevBuf<int> adj_cnt, adj_off, adj_cur, adj, g_count, g_merged;
    DevBuf<unsigned char> g_assigned;
    DevBuf<int> bbox, lcnt, moff_b, queue, seen;
    DevBuf<int> abox;  // [n][nsp][4] bbox of each cluster's pixels in the current assignment
};
struct RefineScratch {
    DevBuf<double2> mray;      // [V][H*W] member rays in CSR order
    DevBuf<int> task_counter;  // persistent-warp work counter
    DevBuf<double4> cand;      // per-warp candidate planes
    DevBuf<double> es;         // per-warp smoothness bounds
    DevBuf<int2> acc;          // per-warp accepted (previous, new) pairs, stats mode
};
struct FuseScratch {
    DevBuf<double> xf;  // [V][12] source -> reference transforms
    DevBuf<int> counts, offsets, cursor;
    DevBuf<float> cdep;
    DevBuf<long long> ckey;
};
struct StagingScratch {
    DevBuf<float> buf;           // [V][H*W*3] upload staging
    DevBuf<unsigned char> buf8;  // [V][H*W*3] 8-bit sRGB upload staging
};

// Pipelined transfers (transfer.cu): a copy stream moves the next step's views into the staging
// buffer and the previous step's results out while the compute stream works.
struct CopyPipe {
    cudaStream_t stream = nullptr;
    cudaEvent_t staged = nullptr, consumed = nullptr, computed = nullptr, downloaded = nullptr;
    int v0 = 0, n = 0;
    bool has_staged = false, has_download = false;
    void destroy() {
        for (cudaEvent_t* e : {&staged, &consumed, &computed, &downloaded})
            if (*e) cudaEventDestroy(*e), *e = nullptr;
        if (stream) cudaStreamDestroy(stream), stream = nullptr;
    }
};

struct Ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    CopyPipe pipe;
    uint64_t launches = 0;
    int sm_count = 148;

    // MultiViewSet
    int V = 0, W = 0, H = 0;
    double d_min = 0, d_max = 0;
    std::vector<lfdg_camera> cams;
    bool identity_rot = false;   // every R is exactly I
    bool canonical_k = false;    // every K has K01 = K10 = K20 = K21 = 0, K22 = 1
    DevBuf<Cam> d_cams;
    DevBuf<float4> lab;

    // SuperpixelGrid (uniform S over views)
    int S = 0, gw = 0, gh = 0, nsp = 0;
    std::vector<char> grid_ready;
    DevBuf<int32_t> labels, moff, mpix, count;
    DevBuf<double> cx, cy;
    DevBuf<float4> color;
    DevBuf<double2> cray;  // [V][nsp] ray through the centroid (geometry.hpp:45), for rasterize

    // PlaneMap
    std::vector<char> planes_ready;
    DevBuf<double4> planes, planes_next;
    DevBuf<float> depth;
    DevBuf<int> sweep_targets;  // [V][N] matching views of the last sweep
    DevBuf<unsigned char> sweep_scratch;  // per-resident-CTA hypothesis slots for L beyond shared memory
    DevBuf<float> fused;        // [V][H*W] stability-fused depth (fusion.hpp:94)
    DevBuf<int4> ras;    // [V][H*W] refine gather raster: (label word, depth, 1/depth), see refine.cu

    // refinement
    RefineTables refine;
    int refine_v0 = 0, refine_n = -1;  // -1: all views
    DevBuf<unsigned long long> counters;  // [4]: accepted, violations, pixel-evals, candidate evals

    SlicScratch slic_s;
    RefineScratch refine_s;
    FuseScratch fuse_s;
    StagingScratch stage_s;

    size_t hw() const { return static_cast<size_t>(W) * H; }
    void require_views() const {
        if (V <= 0) throw Error(LFDG_STATE, "no views: call lfdg_set_views first");
    }
    void require_view(int v) const {
        require_views();
        if (v < 0 || v >= V) throw Error(LFDG_STATE, "view index out of range");
    }
    void require_grid(int v) const {
        require_view(v);
        if (!grid_ready[v]) throw Error(LFDG_STATE, "view has no superpixel grid: segment it first");
    }
};

void set_last_error(const char* m);  // capi.cu

// ---- stage entry points (implemented in the .cu files) ----------------------------------
void ensure_grid_buffers(Ctx& c, int S);
void slic_views(Ctx& c, int v0, int n, const lfdg_slic_params& p);          // slic.cu
void grid_from_labels(Ctx& c, int v, int S, const int32_t* host_labels);     // slic.cu
void sweep_views(Ctx& c, int v0, int n, const lfdg_sweep_params& p, uint64_t seed);  // sweep.cu
void rasterize_views(Ctx& c, int v0, int n);                                   // sweep.cu
std::vector<int> matching_views(const Ctx& c, int view, int max_neighbors);    // sweep.cu
void make_refine_tables(Ctx& c, const lfdg_energy_params& p, int sweep_levels);  // refine.cu
void refine_iteration(Ctx& c, int l, bool recheck);                                         // refine.cu
void upload_images(Ctx& c, int v0, int n, const float* host);                     // transfer.cu
void upload_rgb8(Ctx& c, int v0, int n, const unsigned char* host);              // transfer.cu
void prefetch_images(Ctx& c, int v0, int n, const float* host);                  // transfer.cu
void commit_images(Ctx& c);                                                       // transfer.cu
void download_results_async(Ctx& c, int v0, int n, lfdg_plane* planes, float* depth);  // transfer.cu
void wait_downloads(Ctx& c);                                                      // transfer.cu
void fuse_views(Ctx& c, int v0, int n, double eps);                                // fusion.cu
long long gather_candidates_host(Ctx& c, int ref, int32_t* offsets, float* depths, int32_t* views,
                                 long long capacity);                              // fusion.cu
void stability_fuse_lists(int device, int npx, const int32_t* offsets, const float* depths, const int32_t* views,
                          double eps, float* out);                                 // fusion.cu
void download_results(Ctx& c, int v0, int n, lfdg_plane* planes, float* depth);   // transfer.cu

}  // namespace lfdg
