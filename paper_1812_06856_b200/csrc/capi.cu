// The C-ABI (include/lfdg.h): marshalling, validation and error mapping only.  Every
// function catches lfdg::Error / std::exception and returns the LFDG_* code that matches the
// reference's exception class; nothing throws across the boundary.
#include <cstring>
#include <string>

#include "context.h"

namespace lfdg {
thread_local std::string g_last_error;
void set_last_error(const char* m) { g_last_error = m; }
}  // namespace lfdg

namespace {
using lfdg::g_last_error;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_last_error = e.what();
        return LFDG_CUDA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LFDG_CUDA;
    }
}

lfdg::Ctx* C(lfdg_ctx* p) {
    if (!p) throw lfdg::Error(LFDG_STATE, "null context");
    return reinterpret_cast<lfdg::Ctx*>(p);
}

void activate(lfdg::Ctx* c) { LFDG_CUDA_CHECK(cudaSetDevice(c->device)); }

bool is_identity(const double* R) {
    for (int i = 0; i < 9; ++i)
        if (R[i] != ((i % 4 == 0) ? 1.0 : 0.0)) return false;
    return true;
}

}  // namespace

extern "C" {

const char* lfdg_last_error(void) { return g_last_error.c_str(); }

int lfdg_create(int device, lfdg_ctx** out) {
    return guarded([&] {
        if (!out) throw lfdg::Error(LFDG_STATE, "null output pointer");
        int n = 0;
        LFDG_CUDA_CHECK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw lfdg::Error(LFDG_CUDA, "no such CUDA device");
        LFDG_CUDA_CHECK(cudaSetDevice(device));
        auto* c = new lfdg::Ctx();
        c->device = device;
        cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete c;
            throw lfdg::Error(LFDG_CUDA, cudaGetErrorString(e));
        }
        c->stream = c->own_stream;
        cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
        c->counters.alloc(8);
        *out = reinterpret_cast<lfdg_ctx*>(c);
    });
}

void lfdg_destroy(lfdg_ctx* p) {
    if (!p) return;
    auto* c = reinterpret_cast<lfdg::Ctx*>(p);
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->pipe.stream) cudaStreamSynchronize(c->pipe.stream);
    c->pipe.destroy();
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
}

int lfdg_set_stream(lfdg_ctx* p, void* stream) {
    return guarded([&] {
        auto* c = C(p);
        c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    });
}

int lfdg_synchronize(lfdg_ctx* p) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        if (c->pipe.stream) LFDG_CUDA_CHECK(cudaStreamSynchronize(c->pipe.stream));
    });
}

uint64_t lfdg_launch_count(lfdg_ctx* p) { return p ? reinterpret_cast<lfdg::Ctx*>(p)->launches : 0; }

int lfdg_set_views(lfdg_ctx* p, int n_views, int width, int height, const float* images, const lfdg_camera* cameras,
                   double d_min, double d_max) {
    const lfdg::NvtxRange range_("set_views");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (n_views < 1 || width < 1 || height < 1) throw lfdg::Error(LFDG_INVALID_PARAMS, "invalid view set shape");
        // pixel indices are 32-bit (member CSR, gather rasters, texel offsets)
        if ((size_t)width * height >= ((size_t)1 << 31))
            throw lfdg::Error(LFDG_INVALID_PARAMS, "views of 2^31 pixels or more are not supported");
        if (!images || !cameras) throw lfdg::Error(LFDG_STATE, "null images / cameras");
        if (!(0 < d_min && d_min < d_max)) throw lfdg::Error(LFDG_INVARIANT, "depth range requires 0 < d_min < d_max");
        c->V = n_views;
        c->W = width;
        c->H = height;
        c->d_min = d_min;
        c->d_max = d_max;
        c->cams.assign(cameras, cameras + n_views);
        c->identity_rot = true;
        c->canonical_k = true;
        for (const lfdg_camera& k : c->cams) {
            c->identity_rot = c->identity_rot && is_identity(k.R);
            c->canonical_k = c->canonical_k && k.K[1] == 0.0 && k.K[3] == 0.0 && k.K[6] == 0.0 && k.K[7] == 0.0 &&
                             k.K[8] == 1.0;
        }
        const size_t hw = c->hw();
        c->lab.alloc((size_t)n_views * hw);
        c->d_cams.alloc(n_views);
        static_assert(sizeof(lfdg::Cam) == sizeof(lfdg_camera), "camera layout");
        LFDG_CUDA_CHECK(cudaMemcpyAsync(c->d_cams.p, cameras, n_views * sizeof(lfdg_camera), cudaMemcpyHostToDevice,
                                        c->stream));
        c->S = 0;
        c->labels.release();
        c->depth.release();
        c->grid_ready.assign(n_views, 0);
        c->planes_ready.assign(n_views, 0);
        c->refine.ready = false;
        c->refine_v0 = 0;
        c->refine_n = -1;
        c->depth.alloc((size_t)n_views * hw);
        LFDG_CUDA_CHECK(cudaMemsetAsync(c->depth.p, 0, (size_t)n_views * hw * sizeof(float), c->stream));
        lfdg::upload_images(*c, 0, n_views, images);
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int lfdg_update_images(lfdg_ctx* p, int v0, int n, const float* images) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        c->require_views();
        if (v0 < 0 || n < 0 || v0 + n > c->V) throw lfdg::Error(LFDG_STATE, "view range out of bounds");
        lfdg::upload_images(*c, v0, n, images);
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int lfdg_slic_segment(lfdg_ctx* p, int view, const lfdg_slic_params* params) {
    const lfdg::NvtxRange range_("slic_segment");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!params) throw lfdg::Error(LFDG_STATE, "null params");
        c->require_view(view);
        lfdg::slic_views(*c, view, 1, *params);
    });
}

int lfdg_slic_segment_views(lfdg_ctx* p, int v0, int n, const lfdg_slic_params* params) {
    const lfdg::NvtxRange range_("slic_segment_views");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!params) throw lfdg::Error(LFDG_STATE, "null params");
        lfdg::slic_views(*c, v0, n, *params);
    });
}

int lfdg_grid_shape(lfdg_ctx* p, int view, int* grid_w, int* grid_h, int* cell_size) {
    return guarded([&] {
        auto* c = C(p);
        c->require_grid(view);
        if (grid_w) *grid_w = c->gw;
        if (grid_h) *grid_h = c->gh;
        if (cell_size) *cell_size = c->S;
    });
}

int lfdg_get_grid(lfdg_ctx* p, int view, int32_t* label_map, lfdg_sp_record* records, int32_t* member_offsets,
                  int32_t* member_pixels) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        c->require_grid(view);
        const size_t hw = c->hw();
        const int nsp = c->nsp;
        cudaStream_t st = c->stream;
        if (label_map)
            LFDG_CUDA_CHECK(cudaMemcpyAsync(label_map, c->labels.p + (size_t)view * hw, hw * 4, cudaMemcpyDeviceToHost, st));
        if (member_offsets)
            LFDG_CUDA_CHECK(cudaMemcpyAsync(member_offsets, c->moff.p + (size_t)view * (nsp + 1), (nsp + 1) * 4,
                                            cudaMemcpyDeviceToHost, st));
        if (member_pixels)
            LFDG_CUDA_CHECK(cudaMemcpyAsync(member_pixels, c->mpix.p + (size_t)view * hw, hw * 4, cudaMemcpyDeviceToHost, st));
        if (records) {
            std::vector<double> cx(nsp), cy(nsp);
            std::vector<float4> col(nsp);
            std::vector<int32_t> cnt(nsp);
            LFDG_CUDA_CHECK(cudaMemcpyAsync(cx.data(), c->cx.p + (size_t)view * nsp, nsp * 8, cudaMemcpyDeviceToHost, st));
            LFDG_CUDA_CHECK(cudaMemcpyAsync(cy.data(), c->cy.p + (size_t)view * nsp, nsp * 8, cudaMemcpyDeviceToHost, st));
            LFDG_CUDA_CHECK(cudaMemcpyAsync(col.data(), c->color.p + (size_t)view * nsp, nsp * 16, cudaMemcpyDeviceToHost, st));
            LFDG_CUDA_CHECK(cudaMemcpyAsync(cnt.data(), c->count.p + (size_t)view * nsp, nsp * 4, cudaMemcpyDeviceToHost, st));
            LFDG_CUDA_CHECK(cudaStreamSynchronize(st));
            for (int id = 0; id < nsp; ++id) {
                records[id].cx = cx[id];
                records[id].cy = cy[id];
                records[id].mean_color[0] = col[id].x;
                records[id].mean_color[1] = col[id].y;
                records[id].mean_color[2] = col[id].z;
                records[id].pixel_count = cnt[id];
                records[id].gx = id % c->gw;
                records[id].gy = id / c->gw;
            }
        }
        LFDG_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

int lfdg_set_grid(lfdg_ctx* p, int view, int cell_size, const int32_t* label_map) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!label_map) throw lfdg::Error(LFDG_STATE, "null label map");
        lfdg::grid_from_labels(*c, view, cell_size, label_map);
    });
}

int lfdg_sweep_view(lfdg_ctx* p, int view, const lfdg_sweep_params* params, uint64_t seed, lfdg_plane* planes_out) {
    const lfdg::NvtxRange range_("sweep_view");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!params) throw lfdg::Error(LFDG_STATE, "null params");
        c->require_view(view);
        lfdg::sweep_views(*c, view, 1, *params, seed);
        if (planes_out) {
            LFDG_CUDA_CHECK(cudaMemcpyAsync(planes_out, c->planes.p + (size_t)view * c->nsp, c->nsp * sizeof(lfdg_plane),
                                            cudaMemcpyDeviceToHost, c->stream));
            LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        }
    });
}

int lfdg_sweep_views(lfdg_ctx* p, int v0, int n, const lfdg_sweep_params* params, uint64_t seed) {
    const lfdg::NvtxRange range_("sweep_views");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!params) throw lfdg::Error(LFDG_STATE, "null params");
        lfdg::sweep_views(*c, v0, n, *params, seed);
    });
}

int lfdg_matching_views(lfdg_ctx* p, int view, int max_neighbors, int* out, int* n_out) {
    return guarded([&] {
        auto* c = C(p);
        c->require_view(view);
        const std::vector<int> t = lfdg::matching_views(*c, view, max_neighbors);
        for (size_t i = 0; i < t.size(); ++i) out[i] = t[i];
        *n_out = static_cast<int>(t.size());
    });
}

int lfdg_set_planes(lfdg_ctx* p, int view, const lfdg_plane* planes) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        c->require_grid(view);
        LFDG_CUDA_CHECK(cudaMemcpyAsync(c->planes.p + (size_t)view * c->nsp, planes, c->nsp * sizeof(lfdg_plane),
                                        cudaMemcpyHostToDevice, c->stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        c->planes_ready[view] = 1;
    });
}

int lfdg_get_planes(lfdg_ctx* p, int view, lfdg_plane* planes) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        c->require_grid(view);
        if (!c->planes_ready[view]) throw lfdg::Error(LFDG_STATE, "view has no planes");
        LFDG_CUDA_CHECK(cudaMemcpyAsync(planes, c->planes.p + (size_t)view * c->nsp, c->nsp * sizeof(lfdg_plane),
                                        cudaMemcpyDeviceToHost, c->stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int lfdg_rasterize(lfdg_ctx* p) {
    const lfdg::NvtxRange range_("rasterize");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        c->require_views();
        lfdg::rasterize_views(*c, 0, c->V);
    });
}

int lfdg_rasterize_views(lfdg_ctx* p, int v0, int n) {
    const lfdg::NvtxRange range_("rasterize_views");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        lfdg::rasterize_views(*c, v0, n);
    });
}

int lfdg_get_depth(lfdg_ctx* p, int view, float* depth) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        c->require_view(view);
        LFDG_CUDA_CHECK(cudaMemcpyAsync(depth, c->depth.p + (size_t)view * c->hw(), c->hw() * sizeof(float),
                                        cudaMemcpyDeviceToHost, c->stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int lfdg_set_depth(lfdg_ctx* p, int view, const float* depth) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        c->require_view(view);
        LFDG_CUDA_CHECK(cudaMemcpyAsync(c->depth.p + (size_t)view * c->hw(), depth, c->hw() * sizeof(float),
                                        cudaMemcpyHostToDevice, c->stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int lfdg_make_refine_context(lfdg_ctx* p, const lfdg_energy_params* params, int sweep_levels, double* sigma_out,
                             int* size_init_out) {
    const lfdg::NvtxRange range_("make_refine_context");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!params) throw lfdg::Error(LFDG_STATE, "null params");
        lfdg::make_refine_tables(*c, *params, sweep_levels);
        if (sigma_out) *sigma_out = c->refine.params.sigma;
        if (size_init_out) *size_init_out = c->refine.params.size_init;
    });
}

int lfdg_set_refine_views(lfdg_ctx* p, int v0, int n) {
    return guarded([&] {
        auto* c = C(p);
        c->require_views();
        if (v0 < 0 || n < 0 || v0 + n > c->V) throw lfdg::Error(LFDG_STATE, "view range out of bounds");
        c->refine_v0 = v0;
        c->refine_n = n;
    });
}

int lfdg_refine_iteration(lfdg_ctx* p, int l, uint64_t* accepted, uint64_t* violations) {
    const lfdg::NvtxRange range_("refine_iteration");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!c->refine.ready) throw lfdg::Error(LFDG_STATE, "no refine context: call lfdg_make_refine_context");
        if (l < 1) throw lfdg::Error(LFDG_INVALID_PARAMS, "iteration index must be >= 1");
        LFDG_CUDA_CHECK(cudaMemsetAsync(c->counters.p, 0, 2 * sizeof(unsigned long long), c->stream));  // work counters [2..3] accumulate
        // RefineStats requested (violations != null): the reference's independent re-check of
        // every acceptance (refine.hpp:281-286) runs too
        lfdg::refine_iteration(*c, l, violations != nullptr);
        if (accepted || violations) {
            unsigned long long h[2];
            LFDG_CUDA_CHECK(cudaMemcpyAsync(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
            LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
            if (accepted) *accepted = h[0];
            if (violations) *violations = h[1];
        }
    });
}

int lfdg_run_refinement(lfdg_ctx* p, uint64_t* accepted, uint64_t* violations) {
    const lfdg::NvtxRange range_("run_refinement");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!c->refine.ready) throw lfdg::Error(LFDG_STATE, "no refine context: call lfdg_make_refine_context");
        LFDG_CUDA_CHECK(cudaMemsetAsync(c->counters.p, 0, 2 * sizeof(unsigned long long), c->stream));  // work counters [2..3] accumulate
        for (int l = 1; l <= c->refine.params.iterations; ++l) {
            lfdg::refine_iteration(*c, l, violations != nullptr);
            lfdg::rasterize_views(*c, 0, c->V);
        }
        unsigned long long h[2];
        LFDG_CUDA_CHECK(cudaMemcpyAsync(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        if (accepted) *accepted = h[0];
        if (violations) *violations = h[1];
    });
}

int lfdg_work_counters(lfdg_ctx* p, uint64_t* out, int reset) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!out) throw lfdg::Error(LFDG_STATE, "null output");
        unsigned long long h[8];
        LFDG_CUDA_CHECK(cudaMemcpyAsync(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        for (int i = 0; i < 8; ++i) out[i] = h[i];
        if (reset) LFDG_CUDA_CHECK(cudaMemsetAsync(c->counters.p + 2, 0, 6 * sizeof(unsigned long long), c->stream));
    });
}

int lfdg_refine_work(lfdg_ctx* p, uint64_t* pixel_evals, uint64_t* candidate_evals, int reset) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        unsigned long long h[4];
        LFDG_CUDA_CHECK(cudaMemcpyAsync(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        if (pixel_evals) *pixel_evals = h[2];
        if (candidate_evals) *candidate_evals = h[3];
        if (reset) LFDG_CUDA_CHECK(cudaMemsetAsync(c->counters.p + 2, 0, 2 * sizeof(unsigned long long), c->stream));
    });
}

int lfdg_get_min_nb_sim(lfdg_ctx* p, int view, float* out) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        if (!c->refine.ready) throw lfdg::Error(LFDG_STATE, "no refine context");
        c->require_view(view);
        LFDG_CUDA_CHECK(cudaMemcpyAsync(out, c->refine.min_nb_sim.p + (size_t)view * c->nsp, c->nsp * sizeof(float),
                                        cudaMemcpyDeviceToHost, c->stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int lfdg_fuse_views(lfdg_ctx* p, int v0, int n, double epsilon) {
    const lfdg::NvtxRange range_("fuse_views");
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        lfdg::fuse_views(*c, v0, n, epsilon);
    });
}

int lfdg_get_fused(lfdg_ctx* p, int view, float* out) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        c->require_view(view);
        if (!c->fused.p) throw lfdg::Error(LFDG_STATE, "no fused maps: call lfdg_fuse_views");
        LFDG_CUDA_CHECK(cudaMemcpyAsync(out, c->fused.p + (size_t)view * c->hw(), c->hw() * sizeof(float),
                                        cudaMemcpyDeviceToHost, c->stream));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    });
}

int lfdg_gather_candidates(lfdg_ctx* p, int ref_view, int32_t* offsets, float* depths, int32_t* views,
                           int64_t capacity, int64_t* total) {
    return guarded([&] {
        auto* c = C(p);
        activate(c);
        const long long t = lfdg::gather_candidates_host(*c, ref_view, offsets, depths, views, capacity);
        if (total) *total = t;
    });
}

int lfdg_stability_fuse(int device, int n_pixels, const int32_t* offsets, const float* depths, const int32_t* views,
                        double epsilon, float* out) {
    return guarded([&] { lfdg::stability_fuse_lists(device, n_pixels, offsets, depths, views, epsilon, out); });
}

int lfdg_device_buffer(lfdg_ctx* p, int which, void** ptr, size_t* bytes, size_t* view_stride) {
    return guarded([&] {
        auto* c = C(p);
        c->require_views();
        const size_t hw = c->hw();
        const size_t nsp = static_cast<size_t>(c->nsp);
        void* q = nullptr;
        size_t stride = 0;
        switch (which) {
            case 0: q = c->labels.p; stride = hw * 4; break;
            case 1: q = c->cx.p; stride = nsp * 8; break;
            case 2: q = c->cy.p; stride = nsp * 8; break;
            case 3: q = c->color.p; stride = nsp * 16; break;
            case 4: q = c->count.p; stride = nsp * 4; break;
            case 5: q = c->moff.p; stride = (nsp + 1) * 4; break;
            case 6: q = c->mpix.p; stride = hw * 4; break;
            case 7: q = c->planes.p; stride = nsp * 32; break;
            case 8: q = c->depth.p; stride = hw * 4; break;
            case 9: q = c->cray.p; stride = nsp * 16; break;
            case 10: q = c->lab.p; stride = hw * 16; break;
            default: throw lfdg::Error(LFDG_STATE, "unknown buffer id");
        }
        if (!q) throw lfdg::Error(LFDG_STATE, "buffer not allocated yet");
        *ptr = q;
        if (view_stride) *view_stride = stride;
        if (bytes) *bytes = stride * c->V;
    });
}

int lfdg_mark_views_ready(lfdg_ctx* p, int v0, int n, int what) {
    return guarded([&] {
        auto* c = C(p);
        c->require_views();
        if (v0 < 0 || n < 0 || v0 + n > c->V) throw lfdg::Error(LFDG_STATE, "view range out of bounds");
        for (int v = v0; v < v0 + n; ++v) {
            if (what & 1) c->grid_ready[v] = 1;
            if (what & 2) c->planes_ready[v] = 1;
        }
    });
}

}  // extern "C"
