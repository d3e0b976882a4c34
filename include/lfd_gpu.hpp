// lfd_gpu.hpp — C++ drop-in for the reference's hot path (proj/include/lfd) on B200.
//
// Uses the reference's own value types (ImageBuffer, SlicParams, SuperpixelGrid, MultiViewSet,
// SweepParams, PlaneMap, RefineContext, RefineStats, CandidateRaster), so the reference's
// include directory (proj/include) must be on the include path.  Every
// function has the reference's signature and semantics and marshals through the C-ABI in
// lfdg.h (link with -llfdg):
//
//   lfd::gpu::slic_segment      superpixel.hpp:179
//   lfd::gpu::sweep_view        sweep.hpp:112
//   lfd::gpu::plane_sweep_init  sweep.hpp:141
//   lfd::gpu::rasterize         sweep.hpp:44
//   lfd::gpu::refine_iteration  refine.hpp:253   (takes the reference's RefineContext)
//   lfd::gpu::run_refinement    refine.hpp:325
//   lfd::gpu::gather_candidates fusion.hpp:31
//   lfd::gpu::stability_fuse    fusion.hpp:65
//   lfd::gpu::fuse_all          fusion.hpp:94
//
// Errors are rethrown as the reference's exception classes (InvalidParams, InvariantError,
// std::runtime_error).  `workers` is accepted and ignored: results are bit-identical to the
// reference for any worker count.  A maintainer switches the pipeline over with
// `namespace lfdx = lfd::gpu;` or by qualifying the calls at pipeline.hpp:290/320/328/370-371.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "lfd/fusion.hpp"
#include "lfd/refine.hpp"
#include "lfd/superpixel.hpp"
#include "lfd/sweep.hpp"
#include "lfdg.h"

namespace lfd {
namespace gpu {

namespace detail {

inline void check(int rc) {
    if (rc == LFDG_OK) return;
    const std::string msg = lfdg_last_error();
    if (rc == LFDG_INVALID_PARAMS) throw InvalidParams(msg);
    if (rc == LFDG_INVARIANT) throw InvariantError(msg);
    throw std::runtime_error("lfdg: " + msg);
}

// RAII device context holding a copy of a MultiViewSet (+ grids) on device 0.
class Context {
  public:
    Context() { check(lfdg_create(0, &ctx_)); }
    ~Context() { lfdg_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    lfdg_ctx* get() const { return ctx_; }

    void set_views(const MultiViewSet& mvs) {
        const int V = mvs.num_views();
        const int W = mvs.width(), H = mvs.height();
        std::vector<float> images(static_cast<std::size_t>(V) * W * H * 3);
        std::vector<lfdg_camera> cams(V);
        for (int v = 0; v < V; ++v) {
            std::memcpy(images.data() + static_cast<std::size_t>(v) * W * H * 3, mvs.images[v].data.data(),
                        static_cast<std::size_t>(W) * H * 3 * sizeof(float));
            cams[v] = camera(mvs.cameras[v]);
        }
        check(lfdg_set_views(ctx_, V, W, H, images.data(), cams.data(), mvs.range.d_min, mvs.range.d_max));
    }
    void set_grids(const std::vector<SuperpixelGrid>& grids) {
        for (std::size_t v = 0; v < grids.size(); ++v)
            check(lfdg_set_grid(ctx_, static_cast<int>(v), grids[v].cell_size, grids[v].label_map.data()));
    }
    void set_planes(int v, const std::vector<SuperpixelPlane>& planes) {
        std::vector<lfdg_plane> p(planes.size());
        for (std::size_t i = 0; i < planes.size(); ++i)
            p[i] = lfdg_plane{planes[i].depth, {planes[i].normal.x(), planes[i].normal.y(), planes[i].normal.z()}};
        check(lfdg_set_planes(ctx_, v, p.data()));
    }
    std::vector<SuperpixelPlane> planes(int v, int n) const {
        std::vector<lfdg_plane> p(n);
        check(lfdg_get_planes(ctx_, v, p.data()));
        std::vector<SuperpixelPlane> out(n);
        for (int i = 0; i < n; ++i) out[i] = SuperpixelPlane{p[i].depth, Vec3(p[i].normal[0], p[i].normal[1], p[i].normal[2])};
        return out;
    }
    DepthMap depth(int v, int W, int H) const {
        DepthMap d(W, H, 0.f);
        check(lfdg_get_depth(ctx_, v, d.data.data()));
        return d;
    }
    void set_depth(int v, const DepthMap& d) { check(lfdg_set_depth(ctx_, v, d.data.data())); }

    static lfdg_camera camera(const PinholeCamera& c) {
        lfdg_camera k{};
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) {
                k.K[r * 3 + q] = c.intrinsics(r, q);
                k.R[r * 3 + q] = c.rotation(r, q);
            }
        k.t[0] = c.translation.x();
        k.t[1] = c.translation.y();
        k.t[2] = c.translation.z();
        return k;
    }

  private:
    lfdg_ctx* ctx_ = nullptr;
};

inline SuperpixelGrid grid_from_device(lfdg_ctx* ctx, int view, int W, int H) {
    int gw = 0, gh = 0, s = 0;
    check(lfdg_grid_shape(ctx, view, &gw, &gh, &s));
    SuperpixelGrid g;
    g.width = W;
    g.height = H;
    g.grid_w = gw;
    g.grid_h = gh;
    g.cell_size = s;
    const int n = gw * gh;
    g.label_map.resize(static_cast<std::size_t>(W) * H);
    std::vector<lfdg_sp_record> rec(n);
    std::vector<std::int32_t> off(n + 1), mem(static_cast<std::size_t>(W) * H);
    check(lfdg_get_grid(ctx, view, g.label_map.data(), rec.data(), off.data(), mem.data()));
    g.sp.resize(n);
    g.pixels.resize(n);
    for (int id = 0; id < n; ++id) {
        SuperpixelRecord& r = g.sp[id];
        r.cx = rec[id].cx;
        r.cy = rec[id].cy;
        r.mean_color = {rec[id].mean_color[0], rec[id].mean_color[1], rec[id].mean_color[2]};
        r.pixel_count = rec[id].pixel_count;
        r.gx = rec[id].gx;
        r.gy = rec[id].gy;
        g.pixels[id].assign(mem.begin() + off[id], mem.begin() + off[id + 1]);
    }
    return g;
}

}  // namespace detail

inline SuperpixelGrid slic_segment(const ImageBuffer& image, const SlicParams& params, int workers = 1) {
    (void)workers;
    params.validate();
    if (!image.valid()) throw InvalidParams("invalid image");
    if (image.width < params.size || image.height < params.size)
        throw InvalidParams("image smaller than superpixel size");
    detail::Context c;
    MultiViewSet one;
    one.cameras = {PinholeCamera{}};
    one.images = {image};
    one.range = DepthRange{1, 2};
    c.set_views(one);
    const lfdg_slic_params p{params.size, params.compactness, params.iterations};
    detail::check(lfdg_slic_segment(c.get(), 0, &p));
    return detail::grid_from_device(c.get(), 0, image.width, image.height);
}

inline std::vector<SuperpixelPlane> sweep_view(const MultiViewSet& mvs, const std::vector<SuperpixelGrid>& grids,
                                               int view, const SweepParams& params, std::uint64_t seed,
                                               int workers = 1) {
    (void)workers;
    params.validate();
    mvs.range.validate();
    detail::Context c;
    c.set_views(mvs);
    c.set_grids(grids);
    const lfdg_sweep_params p{params.levels, params.tssd_threshold, params.max_neighbors};
    std::vector<lfdg_plane> out(grids[view].num_superpixels());
    detail::check(lfdg_sweep_view(c.get(), view, &p, seed, out.data()));
    return c.planes(view, grids[view].num_superpixels());
}

inline void rasterize(const MultiViewSet& mvs, const std::vector<SuperpixelGrid>& grids, PlaneMap& pm) {
    detail::Context c;
    c.set_views(mvs);
    c.set_grids(grids);
    for (int v = 0; v < mvs.num_views(); ++v) c.set_planes(v, pm.planes[v]);
    detail::check(lfdg_rasterize(c.get()));
    pm.depth.resize(mvs.num_views());
    for (int v = 0; v < mvs.num_views(); ++v) pm.depth[v] = c.depth(v, grids[v].width, grids[v].height);
}

inline PlaneMap plane_sweep_init(const MultiViewSet& mvs, const std::vector<SuperpixelGrid>& grids,
                                 const SweepParams& params, std::uint64_t seed, int workers = 1) {
    (void)workers;
    params.validate();
    mvs.range.validate();
    detail::Context c;
    c.set_views(mvs);
    c.set_grids(grids);
    const lfdg_sweep_params p{params.levels, params.tssd_threshold, params.max_neighbors};
    detail::check(lfdg_sweep_views(c.get(), 0, mvs.num_views(), &p, seed));
    detail::check(lfdg_rasterize(c.get()));
    PlaneMap pm;
    for (int v = 0; v < mvs.num_views(); ++v) {
        pm.planes.push_back(c.planes(v, grids[v].num_superpixels()));
        pm.depth.push_back(c.depth(v, grids[v].width, grids[v].height));
    }
    return pm;
}

// refine_iteration(ctx, state, l) with the reference's RefineContext (its mvs/grids/params).
inline PlaneMap refine_iteration(const RefineContext& ctx, const PlaneMap& state, int l, int workers = 1,
                                 RefineStats* stats = nullptr) {
    (void)workers;
    const MultiViewSet& mvs = *ctx.mvs;
    const std::vector<SuperpixelGrid>& grids = *ctx.grids;
    detail::Context c;
    c.set_views(mvs);
    c.set_grids(grids);
    for (int v = 0; v < mvs.num_views(); ++v) {
        c.set_planes(v, state.planes[v]);
        c.set_depth(v, state.depth[v]);
    }
    const EnergyParams& e = ctx.params;  // already resolved by make_refine_context
    const lfdg_energy_params p{e.sigma, e.alpha, e.eta, e.size_init, e.steps_init, e.iterations, e.max_neighbors,
                               e.use_smoothness, e.use_consistency, e.use_occlusion};
    detail::check(lfdg_make_refine_context(c.get(), &p, 2, nullptr, nullptr));
    std::uint64_t acc = 0, vio = 0;
    detail::check(lfdg_refine_iteration(c.get(), l, &acc, &vio));
    if (stats) {
        stats->accepted.fetch_add(acc);
        stats->violations.fetch_add(vio);
    }
    PlaneMap out;
    for (int v = 0; v < mvs.num_views(); ++v) out.planes.push_back(c.planes(v, grids[v].num_superpixels()));
    return out;
}

inline PlaneMap run_refinement(const RefineContext& ctx, PlaneMap state, int workers = 1,
                               RefineStats* stats = nullptr) {
    for (int l = 1; l <= ctx.params.iterations; ++l) {
        state = gpu::refine_iteration(ctx, state, l, workers, stats);
        gpu::rasterize(*ctx.mvs, *ctx.grids, state);
    }
    return state;
}

// ---- fusion (fusion.hpp) --------------------------------------------------------------
namespace detail {
// A context over depth maps + cameras only (fusion reads no images).
inline void set_depth_views(Context& c, const std::vector<DepthMap>& maps, const std::vector<PinholeCamera>& cameras) {
    const int V = static_cast<int>(maps.size());
    const int W = maps[0].width, H = maps[0].height;
    std::vector<float> images(static_cast<std::size_t>(V) * W * H * 3, 0.f);
    std::vector<lfdg_camera> cams(V);
    for (int v = 0; v < V; ++v) cams[v] = Context::camera(cameras[v]);
    check(lfdg_set_views(c.get(), V, W, H, images.data(), cams.data(), 1.0, 2.0));
    for (int v = 0; v < V; ++v) c.set_depth(v, maps[v]);
}
}  // namespace detail

inline CandidateRaster gather_candidates(int reference_view, const std::vector<DepthMap>& maps,
                                          const std::vector<PinholeCamera>& cameras) {
    detail::Context c;
    detail::set_depth_views(c, maps, cameras);
    const int W = maps[reference_view].width, H = maps[reference_view].height;
    std::vector<std::int32_t> off(static_cast<std::size_t>(W) * H + 1);
    std::int64_t total = 0;
    detail::check(lfdg_gather_candidates(c.get(), reference_view, off.data(), nullptr, nullptr, 0, &total));
    std::vector<float> dep(total > 0 ? total : 1);
    std::vector<std::int32_t> vw(total > 0 ? total : 1);
    detail::check(lfdg_gather_candidates(c.get(), reference_view, off.data(), dep.data(), vw.data(), total, &total));
    CandidateRaster cr;
    cr.width = W;
    cr.height = H;
    cr.lists.assign(static_cast<std::size_t>(W) * H, {});
    for (std::size_t i = 0; i < cr.lists.size(); ++i)
        for (std::int32_t k = off[i]; k < off[i + 1]; ++k) cr.lists[i].push_back({dep[k], vw[k]});
    return cr;
}

inline DepthMap stability_fuse(const CandidateRaster& candidates, double epsilon, int workers = 1) {
    (void)workers;
    const int npx = static_cast<int>(candidates.lists.size());
    std::vector<std::int32_t> off(npx + 1, 0);
    std::vector<float> dep;
    std::vector<std::int32_t> vw;
    for (int i = 0; i < npx; ++i) {
        for (const auto& c : candidates.lists[i]) {
            dep.push_back(c.depth);
            vw.push_back(c.source_view);
        }
        off[i + 1] = static_cast<std::int32_t>(dep.size());
    }
    DepthMap out(candidates.width, candidates.height, 0.f);
    detail::check(lfdg_stability_fuse(0, npx, off.data(), dep.data(), vw.data(), epsilon, out.data.data()));
    return out;
}

inline std::vector<DepthMap> fuse_all(const std::vector<DepthMap>& maps, const std::vector<PinholeCamera>& cameras,
                                      double epsilon, int workers = 1) {
    (void)workers;
    detail::Context c;
    detail::set_depth_views(c, maps, cameras);
    detail::check(lfdg_fuse_views(c.get(), 0, static_cast<int>(maps.size()), epsilon));
    std::vector<DepthMap> out;
    for (std::size_t v = 0; v < maps.size(); ++v) {
        DepthMap d(maps[v].width, maps[v].height, 0.f);
        detail::check(lfdg_get_fused(c.get(), static_cast<int>(v), d.data.data()));
        out.push_back(std::move(d));
    }
    return out;
}

}  // namespace gpu
}  // namespace lfd
