// C-ABI harness around the UNMODIFIED reference headers (/root/reference/proj/include/lfd).
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/liblfdref.so with the
// Eigen/OpenCV shims under oracle/shim (Eigen3/OpenCV are not installed).
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline leg load it,
// as the checker and the reference CPU timing — never as a product path.
//
// Every function is a thin marshalling wrapper: all arithmetic is the reference's own
// (inc/superpixel.hpp slic_segment, inc/sweep.hpp sweep_view/rasterize/sweep_cost,
// inc/refine.hpp make_refine_context/refine_iteration/energy, inc/fixtures.hpp scenes,
// inc/image.hpp rgb_to_scaled_lab, inc/eval.hpp bad_pixel_rate/compute_nocc_mask).
#include <cstdint>
#include <atomic>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "lfd/eval.hpp"
#include "lfd/fixtures.hpp"
#include "lfd/fusion.hpp"
#include "lfd/pipeline.hpp"
#include "lfd/refine.hpp"
#include "lfd/sweep.hpp"

using namespace lfd;

namespace {

thread_local std::string g_err;

enum { REF_OK = 0, REF_INVALID_PARAMS = 1, REF_INVARIANT = 2, REF_OTHER = 3 };

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return REF_OK;
    } catch (const InvalidParams& e) {
        g_err = e.what();
        return REF_INVALID_PARAMS;
    } catch (const InvariantError& e) {
        g_err = e.what();
        return REF_INVARIANT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return REF_OTHER;
    }
}

struct RecordOut {  // matches include/lfdg.h lfdg_sp_record
    double cx, cy;
    float color[3];
    std::int32_t count, gx, gy;
};
static_assert(sizeof(RecordOut) == 40, "record layout");

void cam_to_array(const PinholeCamera& c, double* out) {
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) {
            out[r * 3 + k] = c.intrinsics(r, k);
            out[9 + r * 3 + k] = c.rotation(r, k);
        }
    out[18] = c.translation.x();
    out[19] = c.translation.y();
    out[20] = c.translation.z();
}

PinholeCamera cam_from_array(const double* in, int id) {
    PinholeCamera c;
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) {
            c.intrinsics(r, k) = in[r * 3 + k];
            c.rotation(r, k) = in[9 + r * 3 + k];
        }
    c.translation = Vec3(in[18], in[19], in[20]);
    c.view_id = id;
    return c;
}

SuperpixelPlane plane_from(const double* p) { return SuperpixelPlane{p[0], Vec3(p[1], p[2], p[3])}; }
void plane_to(const SuperpixelPlane& pl, double* p) {
    p[0] = pl.depth;
    p[1] = pl.normal.x();
    p[2] = pl.normal.y();
    p[3] = pl.normal.z();
}

struct Session {
    MultiViewSet mvs;
    std::vector<SuperpixelGrid> grids;
    PlaneMap state;
    std::unique_ptr<RefineContext> ctx;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Scene kinds follow inc/fixtures.hpp: 0 cluttered_scene, 1 staircase_scene, 2 wall_scene(depth=extra),
// 3 slanted_scene(tilt_deg=extra), 4 occluder_scene.  grid_nx>0 replaces the rig by
// make_grid_rig(grid_nx, grid_ny, f, baseline, W, H) (the pattern of tests/acceptance.cpp:398-399).
// Outputs: scaled-LAB images [V][H][W][3], optional RGB, GT depth [V][H][W], cameras [V][21], range[2].
int ref_render_scene(int kind, int n_views, int width, int height, double f, double baseline, double extra,
                     int grid_nx, int grid_ny, float* lab_out, float* rgb_out, float* gt_out, double* cams_out,
                     double* range_out) {
    return guarded([&] {
        SceneSpec spec;
        switch (kind) {
            case 0: spec = cluttered_scene(n_views, width, height, f, baseline); break;
            case 1: spec = staircase_scene(n_views, width, height, f, baseline); break;
            case 2: spec = wall_scene(n_views, width, height, f, baseline, extra); break;
            case 3: spec = slanted_scene(n_views, width, height, f, baseline, extra); break;
            case 4: spec = occluder_scene(n_views, width, height, f, baseline); break;
            default: throw InvalidParams("unknown scene kind");
        }
        if (grid_nx > 0) spec.cameras = make_grid_rig(grid_nx, grid_ny, f, baseline, width, height);
        const RenderedScene scene = render_scene(spec);
        const int V = scene.views.num_views();
        const std::size_t npx = static_cast<std::size_t>(width) * height;
        for (int v = 0; v < V; ++v) {
            const ImageBuffer lab = rgb_to_scaled_lab(scene.views.images[v]);
            if (lab_out) std::memcpy(lab_out + v * npx * 3, lab.data.data(), npx * 3 * sizeof(float));
            if (rgb_out) std::memcpy(rgb_out + v * npx * 3, scene.views.images[v].data.data(), npx * 3 * sizeof(float));
            if (gt_out) std::memcpy(gt_out + v * npx, scene.ground_truth[v].data.data(), npx * sizeof(float));
            if (cams_out) cam_to_array(scene.views.cameras[v], cams_out + v * 21);
        }
        if (range_out) {
            range_out[0] = spec.range.d_min;
            range_out[1] = spec.range.d_max;
        }
    });
}

int ref_rgb_to_scaled_lab(std::int64_t n_pixels, const float* rgb, float* lab) {
    return guarded([&] {
        for (std::int64_t i = 0; i < n_pixels; ++i) {
            const Color c = rgb_to_scaled_lab(Color{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]});
            lab[3 * i] = c[0];
            lab[3 * i + 1] = c[1];
            lab[3 * i + 2] = c[2];
        }
    });
}

// cams may be null: every view then gets the default PinholeCamera (identity K, R; zero t).
void* ref_session_create(int n_views, int width, int height, const float* images, const double* cams, double d_min,
                         double d_max) {
    auto* s = new Session();
    const std::size_t npx = static_cast<std::size_t>(width) * height;
    for (int v = 0; v < n_views; ++v) {
        ImageBuffer img(width, height);
        std::memcpy(img.data.data(), images + v * npx * 3, npx * 3 * sizeof(float));
        s->mvs.images.push_back(std::move(img));
        s->mvs.cameras.push_back(cams ? cam_from_array(cams + v * 21, v) : PinholeCamera{});
        s->mvs.cameras.back().view_id = v;
    }
    s->mvs.range = DepthRange{d_min, d_max};
    s->grids.resize(n_views);
    s->state.planes.resize(n_views);
    return s;
}

void ref_session_destroy(void* p) { delete static_cast<Session*>(p); }

int ref_slic(void* p, int view, int size, float compactness, int iterations, int workers) {
    auto* s = static_cast<Session*>(p);
    return guarded([&] {
        SlicParams prm;
        prm.size = size;
        prm.compactness = compactness;
        prm.iterations = iterations;
        s->grids[view] = slic_segment(s->mvs.images[view], prm, workers);
    });
}

// Rebuild a grid from a label map (pipeline.hpp:188 grid_from_labels) so GPU labels can be
// fed to the reference stages in lockstep.
int ref_set_grid_from_labels(void* p, int view, const std::int32_t* labels, int cell_size) {
    auto* s = static_cast<Session*>(p);
    return guarded([&] {
        const ImageBuffer& img = s->mvs.images[view];
        std::vector<std::int32_t> lab(labels, labels + static_cast<std::size_t>(img.width) * img.height);
        s->grids[view] = detail::grid_from_labels(img, std::move(lab), cell_size);
    });
}

void ref_grid_dims(void* p, int view, int* grid_w, int* grid_h) {
    auto* s = static_cast<Session*>(p);
    *grid_w = s->grids[view].grid_w;
    *grid_h = s->grids[view].grid_h;
}

// labels [H*W]; records [n]; offsets [n+1]; members [H*W] (CSR of grid.pixels, row-major per sp).
void ref_get_grid(void* p, int view, std::int32_t* labels, void* records, std::int32_t* offsets,
                  std::int32_t* members) {
    auto* s = static_cast<Session*>(p);
    const SuperpixelGrid& g = s->grids[view];
    if (labels) std::memcpy(labels, g.label_map.data(), g.label_map.size() * sizeof(std::int32_t));
    auto* rec = static_cast<RecordOut*>(records);
    std::int32_t off = 0;
    for (int id = 0; id < g.num_superpixels(); ++id) {
        if (rec) {
            const SuperpixelRecord& r = g.sp[id];
            rec[id] = RecordOut{r.cx, r.cy, {r.mean_color[0], r.mean_color[1], r.mean_color[2]}, r.pixel_count, r.gx, r.gy};
        }
        if (offsets) offsets[id] = off;
        if (members) std::memcpy(members + off, g.pixels[id].data(), g.pixels[id].size() * sizeof(std::int32_t));
        off += static_cast<std::int32_t>(g.pixels[id].size());
    }
    if (offsets) offsets[g.num_superpixels()] = off;
}

int ref_matching_views(void* p, int view, int max_neighbors, int* out) {
    auto* s = static_cast<Session*>(p);
    const std::vector<int> t = matching_views(s->mvs, view, max_neighbors);
    for (std::size_t i = 0; i < t.size(); ++i) out[i] = t[i];
    return static_cast<int>(t.size());
}

int ref_sweep(void* p, int view, int levels, float threshold, int max_neighbors, std::uint64_t seed, int workers,
              double* planes_out) {
    auto* s = static_cast<Session*>(p);
    return guarded([&] {
        SweepParams prm;
        prm.levels = levels;
        prm.tssd_threshold = threshold;
        prm.max_neighbors = max_neighbors;
        s->state.planes[view] = sweep_view(s->mvs, s->grids, view, prm, seed, workers);
        if (planes_out)
            for (std::size_t i = 0; i < s->state.planes[view].size(); ++i)
                plane_to(s->state.planes[view][i], planes_out + 4 * i);
    });
}

double ref_sweep_cost(void* p, int view, int sp, double depth, const int* targets, int n_targets, float threshold) {
    auto* s = static_cast<Session*>(p);
    return sweep_cost(s->mvs, s->grids, view, sp, depth, std::vector<int>(targets, targets + n_targets), threshold);
}

void ref_set_planes(void* p, int view, const double* planes) {
    auto* s = static_cast<Session*>(p);
    const int n = s->grids[view].num_superpixels();
    s->state.planes[view].resize(n);
    for (int i = 0; i < n; ++i) s->state.planes[view][i] = plane_from(planes + 4 * i);
}

void ref_get_planes(void* p, int view, double* planes) {
    auto* s = static_cast<Session*>(p);
    for (std::size_t i = 0; i < s->state.planes[view].size(); ++i) plane_to(s->state.planes[view][i], planes + 4 * i);
}

void ref_rasterize(void* p) {
    auto* s = static_cast<Session*>(p);
    rasterize(s->mvs, s->grids, s->state);
}

void ref_get_depth(void* p, int view, float* out) {
    auto* s = static_cast<Session*>(p);
    std::memcpy(out, s->state.depth[view].data.data(), s->state.depth[view].data.size() * sizeof(float));
}

void ref_set_depth(void* p, int view, const float* in) {
    auto* s = static_cast<Session*>(p);
    s->state.depth.resize(s->mvs.num_views());
    const int w = s->mvs.width(), h = s->mvs.height();
    s->state.depth[view] = DepthMap(w, h, 0.f);
    std::memcpy(s->state.depth[view].data.data(), in, static_cast<std::size_t>(w) * h * sizeof(float));
}

// make_refine_context (refine.hpp:53).  Returns the resolved sigma / size_init through the pointers.
int ref_refine_context(void* p, double sigma, float alpha, float eta, int size_init, int steps_init, int iterations,
                       int max_neighbors, int use_smoothness, int use_consistency, int use_occlusion,
                       int sweep_levels, double* sigma_out, int* size_init_out) {
    auto* s = static_cast<Session*>(p);
    return guarded([&] {
        EnergyParams prm;
        prm.sigma = sigma;
        prm.alpha = alpha;
        prm.eta = eta;
        prm.size_init = size_init;
        prm.steps_init = steps_init;
        prm.iterations = iterations;
        prm.max_neighbors = max_neighbors;
        prm.use_smoothness = use_smoothness != 0;
        prm.use_consistency = use_consistency != 0;
        prm.use_occlusion = use_occlusion != 0;
        s->ctx = std::make_unique<RefineContext>(make_refine_context(s->mvs, s->grids, prm, sweep_levels));
        if (sigma_out) *sigma_out = s->ctx->params.sigma;
        if (size_init_out) *size_init_out = s->ctx->params.size_init;
    });
}

void ref_min_nb_sim(void* p, int view, float* out) {
    auto* s = static_cast<Session*>(p);
    const auto& m = s->ctx->min_nb_sim[view];
    std::memcpy(out, m.data(), m.size() * sizeof(float));
}

// state.planes <- refine_iteration(ctx, state, l) (refine.hpp:253); depth rasters are NOT
// recomputed (the caller runs ref_rasterize, exactly as run_refinement does).
int ref_refine_iteration(void* p, int l, int workers, int with_stats, std::uint64_t* accepted,
                         std::uint64_t* violations) {
    auto* s = static_cast<Session*>(p);
    return guarded([&] {
        RefineStats stats;
        PlaneMap next = refine_iteration(*s->ctx, s->state, l, workers, with_stats ? &stats : nullptr);
        s->state.planes = std::move(next.planes);
        if (accepted) *accepted = stats.accepted.load();
        if (violations) *violations = stats.violations.load();
    });
}

double ref_energy(void* p, int view, int sp, const double* plane) {
    auto* s = static_cast<Session*>(p);
    return energy(*s->ctx, view, sp, plane_from(plane), s->state);
}

double ref_smoothness_term(void* p, int view, int sp, const double* plane) {
    auto* s = static_cast<Session*>(p);
    return smoothness_term(*s->ctx, view, sp, plane_from(plane), s->state);
}

double ref_consistency_term(void* p, int view, int sp, const double* plane) {
    auto* s = static_cast<Session*>(p);
    return consistency_term(*s->ctx, view, sp, plane_from(plane), s->state);
}

// pair_stats (refine.hpp:111): out = {photo, visibility, occlusion, x_count, y_nonempty}.
void ref_pair_stats(void* p, int view, int sp, const double* plane, int target, double* out) {
    auto* s = static_cast<Session*>(p);
    const ViewPairStats st = pair_stats(*s->ctx, view, sp, plane_from(plane), target, s->state);
    out[0] = st.photo;
    out[1] = st.visibility;
    out[2] = st.occlusion;
    out[3] = st.x_count;
    out[4] = st.y_nonempty ? 1.0 : 0.0;
}

int ref_normal_candidates(void* p, int view, int sp, double* out) {
    auto* s = static_cast<Session*>(p);
    const auto n = normal_candidates(*s->ctx, view, sp, s->state);
    for (std::size_t i = 0; i < n.size(); ++i) {
        out[3 * i] = n[i].x();
        out[3 * i + 1] = n[i].y();
        out[3 * i + 2] = n[i].z();
    }
    return static_cast<int>(n.size());
}

int ref_grid_neighbors(void* p, int view, int sp, int kernel, int size_px, int step_sp, int* out) {
    auto* s = static_cast<Session*>(p);
    const auto nb = grid_neighbors(s->grids[view], sp, kernel ? NeighborPattern::Kernel : NeighborPattern::Immediate8,
                                   size_px, step_sp);
    for (std::size_t i = 0; i < nb.size(); ++i) out[i] = nb[i];
    return static_cast<int>(nb.size());
}

// Bad-pixel rate (eval.hpp:45) of `est` against `gt` for one view, in the reference's
// pipeline convention (pipeline.hpp:452-466): nocc mask from all GT maps at 2*step, and the
// disparity domain with focal*baseline when both are > 0, else inverse depth.
// region: 0 nocc, 1 all, 2 disc.  Returns -1 for an empty region.
double ref_bad_pixel_rate(int n_views, int width, int height, const float* gt_all, const double* cams, int view,
                          const float* est, double inv_depth_tol, double focal, double baseline, int region,
                          double threshold) {
    std::vector<DepthMap> gts;
    std::vector<PinholeCamera> cameras;
    const std::size_t npx = static_cast<std::size_t>(width) * height;
    for (int v = 0; v < n_views; ++v) {
        DepthMap d(width, height);
        std::memcpy(d.data.data(), gt_all + v * npx, npx * sizeof(float));
        gts.push_back(std::move(d));
        cameras.push_back(cam_from_array(cams + v * 21, v));
    }
    EvalMask mask = compute_nocc_mask(gts, cameras, view, inv_depth_tol);
    DepthMap e(width, height);
    std::memcpy(e.data.data(), est, npx * sizeof(float));
    DepthMap g = gts[view];
    const bool disp = focal > 0 && baseline > 0;
    e = depth_to_disparity(e, disp ? focal : 1.0, disp ? baseline : 1.0);
    g = depth_to_disparity(g, disp ? focal : 1.0, disp ? baseline : 1.0);
    if (disp) mark_disc(mask, g);
    const Region r = region == 0 ? Region::Nocc : region == 1 ? Region::All : Region::Disc;
    try {
        return bad_pixel_rate(e, g, mask, r, threshold);
    } catch (const EmptyRegion&) {
        return -1.0;
    }
}


// fuse_all (fusion.hpp:94) of the session's current depth rasters -> out [V][H*W].
int ref_fuse_all(void* p, double epsilon, int workers, float* out) {
    auto* s = static_cast<Session*>(p);
    return guarded([&] {
        const std::vector<DepthMap> fused = fuse_all(s->state.depth, s->mvs.cameras, epsilon, workers);
        const std::size_t npx = static_cast<std::size_t>(s->mvs.width()) * s->mvs.height();
        for (std::size_t v = 0; v < fused.size(); ++v) std::memcpy(out + v * npx, fused[v].data.data(), npx * 4);
    });
}

// gather_candidates (fusion.hpp:31) as CSR; depths / views filled when capacity >= total.
int ref_gather_candidates(void* p, int ref, std::int32_t* offsets, float* depths, std::int32_t* views,
                          std::int64_t capacity, std::int64_t* total) {
    auto* s = static_cast<Session*>(p);
    return guarded([&] {
        const CandidateRaster cr = gather_candidates(ref, s->state.depth, s->mvs.cameras);
        std::int64_t k = 0;
        for (std::size_t i = 0; i < cr.lists.size(); ++i) {
            offsets[i] = static_cast<std::int32_t>(k);
            k += static_cast<std::int64_t>(cr.lists[i].size());
        }
        offsets[cr.lists.size()] = static_cast<std::int32_t>(k);
        *total = k;
        if (!depths || !views || capacity < k) return;
        k = 0;
        for (const auto& l : cr.lists)
            for (const auto& c : l) {
                depths[k] = c.depth;
                views[k] = c.source_view;
                ++k;
            }
    });
}

// ---- bounded samples of the reference's per-task loop bodies (bench.py reference arm) -----
//
// sweep_view's task body (sweep.hpp:119-137) for a list of superpixels, parallel over
// `workers` with the reference's own parallel_for; planes_out receives the winners.
int ref_sweep_sample(void* p, int view, const int* sps, int n, int levels, float threshold, int max_neighbors,
                     std::uint64_t seed, int workers, double* planes_out) {
    auto* s = static_cast<Session*>(p);
    return guarded([&] {
        SweepParams prm;
        prm.levels = levels;
        prm.tssd_threshold = threshold;
        prm.max_neighbors = max_neighbors;
        prm.validate();
        const std::vector<int> targets = matching_views(s->mvs, view, prm.max_neighbors);
        parallel_for(static_cast<std::size_t>(n), workers, [&](std::size_t task) {
            const std::int32_t sp = sps[task];
            RandomStream rng = derive_stream(seed, static_cast<std::uint64_t>(view), static_cast<std::uint64_t>(sp));
            const std::vector<double> depths = sample_inverse_depths(s->mvs.range, prm.levels, rng);
            double best_cost = 0, best_depth = 0;
            bool first = true;
            for (auto it = depths.rbegin(); it != depths.rend(); ++it) {
                const double c = sweep_cost(s->mvs, s->grids, view, sp, *it, targets, prm.tssd_threshold);
                if (first || c < best_cost || (c == best_cost && *it < best_depth)) {
                    best_cost = c;
                    best_depth = *it;
                    first = false;
                }
            }
            plane_to(SuperpixelPlane{best_depth, Vec3(0, 0, -1)}, planes_out + 4 * task);
        });
    });
}

// refine_iteration's task body (refine.hpp:269-320) for a list of (view, sp) tasks, built from
// the reference's public term functions exactly as the lambda composes them; parallel over
// `workers`.  Writes the new planes and the accepted count (no violation re-check, like the
// pipeline's stats-free call at pipeline.hpp:370).
int ref_refine_tasks(void* p, int l, const int* views, const int* sps, int n, int workers, double* planes_out,
                     std::uint64_t* accepted, std::uint64_t* consistency_evals, std::uint64_t* pixel_evals) {
    auto* s = static_cast<Session*>(p);
    return guarded([&] {
        const RefineContext& ctx = *s->ctx;
        const MultiViewSet& mvs = *ctx.mvs;
        const PlaneMap& state = s->state;
        const int kernel_px = static_cast<int>(ctx.params.size_init / static_cast<double>(l));
        const int kernel_step =
            std::max(1, static_cast<int>(std::lround(ctx.params.steps_init / static_cast<double>(l))));
        const double max_consistency = ctx.params.use_occlusion ? 1.0 + ctx.params.eta : 1.0;
        std::atomic<std::uint64_t> acc{0}, cev{0}, pev{0};
        parallel_for(static_cast<std::size_t>(n), workers, [&](std::size_t task) {
            const int v = views[task];
            const std::int32_t sp = sps[task];
            const SuperpixelGrid& grid = ctx.grid(v);
            const PinholeCamera& cam = mvs.cameras[v];
            const Vec2 centroid(grid.sp[sp].cx, grid.sp[sp].cy);
            SuperpixelPlane current = state.planes[v][sp];
            const std::uint64_t task_pix = grid.pixels[sp].size() * ctx.targets[v].size();
            double e_cur = energy(ctx, v, sp, current, state);
            if (ctx.params.use_consistency) {
                cev.fetch_add(1, std::memory_order_relaxed);
                pev.fetch_add(task_pix, std::memory_order_relaxed);
            }
            auto accept_if_better = [&](const SuperpixelPlane& cand, double e) {
                if (!(e > e_cur)) return;
                acc.fetch_add(1, std::memory_order_relaxed);
                current = cand;
                e_cur = e;
            };
            auto try_candidate = [&](const SuperpixelPlane& cand) {
                if (cand.depth == current.depth && cand.normal == current.normal) return;
                if (cand.depth < mvs.range.d_min || cand.depth > mvs.range.d_max) return;
                if (ctx.params.use_smoothness && ctx.params.use_consistency) {
                    const double es = smoothness_term(ctx, v, sp, cand, state);
                    if (es * max_consistency <= e_cur) return;
                    cev.fetch_add(1, std::memory_order_relaxed);
                    pev.fetch_add(task_pix, std::memory_order_relaxed);
                    accept_if_better(cand, es * consistency_term(ctx, v, sp, cand, state));
                    return;
                }
                if (ctx.params.use_consistency) {
                    cev.fetch_add(1, std::memory_order_relaxed);
                    pev.fetch_add(task_pix, std::memory_order_relaxed);
                }
                accept_if_better(cand, energy(ctx, v, sp, cand, state));
            };
            for (const std::int32_t nb : grid_neighbors(grid, sp, NeighborPattern::Kernel, kernel_px, kernel_step)) {
                const SuperpixelPlane& nb_plane = state.planes[v][nb];
                const Vec2 nb_centroid(grid.sp[nb].cx, grid.sp[nb].cy);
                const auto d = plane_depth_at(cam, nb_plane, nb_centroid, centroid);
                if (!d || *d <= 0) continue;
                try_candidate(SuperpixelPlane{*d, nb_plane.normal});
            }
            for (const Vec3& nrm : normal_candidates(ctx, v, sp, state)) try_candidate(SuperpixelPlane{current.depth, nrm});
            plane_to(current, planes_out + 4 * task);
        });
        if (accepted) *accepted = acc.load();
        if (consistency_evals) *consistency_evals = cev.load();
        if (pixel_evals) *pixel_evals = pev.load();
    });
}

// Analysis helper (not a parity path): every candidate of one refine_iteration task in the
// reference's order (refine.hpp:305-318) with its smoothness and consistency terms computed
// unconditionally from the snapshot; phase 1 = propagation, 2 = normals (at the phase-A winner's
// depth, found by the reference's greedy).  planes_out [max][4], es/ec [max]; returns the count.
int ref_task_candidates(void* p, int l, int v, int sp, int max_out, double* planes_out, double* es_out,
                        double* ec_out, int* phase_out, double* e_init) {
    auto* s = static_cast<Session*>(p);
    int count = 0;
    const int rc = guarded([&] {
        const RefineContext& ctx = *s->ctx;
        const MultiViewSet& mvs = *ctx.mvs;
        const PlaneMap& state = s->state;
        const int kernel_px = static_cast<int>(ctx.params.size_init / static_cast<double>(l));
        const int kernel_step =
            std::max(1, static_cast<int>(std::lround(ctx.params.steps_init / static_cast<double>(l))));
        const SuperpixelGrid& grid = ctx.grid(v);
        const PinholeCamera& cam = mvs.cameras[v];
        const Vec2 centroid(grid.sp[sp].cx, grid.sp[sp].cy);
        SuperpixelPlane current = state.planes[v][sp];
        double e_cur = energy(ctx, v, sp, current, state);
        *e_init = e_cur;
        auto record = [&](const SuperpixelPlane& c, int phase) {
            if (count >= max_out) return;
            plane_to(c, planes_out + 4 * count);
            es_out[count] = smoothness_term(ctx, v, sp, c, state);
            ec_out[count] = consistency_term(ctx, v, sp, c, state);
            phase_out[count] = phase;
            ++count;
        };
        auto greedy = [&](const SuperpixelPlane& c) {
            if (c.depth == current.depth && c.normal == current.normal) return;
            if (c.depth < mvs.range.d_min || c.depth > mvs.range.d_max) return;
            const double e = energy(ctx, v, sp, c, state);
            if (e > e_cur) {
                current = c;
                e_cur = e;
            }
        };
        for (const std::int32_t nb : grid_neighbors(grid, sp, NeighborPattern::Kernel, kernel_px, kernel_step)) {
            const SuperpixelPlane& nb_plane = state.planes[v][nb];
            const Vec2 nb_centroid(grid.sp[nb].cx, grid.sp[nb].cy);
            const auto d = plane_depth_at(cam, nb_plane, nb_centroid, centroid);
            if (!d || *d <= 0) continue;
            const SuperpixelPlane c{*d, nb_plane.normal};
            if (c.depth < mvs.range.d_min || c.depth > mvs.range.d_max) continue;
            record(c, 1);
            greedy(c);
        }
        for (const Vec3& nrm : normal_candidates(ctx, v, sp, state)) {
            const SuperpixelPlane c{current.depth, nrm};
            if (c.depth < mvs.range.d_min || c.depth > mvs.range.d_max) continue;
            record(c, 2);
            greedy(c);
        }
    });
    return rc == 0 ? count : -1;
}

}  // extern "C"
