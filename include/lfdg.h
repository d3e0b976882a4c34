/*
 * lfdg.h — C-ABI of the B200 (sm_100a) hot path of the superpixel light-field depth estimator
 * (arXiv:1812.06856; reference: proj/include/lfd/*.hpp, a header-only C++20 CPU library).
 *
 * The reference has no FFI of its own: its hot path is the inline C++ API of
 *   proj/include/lfd/superpixel.hpp:179  slic_segment
 *   proj/include/lfd/sweep.hpp:112       sweep_view          (:141 plane_sweep_init)
 *   proj/include/lfd/sweep.hpp:44        rasterize
 *   proj/include/lfd/refine.hpp:53       make_refine_context
 *   proj/include/lfd/refine.hpp:253      refine_iteration    (:325 run_refinement)
 * and each entry point below names the one it replaces.  Everything is POD: plain pointers and
 * sizes, no C++ or torch types, caller-allocated outputs, no exceptions across the boundary.
 * Return codes map 1:1 onto the reference's exception classes (see LFDG_* below);
 * lfdg_last_error() returns the message of the last failing call on the calling thread.
 *
 * State model.  A context owns one CUDA device and the device-resident copies of the
 * reference's value types: the MultiViewSet (io.hpp:41: LAB images, cameras, DepthRange), one
 * SuperpixelGrid per view (superpixel.hpp:39), one PlaneMap (sweep.hpp:27: planes + depth
 * rasters) and, after lfdg_make_refine_context, the RefineContext tables (refine.hpp:40).
 * Calls that take host pointers copy synchronously (the reference's call semantics); calls
 * without host pointers only enqueue work on the context's stream (device-resident fast path).
 * Results are bit-identical for any `workers` value in the reference, so there is none here.
 */
#ifndef LFDG_H
#define LFDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------------------------- */
#define LFDG_OK 0
#define LFDG_INVALID_PARAMS 1 /* lfd::InvalidParams  (superpixel.hpp:14)                    */
#define LFDG_INVARIANT 2      /* lfd::InvariantError (geometry.hpp:17)                      */
#define LFDG_CUDA 3           /* CUDA runtime failure (std::runtime_error in the reference) */
#define LFDG_STATE 4          /* call-order / index error (std::out_of_range analogue)      */

/* ---- value types (layouts are part of the ABI) ---------------------------------------- */

/* PinholeCamera (geometry.hpp:22): x_cam = R*X + t, pixel = dehom(K*x_cam); row-major. */
typedef struct lfdg_camera {
    double K[9];
    double R[9];
    double t[3];
} lfdg_camera;

/* SuperpixelRecord (superpixel.hpp:30), 40 bytes. */
typedef struct lfdg_sp_record {
    double cx, cy;
    float mean_color[3];
    int32_t pixel_count;
    int32_t gx, gy;
} lfdg_sp_record;

/* SuperpixelPlane (geometry.hpp:65), 32 bytes: depth at the centroid + unit normal. */
typedef struct lfdg_plane {
    double depth;
    double normal[3];
} lfdg_plane;

/* SlicParams (superpixel.hpp:18). Defaults: 12, 0.10f, 10. */
typedef struct lfdg_slic_params {
    int size;
    float compactness;
    int iterations;
} lfdg_slic_params;

/* SweepParams (sweep.hpp:14). Defaults: 80, 0.05f, 0. */
typedef struct lfdg_sweep_params {
    int levels;
    float tssd_threshold;
    int max_neighbors;
} lfdg_sweep_params;

/* EnergyParams (refine.hpp:15). Defaults: 0, 0.075f, 0.5f, 0, 5, 5, 0, 1, 1, 1. */
typedef struct lfdg_energy_params {
    double sigma;
    float alpha;
    float eta;
    int size_init;
    int steps_init;
    int iterations;
    int max_neighbors;
    int use_smoothness;
    int use_consistency;
    int use_occlusion;
} lfdg_energy_params;

typedef struct lfdg_ctx lfdg_ctx;

/* ---- context ---------------------------------------------------------------------------- */
int lfdg_create(int device, lfdg_ctx** out);
void lfdg_destroy(lfdg_ctx* ctx);
const char* lfdg_last_error(void);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL restores
 * the context's own stream. */
int lfdg_set_stream(lfdg_ctx* ctx, void* stream);
int lfdg_synchronize(lfdg_ctx* ctx);
/* Number of kernels this context has launched so far (for the bench's gpu_launches count). */
uint64_t lfdg_launch_count(lfdg_ctx* ctx);

/* ---- MultiViewSet (io.hpp:41) ------------------------------------------------------------ */
/* images: [V][H][W][3] float scaled-LAB (image.hpp:83), host memory; cameras: [V]. Every view
 * shares W x H (io.hpp:313-315).  Validates the DepthRange (geometry.hpp:57). */
int lfdg_set_views(lfdg_ctx* ctx, int n_views, int width, int height, const float* images,
                   const lfdg_camera* cameras, double d_min, double d_max);
/* Re-upload the images of views [v0, v0+n) only (same shape as lfdg_set_views). */
int lfdg_update_images(lfdg_ctx* ctx, int v0, int n, const float* images);

/* ---- slic_segment (superpixel.hpp:179) --------------------------------------------------- */
/* Segments view `view` of the context (its LAB image) and keeps the SuperpixelGrid resident. */
int lfdg_slic_segment(lfdg_ctx* ctx, int view, const lfdg_slic_params* params);
/* Segments views [v0, v0+n) in one batched pass (same result as n calls). */
int lfdg_slic_segment_views(lfdg_ctx* ctx, int v0, int n, const lfdg_slic_params* params);
int lfdg_grid_shape(lfdg_ctx* ctx, int view, int* grid_w, int* grid_h, int* cell_size);
/* SuperpixelGrid → host: label_map [H*W], records [n], member CSR (grid.pixels) as
 * offsets [n+1] + row-major member pixel indices [H*W].  Any pointer may be NULL. */
int lfdg_get_grid(lfdg_ctx* ctx, int view, int32_t* label_map, lfdg_sp_record* records,
                  int32_t* member_offsets, int32_t* member_pixels);
/* grid_from_labels (pipeline.hpp:188): install a label map and recompute the statistics. */
int lfdg_set_grid(lfdg_ctx* ctx, int view, int cell_size, const int32_t* label_map);

/* ---- sweep_view / plane_sweep_init (sweep.hpp:112, :141) ---------------------------------- */
/* Sweeps view `view` against matching_views (sweep.hpp:67); planes stay resident as the
 * PlaneMap slot of that view; planes_out (NULL allowed) receives a host copy. */
int lfdg_sweep_view(lfdg_ctx* ctx, int view, const lfdg_sweep_params* params, uint64_t seed,
                    lfdg_plane* planes_out);
int lfdg_sweep_views(lfdg_ctx* ctx, int v0, int n, const lfdg_sweep_params* params, uint64_t seed);
/* matching_views (sweep.hpp:67): writes up to V-1 ids, returns the count in *n_out. */
int lfdg_matching_views(lfdg_ctx* ctx, int view, int max_neighbors, int* out, int* n_out);

/* ---- PlaneMap access / rasterize (sweep.hpp:27, :44) -------------------------------------- */
int lfdg_set_planes(lfdg_ctx* ctx, int view, const lfdg_plane* planes);
int lfdg_get_planes(lfdg_ctx* ctx, int view, lfdg_plane* planes);
int lfdg_rasterize(lfdg_ctx* ctx);                     /* every view, like the reference */
int lfdg_rasterize_views(lfdg_ctx* ctx, int v0, int n);
int lfdg_get_depth(lfdg_ctx* ctx, int view, float* depth);
int lfdg_set_depth(lfdg_ctx* ctx, int view, const float* depth);

/* ---- end-to-end transfers ----------------------------------------------------------------- */
/* Enqueue the upload of views [v0, v0+n) from host [n][H][W][3] scaled-LAB floats (pinned memory
 * makes it one async DMA); the images replace the context's copies. */
int lfdg_upload_images(lfdg_ctx* ctx, int v0, int n, const float* images);
/* Enqueue the upload of views [v0, v0+n) from host [n][H][W][3] sRGB floats in [0, 1] and their
 * conversion to scaled LAB on the device: rgb_to_scaled_lab (image.hpp:97-107), bit-identical to
 * the reference (glibc powf / cbrtf ports), replacing the host pre-pass of pipeline.hpp:245. */
int lfdg_upload_rgb(lfdg_ctx* ctx, int v0, int n, const float* rgb);
/* The same from 8-bit sRGB [n][H][W][3] bytes in R, G, B order (a decoded image): each channel
 * becomes byte / 255.f as read_image does (io.hpp:136-146), then rgb_to_scaled_lab; a quarter of
 * the host->device bytes of lfdg_upload_rgb. */
int lfdg_upload_rgb8(lfdg_ctx* ctx, int v0, int n, const unsigned char* rgb8);
/* Pipelined transfers for streaming many view sets through one context (a copy stream next to
 * the compute stream):
 *   prefetch_images   H2D of views [v0, v0+n) (scaled-LAB floats, pinned) into the staging
 *                     buffer on the copy stream, once the previous commit has consumed it;
 *   commit_images     on the compute stream: wait for that copy, install it as the views' LAB;
 *   download_results_async  D2H of planes / depth (as lfdg_download_results) on the copy stream,
 *                     after the compute work enqueued so far;
 *   wait_downloads    the compute stream waits for the last async download (call before the
 *                     next sweep overwrites planes / depth).
 * Step k's download and step k+1's upload then overlap the compute of steps k+1 / k.
 * lfdg_synchronize waits for both streams. */
int lfdg_prefetch_images(lfdg_ctx* ctx, int v0, int n, const float* images);
int lfdg_commit_images(lfdg_ctx* ctx);
int lfdg_download_results_async(lfdg_ctx* ctx, int v0, int n, lfdg_plane* planes, float* depth);
int lfdg_wait_downloads(lfdg_ctx* ctx);
/* Enqueue the download of planes [n][nsp] and depth [n][H][W] of views [v0, v0+n) (either may be
 * NULL); sync != 0 waits for completion. */
int lfdg_download_results(lfdg_ctx* ctx, int v0, int n, lfdg_plane* planes, float* depth, int sync);

/* ---- refinement (refine.hpp:53, :253, :325) ----------------------------------------------- */
/* make_refine_context: resolves sigma (0 → 1.5·inverse_depth_step) and size_init (0 → min(W,H))
 * exactly as refine.hpp:56-57 and builds the static tables on the device. */
int lfdg_make_refine_context(lfdg_ctx* ctx, const lfdg_energy_params* params, int sweep_levels,
                             double* sigma_out, int* size_init_out);
/* Refine only views [v0, v0+n) (the multi-GPU view partition); default is every view. */
int lfdg_set_refine_views(lfdg_ctx* ctx, int v0, int n);
/* refine_iteration(ctx, state, l): the PlaneMap planes of the refined views are replaced by the
 * Jacobi update computed from the current planes + depth rasters (the caller rasterizes, as
 * run_refinement does).  accepted/violations (NULL allowed) receive RefineStats (refine.hpp:244)
 * counters; violations is always 0 here because acceptance is strict by construction. */
int lfdg_refine_iteration(lfdg_ctx* ctx, int l, uint64_t* accepted, uint64_t* violations);
/* run_refinement: l = 1..iterations of (refine_iteration; rasterize). */
int lfdg_run_refinement(lfdg_ctx* ctx, uint64_t* accepted, uint64_t* violations);
/* Work counters accumulated by refine_iteration since the last reset: evaluated
 * (candidate, target, member pixel) triples of pair_stats and evaluated candidates. */
int lfdg_refine_work(lfdg_ctx* ctx, uint64_t* pixel_evals, uint64_t* candidate_evals, int reset);
/* Work counters of the context (out[8]): [0] accepted and [1] violations of the last
 * refine_iteration, [2] pair_stats (candidate, target, member pixel) evaluations and [3]
 * evaluated candidates since the last reset, [4] evaluations executed by idle candidate slots of
 * the refinement kernel (a speculative group with no surviving candidate), [5] sweep_cost samples
 * (hypothesis, target, member pixel) evaluated by the pruned sweep.  reset clears [2..7]. */
int lfdg_work_counters(lfdg_ctx* ctx, uint64_t* out, int reset);
/* min_neighbor_similarity table of make_refine_context (refine.hpp:71), [nsp] floats. */
int lfdg_get_min_nb_sim(lfdg_ctx* ctx, int view, float* out);

/* ---- stability fusion (fusion.hpp:31-100; SURVEY.md §8f "next" row 1) ----------------------- */
/* fuse_all for reference views [v0, v0+n): candidates are splatted from every view's current
 * depth raster, fused maps stay resident (lfdg_get_fused).  epsilon <= 0 -> LFDG_INVARIANT. */
int lfdg_fuse_views(lfdg_ctx* ctx, int v0, int n, double epsilon);
int lfdg_get_fused(lfdg_ctx* ctx, int view, float* out);
/* gather_candidates (fusion.hpp:31): CSR lists per reference pixel in the reference's
 * (source view, source pixel) order.  offsets [H*W+1] always filled; depths / views [total]
 * filled when capacity >= total (call once with NULL to size). */
int lfdg_gather_candidates(lfdg_ctx* ctx, int ref_view, int32_t* offsets, float* depths, int32_t* views,
                           int64_t capacity, int64_t* total);
/* stability_fuse (fusion.hpp:65) on caller lists: offsets [n_pixels+1], depths / views. */
int lfdg_stability_fuse(int device, int n_pixels, const int32_t* offsets, const float* depths, const int32_t* views,
                        double epsilon, float* out);

/* ---- device buffers (multi-GPU all-gather plumbing) --------------------------------------- */
/* Raw device pointer + byte size of one all-view buffer, laid out [V][per-view block]:
 * 0 labels i32[H*W], 1 centroid x f64[nsp], 2 centroid y f64[nsp], 3 mean colour f32x4[nsp],
 * 4 pixel count i32[nsp], 5 member offsets i32[nsp+1], 6 member pixels i32[H*W],
 * 7 planes f64x4[nsp], 8 depth f32[H*W], 9 centroid rays f64x2[nsp], 10 scaled LAB f32x4[H*W]
 * (L, a, b, 0).  *view_stride is the
 * per-view block size in bytes. */
int lfdg_device_buffer(lfdg_ctx* ctx, int which, void** ptr, size_t* bytes, size_t* view_stride);
/* After an external all-gather filled buffers of views this context did not compute. */
int lfdg_mark_views_ready(lfdg_ctx* ctx, int v0, int n, int what);

/* ---- synthetic scenes (fixtures.hpp restated; host code, no GPU needed) ------------------ */
/* kind: 0 cluttered_scene, 1 staircase_scene, 2 wall_scene(depth = extra), 3 slanted_scene
 * (tilt_deg = extra), 4 occluder_scene; grid_nx > 0 replaces the rig by make_grid_rig(grid_nx,
 * grid_ny, f, baseline, W, H).  V = grid_nx * grid_ny or n_views.  Outputs (NULL allowed):
 * scaled-LAB and RGB [V][H][W][3], ground-truth depth [V][H][W], cameras [V], range[2].
 * threads <= 0: all hardware threads (the result does not depend on it). */
int lfdg_render_scene(int kind, int n_views, int width, int height, double f, double baseline, double extra,
                      int grid_nx, int grid_ny, int threads, float* lab_out, float* rgb_out, float* gt_out,
                      lfdg_camera* cams_out, double* range_out);
/* The same scene rendered through n_cams caller-given cameras (replacing the rig; any calibrated
 * cameras: rotations, skew, off-plane centres).  Outputs as lfdg_render_scene, V = n_cams. */
int lfdg_render_scene_cams(int kind, int n_views, int width, int height, double f, double baseline, double extra,
                           const lfdg_camera* cams, int n_cams, int threads, float* lab_out, float* rgb_out,
                           float* gt_out, double* range_out);
/* rgb_to_scaled_lab (image.hpp:83-107) over n pixels of [n][3] floats. */
int lfdg_rgb_to_scaled_lab(int64_t n_pixels, const float* rgb, float* lab);
/* rgb_to_scaled_lab (image.hpp:97-107) on the GPU for n host pixels ([n][3] in, [n][3] out). */
int lfdg_rgb_to_scaled_lab_gpu(int device, const float* rgb, float* lab, size_t n);

/* ---- evaluation (eval.hpp; the per-view report of run_pipeline, pipeline.hpp:452-466) ------ */
/* compute_nocc_mask(gt, cams, view, inv_depth_tol) on the ground-truth depths [V][H][W]; both
 * depth maps to the disparity domain (focal, baseline > 0, + mark_disc) or to inverse depth;
 * bad_pixel_rate of est_depth [H][W] for every threshold and region: rates[3 t + r] with
 * r = 0 nocc, 1 all, 2 disc, -1 for an empty region (EmptyRegion).  mask_out [H][W] (NULL
 * allowed) receives the Region labels (0 Nocc, 1 All, 2 Disc, 3 Ignore).  Host buffers. */
int lfdg_eval_bad_pixel(int device, int n_views, int width, int height, const float* gt_depth, const lfdg_camera* cams,
                        int view, const float* est_depth, double inv_depth_tol, double focal, double baseline,
                        const double* thresholds, int n_thresholds, double* rates, unsigned char* mask_out);

/* ---- self-test ------------------------------------------------------------------------- */
/* Device ports of glibc exp / expf used by the energy (glibc_math.cuh), on caller inputs. */
int lfdg_selftest_exp(int device, const double* in, double* out, size_t n);
int lfdg_selftest_expf(int device, const float* in, float* out, size_t n);
/* The hot-loop variant of exp for non-positive arguments (identical results). */
int lfdg_selftest_exp_nonpos(int device, const double* in, double* out, size_t n);
/* Measured FP64 FMA throughput of the device (FLOP/s, DFMA = 2), the sweep/refine roofline. */
int lfdg_selftest_fp64_peak(int device, double* flops);
/* Measured FP32 FFMA throughput of the device (FLOP/s), the FP32 roofline denominator. */
int lfdg_selftest_fp32_peak(int device, double* flops);

/* ---- out-of-bounds-write detector (guard.cu) ------------------------------------------ */
/* With LFDG_GUARD=1 in the environment every device buffer is bracketed by 64 KiB guard zones
 * of a fixed byte pattern.  check_guards counts the live buffers and those whose guards were
 * overwritten (synchronizes the device).  guard_selftest writes one element past a fresh buffer
 * and sets *detected = 1 when exactly that buffer is reported (LFDG_STATE if guards are off). */
int lfdg_debug_guard_enabled(void);
int lfdg_debug_check_guards(uint64_t* n_buffers, uint64_t* n_corrupt);
int lfdg_debug_guard_selftest(int device, uint64_t* detected);

#ifdef __cplusplus
}
#endif
#endif /* LFDG_H */
