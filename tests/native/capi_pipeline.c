/* The hot path driven from plain C through include/lfdg.h only (the INTEGRATION.md recipe):
 * render a scene, set the views, SLIC -> sweep -> rasterize -> make_refine_context ->
 * run_refinement, download planes and depth, and write them to the file given as argv[1]
 * (raw: planes [V][nsp] lfdg_plane, then depth [V][H][W] float) for the test to compare. */
#include <stdio.h>
#include <stdlib.h>

#include "lfdg.h"

#define CHECK(x)                                                              \
    do {                                                                      \
        int rc_ = (x);                                                        \
        if (rc_ != LFDG_OK) {                                                 \
            fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, lfdg_last_error()); \
            return 1;                                                         \
        }                                                                     \
    } while (0)

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const int V = 3, W = 160, H = 120;
    float* lab = malloc(sizeof(float) * V * W * H * 3);
    lfdg_camera cams[3];
    double range[2];
    CHECK(lfdg_render_scene(0, V, W, H, 160.0, 0.1, 0.0, 0, 0, 0, lab, NULL, NULL, cams, range));
    lfdg_ctx* ctx = NULL;
    CHECK(lfdg_create(0, &ctx));
    CHECK(lfdg_set_views(ctx, V, W, H, lab, cams, range[0], range[1]));
    lfdg_slic_params sp = {12, 0.10f, 10};
    CHECK(lfdg_slic_segment_views(ctx, 0, V, &sp));
    lfdg_sweep_params wp = {32, 0.05f, 0};
    CHECK(lfdg_sweep_views(ctx, 0, V, &wp, 0));
    CHECK(lfdg_rasterize(ctx));
    lfdg_energy_params ep = {0, 0.075f, 0.5f, 0, 5, 2, 0, 1, 1, 1};
    CHECK(lfdg_make_refine_context(ctx, &ep, 32, NULL, NULL));
    uint64_t accepted = 0, violations = 0;
    CHECK(lfdg_run_refinement(ctx, &accepted, &violations));
    int gw = 0, gh = 0, cs = 0;
    CHECK(lfdg_grid_shape(ctx, 0, &gw, &gh, &cs));
    const int nsp = gw * gh;
    lfdg_plane* planes = malloc(sizeof(lfdg_plane) * V * nsp);
    float* depth = malloc(sizeof(float) * V * W * H);
    CHECK(lfdg_download_results(ctx, 0, V, planes, depth, 1));
    /* an invalid call reports the reference's exception class */
    lfdg_slic_params bad = {0, 0.10f, 10};
    if (lfdg_slic_segment(ctx, 0, &bad) != LFDG_INVALID_PARAMS) return 3;
    lfdg_destroy(ctx);
    FILE* f = fopen(argv[1], "wb");
    if (!f) return 4;
    fwrite(planes, sizeof(lfdg_plane), (size_t)V * nsp, f);
    fwrite(depth, sizeof(float), (size_t)V * W * H, f);
    fclose(f);
    printf("nsp %d accepted %llu violations %llu\n", nsp, (unsigned long long)accepted,
           (unsigned long long)violations);
    free(lab);
    free(planes);
    free(depth);
    return 0;
}
