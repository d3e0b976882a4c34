/* lfd_oracle.h — plain-C restatement of the reference's hot path (TEST INFRASTRUCTURE ONLY).
 *
 * An independent CPU restatement of proj/include/lfd/{superpixel,sweep,refine,geometry,image,rng}.hpp
 * in C11, used by tests/ as a second checker beside oracle/_ref (the reference itself).  It is
 * pinned against the reference: tests/test_oracle_restatement.py requires bit-identical outputs
 * to oracle/_ref and to the frozen golden vectors in tests/golden/.  Single-threaded, scalar
 * ("port" kind in bench.py's vocabulary).  Layouts match include/lfdg.h.
 */
#ifndef LFD_ORACLE_H
#define LFD_ORACLE_H
#include <stdint.h>

typedef struct {
    double cx, cy;
    float color[3];
    int32_t count, gx, gy;
} lfdo_record; /* SuperpixelRecord (superpixel.hpp:30) */

typedef struct {
    int W, H, S, gw, gh;
    int32_t* labels;     /* [H*W]   */
    lfdo_record* rec;    /* [nsp]   */
    int32_t* off;        /* [nsp+1] */
    int32_t* mem;        /* [H*W]   */
} lfdo_grid;             /* SuperpixelGrid (superpixel.hpp:39), caller-owned buffers */

typedef struct {
    double sigma;
    float alpha, eta;
    int size_init, steps_init, iterations, max_neighbors;
    int use_smoothness, use_consistency, use_occlusion;
} lfdo_energy; /* EnergyParams (refine.hpp:15), sigma / size_init already resolved */

/* slic_segment (superpixel.hpp:179) on one [H][W][3] image; fills g (g->labels etc. allocated
 * by the caller with the sizes above).  Returns 0, or 1 on invalid parameters. */
int lfdo_slic_segment(int W, int H, const float* img, int S, float compactness, int iterations, lfdo_grid* g);

/* sweep_view (sweep.hpp:112) for `view` of a V-view set: images [V][H][W][3], cams [V][21]
 * (K, R row-major, t); planes_out [nsp][4]. */
int lfdo_sweep_view(int V, const float* images, const double* cams, double d_min, double d_max, const lfdo_grid* grids,
                    int view, int levels, float threshold, int max_neighbors, uint64_t seed, double* planes_out);

/* rasterize (sweep.hpp:44) of one view: planes [nsp][4] -> depth [H*W]. */
void lfdo_rasterize(const double* cam, const lfdo_grid* g, const double* planes, float* depth_out);

/* refine_iteration (refine.hpp:253) over every (view, sp): planes_all [V][nsp][4] and depth_all
 * [V][H*W] are the snapshot; planes_out [V][nsp][4]; accepted may be NULL. */
int lfdo_refine_iteration(int V, const double* cams, double d_min, double d_max, const lfdo_grid* grids,
                          const lfdo_energy* p, const double* planes_all, const float* depth_all, int l,
                          double* planes_out, uint64_t* accepted);

#endif
