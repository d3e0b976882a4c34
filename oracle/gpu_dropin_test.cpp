// Compiles one of the reference's OWN unit-test sources (proj/tests/test_*.cpp) against the GPU
// drop-in (include/lfd_gpu.hpp): the hot-path entry points the test calls are redirected to
// lfd::gpu::*, everything else (the tests' own brute-force oracles, energy terms, fixtures)
// stays the reference's CPU code.  TEST INFRASTRUCTURE ONLY (oracle/Makefile gpu-dropin-tests).
#include "lfd/fixtures.hpp"
#include "lfd/fusion.hpp"
#include "lfd/refine.hpp"
#include "lfd/superpixel.hpp"
#include "lfd/sweep.hpp"
#include "lfd_gpu.hpp"

#define slic_segment ::lfd::gpu::slic_segment
#define sweep_view ::lfd::gpu::sweep_view
#define plane_sweep_init ::lfd::gpu::plane_sweep_init
#define rasterize ::lfd::gpu::rasterize
#define refine_iteration ::lfd::gpu::refine_iteration
#define run_refinement ::lfd::gpu::run_refinement
#define gather_candidates ::lfd::gpu::gather_candidates
#define stability_fuse ::lfd::gpu::stability_fuse
#define fuse_all ::lfd::gpu::fuse_all

#include REF_TEST_SOURCE
