// Compiles the reference's OWN acceptance suite (proj/tests/acceptance.cpp)
// against the GPU drop-in (include/lfd_gpu.hpp): every hot-path call of the suite AND of the
// reference's run_pipeline (pipeline.hpp:290/320/328/354/370-371/420, criterion 8) goes to
// lfd::gpu::*; the suite's brute-force oracles, energy ablation bookkeeping, evaluation,
// synthesis and SSIM stay the reference's CPU code.  File I/O of criterion 8 goes through the
// raw round-trip OpenCV stand-in (shim/opencv2/imgcodecs.hpp, LFD_STUB_RAW_IO).
// TEST INFRASTRUCTURE ONLY (oracle/Makefile gpu-acceptance; tests/test_gpu_acceptance.py).
#include "lfd/eval.hpp"
#include "lfd/fixtures.hpp"
#include "lfd/fusion.hpp"
#include "lfd/io.hpp"
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

#include "lfd/pipeline.hpp"  // run_pipeline's stage calls now resolve to the drop-in
#include REF_ACCEPTANCE_SOURCE
