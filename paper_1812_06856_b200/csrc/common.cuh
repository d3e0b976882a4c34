// Shared device helpers for the sm_100a hot path.
//
// Bit-exactness contract: every FP expression below is written in the
// reference's operation order (Eigen fixed-size order: (t0 + t1) + t2)
// and the whole library is compiled with --fmad=false, so no multiply-add is contracted.
// Divisions and square roots are IEEE round-to-nearest (never --use_fast_math).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lfdg.h"

#define LFDG_FULL_MASK 0xffffffffu

namespace lfdg {

// PinholeCamera (geometry.hpp:22), row-major K, R and t.
struct Cam {
    double K[9];
    double R[9];
    double t[3];
};

// PinholeCamera::ray (geometry.hpp:45-50): closed-form K^-1 with K(2,2) == 1, z = 1.
__device__ __forceinline__ void cam_ray(const Cam& c, double px, double py, double& rx, double& ry) {
    const double y = (py - c.K[5]) / c.K[4];
    const double x = ((px - c.K[2]) - c.K[1] * y) / c.K[0];
    rx = x;
    ry = y;
}

// Eigen dot of two 3-vectors: (a0 b0 + a1 b1) + a2 b2.
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
    return (a0 * b0 + a1 * b1) + a2 * b2;
}

// splitmix64 (rng.hpp:13-18) evaluated at an explicit counter: the k-th draw (0-based) of a
// stream with initial state s0 is mix(s0 + (k + 1) * gamma), so hypothesis k is O(1).
__device__ __forceinline__ uint64_t splitmix_at(uint64_t s0, uint64_t k) {
    uint64_t z = s0 + (k + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// derive_stream (rng.hpp:31-39): initial state of the (seed, view, sp) stream.
__host__ __device__ __forceinline__ uint64_t derive_stream_state(uint64_t seed, uint64_t view, uint64_t sp) {
    uint64_t h = seed;
    h ^= (view + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2));
    h *= 0xFF51AFD7ED558CCDull;
    h ^= (sp + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2));
    h *= 0xC4CEB9FE1A85EC53ull;
    h ^= h >> 33;
    return h;
}

// RandomStream::next_double (rng.hpp:21-23).
__device__ __forceinline__ double u64_to_unit(uint64_t v) { return (double)(v >> 11) * 0x1.0p-53; }

// color_dist2 (image.hpp:13-16) in float: (d0 d0 + d1 d1) + d2 d2.
__device__ __forceinline__ float color_dist2(float a0, float a1, float a2, float b0, float b1, float b2) {
    const float d0 = a0 - b0, d1 = a1 - b1, d2 = a2 - b2;
    return (d0 * d0 + d1 * d1) + d2 * d2;
}

}  // namespace lfdg
