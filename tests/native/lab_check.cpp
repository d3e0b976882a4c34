// Host check of the glibc powf / cbrtf ports and of rgb_to_scaled_lab
// (paper_1812_06856_b200/csrc/glibc_math.cuh) against the host libm: every float the
// conversion can feed them — powf((v + 0.055f) / 1.055f, 2.4f) for every float v in
// (0.04045, 1.5] and cbrtf(t) for every float t in (216/24389, 1.5] — plus random
// and special operands, and rgb_to_scaled_lab on random colours against the same expression
// evaluated with std::pow / std::cbrt (image.hpp:70-95).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

#include "glibc_math.cuh"

static bool same(float a, float b) { return std::memcmp(&a, &b, 4) == 0 || (std::isnan(a) && std::isnan(b)); }

static float ref_srgb(float v) { return v <= 0.04045f ? v / 12.92f : std::pow((v + 0.055f) / 1.055f, 2.4f); }
static float ref_lab_f(float t) {
    constexpr float kEps = 216.f / 24389.f;
    constexpr float kKappa = 24389.f / 27.f;
    return t > kEps ? std::cbrt(t) : (kKappa * t + 16.f) / 116.f;
}

int main() {
    uint64_t bad_pow = 0, bad_cbrt = 0, bad_lab = 0, n_pow = 0, n_cbrt = 0;
    for (float v = std::nextafter(0.04045f, 2.f); v <= 1.5f; v = std::nextafter(v, 2.f)) {
        const float x = (v + 0.055f) / 1.055f;
        const float a = ::powf(x, 2.4f), c = lfdg::libm::powf_pos(x, 2.4f);
        ++n_pow;
        if (!same(a, c)) {
            if (bad_pow < 5) std::printf("powf x=%a libm=%a port=%a\n", x, a, c);
            ++bad_pow;
        }
    }
    for (float t = std::nextafter(216.f / 24389.f, 2.f); t <= 1.5f; t = std::nextafter(t, 2.f)) {
        const float a = ::cbrtf(t), c = lfdg::libm::cbrtf_(t);
        ++n_cbrt;
        if (!same(a, c)) {
            if (bad_cbrt < 5) std::printf("cbrtf t=%a libm=%a port=%a\n", t, a, c);
            ++bad_cbrt;
        }
    }
    std::mt19937_64 rng(7);
    for (int i = 0; i < 4000000; ++i) {  // random bit patterns: positive x for powf, any t for cbrtf
        const uint32_t u = static_cast<uint32_t>(rng());
        float x;
        std::memcpy(&x, &u, 4);
        if (!same(::cbrtf(x), lfdg::libm::cbrtf_(x))) {
            if (bad_cbrt < 10) std::printf("cbrtf x=%a libm=%a port=%a\n", x, ::cbrtf(x), lfdg::libm::cbrtf_(x));
            ++bad_cbrt;
        }
        const float xp = std::fabs(x);
        const float ys[] = {2.4f, 0.5f, 3.0f, -1.7f};
        const float y = ys[i & 3];
        if (xp > 0.f && !same(::powf(xp, y), lfdg::libm::powf_pos(xp, y))) {
            if (bad_pow < 10) std::printf("powf x=%a y=%a libm=%a port=%a\n", xp, y, ::powf(xp, y), lfdg::libm::powf_pos(xp, y));
            ++bad_pow;
        }
    }
    std::uniform_real_distribution<float> U(-0.1f, 1.2f);
    for (int i = 0; i < 3000000; ++i) {
        const float r0 = i % 97 == 0 ? 0.04045f : U(rng), g0 = U(rng), b0 = i % 89 == 0 ? 1.0f : U(rng);
        const float r = ref_srgb(r0), g = ref_srgb(g0), b = ref_srgb(b0);
        const float xr = (0.4124564f * r + 0.3575761f * g + 0.1804375f * b) / 0.95047f;
        const float yr = (0.2126729f * r + 0.7151522f * g + 0.0721750f * b);
        const float zr = (0.0193339f * r + 0.1191920f * g + 0.9503041f * b) / 1.08883f;
        const float fx = ref_lab_f(xr), fy = ref_lab_f(yr), fz = ref_lab_f(zr);
        const float want[3] = {(116.f * fy - 16.f) / 100.f, (500.f * (fx - fy)) / 100.f, (200.f * (fy - fz)) / 100.f};
        float got[3];
        lfdg::libm::rgb_to_scaled_lab(r0, g0, b0, got[0], got[1], got[2]);
        if (!same(got[0], want[0]) || !same(got[1], want[1]) || !same(got[2], want[2])) {
            if (bad_lab < 5) std::printf("lab rgb=(%a %a %a)\n", r0, g0, b0);
            ++bad_lab;
        }
    }
    std::printf("powf operands %llu mismatches: %llu\n", (unsigned long long)n_pow, (unsigned long long)bad_pow);
    std::printf("cbrtf operands %llu mismatches: %llu\n", (unsigned long long)n_cbrt, (unsigned long long)bad_cbrt);
    std::printf("lab mismatches: %llu\n", (unsigned long long)bad_lab);
    return (bad_pow || bad_cbrt || bad_lab) ? 1 : 0;
}
