// Host check of the glibc exp/expf ports (paper_1812_06856_b200/csrc/glibc_math.cuh) against
// the host libm.  Default: expf on every 61st float bit pattern, exp on 3e7 samples over
// random / special ranges incl. [-1100, -700].  --exhaustive: every float for expf.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

#include "glibc_math.cuh"

int main(int argc, char** argv) {
    const bool exhaustive = argc > 1 && !std::strcmp(argv[1], "--exhaustive");
    const uint64_t stride = exhaustive ? 1 : 61;
    uint64_t bad = 0;
    for (uint64_t u = 0; u < (1ull << 32); u += stride) {
        const uint32_t b = static_cast<uint32_t>(u);
        float x;
        std::memcpy(&x, &b, 4);
        const float a = ::expf(x), c = lfdg::libm::expf(x);
        if (std::memcmp(&a, &c, 4) != 0 && !(std::isnan(a) && std::isnan(c))) {
            if (bad < 5) std::printf("expf x=%a libm=%a port=%a\n", x, a, c);
            ++bad;
        }
    }
    std::printf("expf mismatches: %llu\n", static_cast<unsigned long long>(bad));
    uint64_t bad_d = 0;
    std::mt19937_64 rng(1);
    const double ranges[][2] = {{-800, 5}, {-1100, -700}, {-746.5, -745.0}, {-1100, 1100}, {-1, 1}, {-30, 0}};
    for (const auto& r : ranges) {
        std::uniform_real_distribution<double> U(r[0], r[1]);
        for (int i = 0; i < 4000000; ++i) {
            const double x = U(rng);
            const double a = ::exp(x), c = lfdg::libm::exp(x);
            if (std::memcmp(&a, &c, 8) != 0) {
                if (bad_d < 5) std::printf("exp x=%a libm=%a port=%a\n", x, a, c);
                ++bad_d;
            }
        }
    }
    for (int i = 0; i < 6000000; ++i) {
        const uint64_t u = rng();
        double x;
        std::memcpy(&x, &u, 8);
        const double a = ::exp(x), c = lfdg::libm::exp(x);
        if (std::memcmp(&a, &c, 8) != 0 && !(std::isnan(a) && std::isnan(c))) {
            if (bad_d < 10) std::printf("exp x=%a libm=%a port=%a\n", x, a, c);
            ++bad_d;
        }
    }
    // exp_nonpos (the hot-loop variant) on the non-positive half, incl. the special ranges
    std::uniform_real_distribution<double> N1(-1100, 0), N2(-800, -500), N3(-1e-15, 0);
    for (int i = 0; i < 12000000; ++i) {
        const double x = i % 3 == 0 ? N1(rng) : i % 3 == 1 ? N2(rng) : N3(rng);
        const double a = ::exp(x), c = lfdg::libm::exp_nonpos(x);
        if (std::memcmp(&a, &c, 8) != 0) {
            if (bad_d < 15) std::printf("exp_nonpos x=%a libm=%a port=%a\n", x, a, c);
            ++bad_d;
        }
    }
    for (const double x : {0.0, -0.0, -0x1p-54, -0x1.fffffffffffffp-55, -512.0, -745.13321910194110842, -746.0,
                           -1024.0, -1e300, -(double)INFINITY, (double)NAN}) {
        const double a = ::exp(x), c = lfdg::libm::exp_nonpos(x);
        if (std::memcmp(&a, &c, 8) != 0 && !(std::isnan(a) && std::isnan(c))) {
            std::printf("exp_nonpos x=%a libm=%a port=%a\n", x, a, c);
            ++bad_d;
        }
    }
    std::printf("exp mismatches: %llu\n", static_cast<unsigned long long>(bad_d));
    return (bad || bad_d) ? 1 : 0;
}
