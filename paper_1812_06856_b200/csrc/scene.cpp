// Synthetic camera-array scenes for the bench and the parity tests: a host C++ restatement of
// the reference's fixture generator (proj/include/lfd/fixtures.hpp) and of its sRGB ->
// scaled-LAB conversion (image.hpp:71-107), so the product's bench can build BASELINE.json's
// configs without the reference.  Arithmetic follows the reference operation by operation
// (Eigen fixed-size order, -ffp-contract=off, glibc powf/cbrtf), so the images are
// byte-identical to the reference's (tests/test_scene.py checks this against oracle/_ref).
// Rendering is parallelised over rows with std::thread; the result does not depend on the
// thread count (each pixel is written once).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/lfdg.h"

namespace {

struct V3 {
    double x, y, z;
};
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 scale(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline V3 normalized(V3 a) {
    const double z = dot(a, a);
    if (z > 0) {
        const double n = std::sqrt(z);
        return {a.x / n, a.y / n, a.z / n};
    }
    return a;
}

// splitmix64 / derive_stream (rng.hpp:9-39)
inline uint64_t mix64(uint64_t& state) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline uint64_t derive(uint64_t seed, uint64_t view, uint64_t sp) {
    uint64_t h = seed;
    h ^= (view + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2));
    h *= 0xFF51AFD7ED558CCDull;
    h ^= (sp + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2));
    h *= 0xC4CEB9FE1A85EC53ull;
    h ^= h >> 33;
    return h;
}

// PatchTexture (fixtures.hpp:20-53)
struct Texture {
    bool noise = false;
    double scale = 0.1;
    float a[3] = {0.9f, 0.9f, 0.9f};
    float b[3] = {0.1f, 0.1f, 0.1f};
    uint64_t seed = 0;

    void sample(double u, double v, float out[3]) const {
        if (!noise) {
            const long long ia = static_cast<long long>(std::floor(u / scale));
            const long long ib = static_cast<long long>(std::floor(v / scale));
            const float* c = ((ia + ib) & 1) ? b : a;
            out[0] = c[0];
            out[1] = c[1];
            out[2] = c[2];
            return;
        }
        const double fa = u / scale, fb = v / scale;
        const long long ia = static_cast<long long>(std::floor(fa));
        const long long ib = static_cast<long long>(std::floor(fb));
        const double ta = fa - ia, tb = fb - ib;
        auto lattice = [this](long long i, long long j, int c) {
            uint64_t st = derive(seed, static_cast<uint64_t>(i * 0x9E3779B9ll + c), static_cast<uint64_t>(j));
            return static_cast<float>(static_cast<double>(mix64(st) >> 11) * 0x1.0p-53);
        };
        for (int c = 0; c < 3; ++c) {
            const double v00 = lattice(ia, ib, c), v10 = lattice(ia + 1, ib, c);
            const double v01 = lattice(ia, ib + 1, c), v11 = lattice(ia + 1, ib + 1, c);
            const double top = v00 + ta * (v10 - v00);
            const double bot = v01 + ta * (v11 - v01);
            const double val = top + tb * (bot - top);
            out[c] = static_cast<float>(a[c] + val * (b[c] - a[c]));
        }
    }
};

struct Patch {  // ScenePatch (fixtures.hpp:57-65)
    V3 origin{0, 0, 0};
    V3 au{1, 0, 0};
    V3 av{0, 1, 0};
    double hu = 1, hv = 1;
    Texture tex;
};

struct Scene {
    std::vector<Patch> patches;
    std::vector<lfdg_camera> cams;
    int W = 0, H = 0;
    double dmin = 0, dmax = 0;
};

lfdg_camera make_pinhole(double f, double cx, double cy, V3 pos) {  // fixtures.hpp:127-132
    lfdg_camera c{};
    const double K[9] = {f, 0, cx, 0, f, cy, 0, 0, 1};
    std::memcpy(c.K, K, sizeof(K));
    for (int i = 0; i < 9; ++i) c.R[i] = (i % 4 == 0) ? 1.0 : 0.0;
    c.t[0] = -pos.x;  // translation = -position (Eigen unary minus)
    c.t[1] = -pos.y;
    c.t[2] = -pos.z;
    return c;
}

std::vector<lfdg_camera> rectified_rig(int n, double f, double B, int w, int h) {  // fixtures.hpp:135-143
    std::vector<lfdg_camera> out;
    for (int i = 0; i < n; ++i) out.push_back(make_pinhole(f, w / 2.0, h / 2.0, V3{i * B, 0, 0}));
    return out;
}

std::vector<lfdg_camera> grid_rig(int nx, int ny, double f, double B, int w, int h) {  // fixtures.hpp:146-155
    std::vector<lfdg_camera> out;
    for (int gy = 0; gy < ny; ++gy)
        for (int gx = 0; gx < nx; ++gx) out.push_back(make_pinhole(f, w / 2.0, h / 2.0, V3{gx * B, gy * B, 0}));
    return out;
}

Patch fronto(double cxf, double cyf, double d, double huf, double hvf, int w, int h, double f, const Texture& t) {
    Patch p;  // fixtures.hpp:209-219
    p.origin = V3{(cxf - 0.5) * w / f * d, (cyf - 0.5) * h / f * d, d};
    p.au = V3{1, 0, 0};
    p.av = V3{0, 1, 0};
    p.hu = huf * w / f * d;
    p.hv = hvf * h / f * d;
    p.tex = t;
    return p;
}

Texture noise_tex(double scale, uint64_t seed, const float a[3], const float b[3]) {
    Texture t;
    t.noise = true;
    t.scale = scale;
    t.seed = seed;
    std::memcpy(t.a, a, sizeof(t.a));
    std::memcpy(t.b, b, sizeof(t.b));
    return t;
}

Scene cluttered(int n, int w, int h, double f, double B) {  // fixtures.hpp:323-383
    Scene s;
    s.W = w;
    s.H = h;
    s.cams = rectified_rig(n, f, B, w, h);
    s.dmin = 2.5;
    s.dmax = 12.0;
    {
        const float a[3] = {0.38f, 0.42f, 0.46f}, b[3] = {0.60f, 0.62f, 0.64f};
        s.patches.push_back(fronto(0.5, 0.5, 11.0, 2.0, 2.0, w, h, f, noise_tex(0.35, 41, a, b)));
    }
    {
        Patch p;
        const double d = 7.0;
        p.origin = V3{-0.20 * w / f * d, 0.12 * h / f * d, d};
        const double t = 35.0 * M_PI / 180.0;
        p.au = V3{std::cos(t), 0, std::sin(t)};
        p.av = V3{0, 1, 0};
        p.hu = 0.35 * w / f * d;
        p.hv = 0.28 * h / f * d;
        const float a[3] = {0.48f, 0.40f, 0.30f}, b[3] = {0.70f, 0.60f, 0.44f};
        p.tex = noise_tex(0.22, 43, a, b);
        s.patches.push_back(p);
    }
    {
        const float a[3] = {0.62f, 0.35f, 0.30f}, b[3] = {0.82f, 0.52f, 0.44f};
        s.patches.push_back(fronto(0.68, 0.40, 5.2, 0.14, 0.20, w, h, f, noise_tex(0.12, 47, a, b)));
    }
    {
        const float a[3] = {0.30f, 0.54f, 0.34f}, b[3] = {0.52f, 0.76f, 0.54f};
        s.patches.push_back(fronto(0.22, 0.30, 6.0, 0.16, 0.14, w, h, f, noise_tex(0.16, 53, a, b)));
    }
    {
        const float a[3] = {0.30f, 0.40f, 0.60f}, b[3] = {0.50f, 0.60f, 0.84f};
        s.patches.push_back(fronto(0.50, 0.72, 4.2, 0.12, 0.10, w, h, f, noise_tex(0.10, 59, a, b)));
    }
    {
        Texture flat;  // checker with one giant cell = constant colour
        flat.noise = false;
        flat.scale = 1e6;
        flat.a[0] = 0.55f;
        flat.a[1] = 0.55f;
        flat.a[2] = 0.6f;
        s.patches.push_back(fronto(0.82, 0.70, 8.5, 0.09, 0.11, w, h, f, flat));
    }
    return s;
}

Scene staircase(int n, int w, int h, double f, double B) {  // fixtures.hpp:242-271
    Scene s;
    s.W = w;
    s.H = h;
    s.cams = rectified_rig(n, f, B, w, h);
    const double depths[3] = {4.0, 6.0, 9.0};
    s.dmin = 3.0;
    s.dmax = 12.0;
    const float sa[3][3] = {{0.45f, 0.25f, 0.20f}, {0.18f, 0.42f, 0.25f}, {0.20f, 0.30f, 0.50f}};
    const float sb[3][3] = {{0.90f, 0.70f, 0.60f}, {0.62f, 0.88f, 0.68f}, {0.62f, 0.72f, 0.95f}};
    for (int k = 0; k < 3; ++k) {
        Patch p = fronto((k + 0.5) / 3.0, 0.5, depths[k], 1.15 / 6.0, 0.8, w, h, f,
                         noise_tex(0.04 * depths[k], 11 + static_cast<uint64_t>(k), sa[k], sb[k]));
        p.hu += B;
        s.patches.push_back(p);
    }
    const float ba[3] = {0.22f, 0.22f, 0.25f}, bb[3] = {0.60f, 0.60f, 0.65f};
    s.patches.push_back(fronto(0.5, 0.5, 11.0, 1.0, 1.0, w, h, f, noise_tex(0.4, 17, ba, bb)));
    s.patches.back().hu += B * n;
    return s;
}

Scene wall(int n, int w, int h, double f, double B, double depth) {  // fixtures.hpp:222-238
    Scene s;
    s.W = w;
    s.H = h;
    s.cams = rectified_rig(n, f, B, w, h);
    s.dmin = depth * 0.5;
    s.dmax = depth * 2.0;
    const float a[3] = {0.25f, 0.32f, 0.40f}, b[3] = {0.78f, 0.75f, 0.65f};
    s.patches.push_back(fronto(0.5, 0.5, depth, 1.0, 1.0, w, h, f, noise_tex(0.05 * depth, 7, a, b)));
    s.patches.back().hu += B * n;
    return s;
}

Scene slanted(int n, int w, int h, double f, double B, double tilt_deg) {  // fixtures.hpp:274-297
    const double center_depth = 6.0;
    Scene s;
    s.W = w;
    s.H = h;
    s.cams = rectified_rig(n, f, B, w, h);
    s.dmin = center_depth * 0.55;
    s.dmax = center_depth * 1.7;
    const double t = tilt_deg * M_PI / 180.0;
    Patch p;
    p.origin = V3{0, 0, center_depth};
    p.au = V3{std::cos(t), 0, std::sin(t)};
    p.av = V3{0, 1, 0};
    p.hu = 3.0 * w / f * center_depth;
    p.hv = 3.0 * h / f * center_depth;
    const float a[3] = {0.40f, 0.45f, 0.40f}, b[3] = {0.70f, 0.72f, 0.65f};
    p.tex = noise_tex(0.05 * center_depth, 23, a, b);
    s.patches.push_back(p);
    return s;
}

Scene occluder(int n, int w, int h, double f, double B) {  // fixtures.hpp:300-319
    Scene s;
    s.W = w;
    s.H = h;
    s.cams = rectified_rig(n, f, B, w, h);
    s.dmin = 2.0;
    s.dmax = 10.0;
    const float a0[3] = {0.20f, 0.28f, 0.45f}, b0[3] = {0.65f, 0.70f, 0.85f};
    s.patches.push_back(fronto(0.5, 0.5, 8.0, 2.0, 2.0, w, h, f, noise_tex(0.3, 31, a0, b0)));
    const float a1[3] = {0.62f, 0.35f, 0.20f}, b1[3] = {0.98f, 0.75f, 0.55f};
    s.patches.push_back(fronto(0.5, 0.5, 3.0, 0.2, 0.25, w, h, f, noise_tex(0.08, 37, a1, b1)));
    return s;
}

// render_scene (fixtures.hpp:85-123) for one view, rows [y0, y1).
void render_rows(const Scene& s, int v, int y0, int y1, float* rgb, float* gt) {
    const lfdg_camera& cam = s.cams[v];
    const double* R = cam.R;
    const double* t = cam.t;
    // center() = -R^T t (geometry.hpp:41)
    const V3 center{((-R[0]) * t[0] + (-R[3]) * t[1]) + (-R[6]) * t[2],
                    ((-R[1]) * t[0] + (-R[4]) * t[1]) + (-R[7]) * t[2],
                    ((-R[2]) * t[0] + (-R[5]) * t[1]) + (-R[8]) * t[2]};
    const double* K = cam.K;
    std::vector<V3> normals;
    for (const Patch& p : s.patches) normals.push_back(normalized(cross(p.au, p.av)));
    for (int y = y0; y < y1; ++y) {
        for (int x = 0; x < s.W; ++x) {
            const double ry = (y - K[5]) / K[4];
            const double rx = ((x - K[2]) - K[1] * ry) / K[0];
            const V3 ray{rx, ry, 1.0};
            const V3 dir{(R[0] * ray.x + R[3] * ray.y) + R[6] * ray.z, (R[1] * ray.x + R[4] * ray.y) + R[7] * ray.z,
                         (R[2] * ray.x + R[5] * ray.y) + R[8] * ray.z};
            double best = 0;
            float color[3] = {0, 0, 0};
            for (size_t k = 0; k < s.patches.size(); ++k) {
                const Patch& p = s.patches[k];
                const V3 n = normals[k];
                const double denom = dot(n, dir);
                if (std::abs(denom) <= 1e-12) continue;
                const double sd = dot(n, sub(p.origin, center)) / denom;
                if (sd <= 0) continue;
                const V3 pt = add(center, scale(sd, dir));
                const double a = dot(sub(pt, p.origin), p.au);
                const double b = dot(sub(pt, p.origin), p.av);
                if (std::abs(a) > p.hu || std::abs(b) > p.hv) continue;
                if (best == 0 || sd < best) {
                    best = sd;
                    p.tex.sample(a, b, color);
                }
            }
            const size_t i = static_cast<size_t>(y) * s.W + x;
            if (gt) gt[i] = static_cast<float>(best);
            if (best > 0) {
                rgb[3 * i] = color[0];
                rgb[3 * i + 1] = color[1];
                rgb[3 * i + 2] = color[2];
            } else {
                rgb[3 * i] = rgb[3 * i + 1] = rgb[3 * i + 2] = 0.f;
            }
        }
    }
}

// rgb_to_scaled_lab (image.hpp:71-95)
inline float srgb_to_linear(float v) { return v <= 0.04045f ? v / 12.92f : std::pow((v + 0.055f) / 1.055f, 2.4f); }
inline float lab_f(float t) {
    constexpr float kEps = 216.f / 24389.f;
    constexpr float kKappa = 24389.f / 27.f;
    return t > kEps ? std::cbrt(t) : (kKappa * t + 16.f) / 116.f;
}
inline void to_lab(const float* rgb, float* lab) {
    const float r = srgb_to_linear(rgb[0]);
    const float g = srgb_to_linear(rgb[1]);
    const float b = srgb_to_linear(rgb[2]);
    const float xr = (0.4124564f * r + 0.3575761f * g + 0.1804375f * b) / 0.95047f;
    const float yr = (0.2126729f * r + 0.7151522f * g + 0.0721750f * b);
    const float zr = (0.0193339f * r + 0.1191920f * g + 0.9503041f * b) / 1.08883f;
    const float fx = lab_f(xr);
    const float fy = lab_f(yr);
    const float fz = lab_f(zr);
    lab[0] = (116.f * fy - 16.f) / 100.f;
    lab[1] = (500.f * (fx - fy)) / 100.f;
    lab[2] = (200.f * (fy - fz)) / 100.f;
}

template <typename Fn>
void parallel_rows(int n, int threads, Fn&& fn) {
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    threads = std::min(threads, n);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        const int lo = static_cast<int>(static_cast<long long>(n) * t / threads);
        const int hi = static_cast<int>(static_cast<long long>(n) * (t + 1) / threads);
        pool.emplace_back([lo, hi, &fn] { fn(lo, hi); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// Scene kinds as in oracle/ref_harness.cpp: 0 cluttered, 1 staircase, 2 wall(depth = extra),
// 3 slanted(tilt = extra), 4 occluder; grid_nx > 0 replaces the rig by make_grid_rig.
// Outputs (any may be NULL): lab/rgb [V][H][W][3], gt [V][H][W], cameras [V], range[2].
static int render_impl(int kind, int n_views, int width, int height, double f, double baseline, double extra,
                       int grid_nx, int grid_ny, const lfdg_camera* cams_in, int n_cams_in, int threads,
                       float* lab_out, float* rgb_out, float* gt_out, lfdg_camera* cams_out, double* range_out) {
    if (width < 1 || height < 1 || n_views < 1) return LFDG_INVALID_PARAMS;
    Scene s;
    switch (kind) {
        case 0: s = cluttered(n_views, width, height, f, baseline); break;
        case 1: s = staircase(n_views, width, height, f, baseline); break;
        case 2: s = wall(n_views, width, height, f, baseline, extra); break;
        case 3: s = slanted(n_views, width, height, f, baseline, extra); break;
        case 4: s = occluder(n_views, width, height, f, baseline); break;
        default: return LFDG_INVALID_PARAMS;
    }
    if (grid_nx > 0) s.cams = grid_rig(grid_nx, grid_ny, f, baseline, width, height);
    if (cams_in) s.cams.assign(cams_in, cams_in + n_cams_in);  // the scene under caller-given cameras
    if (s.cams.size() < 2) return LFDG_INVARIANT;  // SceneSpec::validate (fixtures.hpp:74)
    const int V = static_cast<int>(s.cams.size());
    const size_t hw = static_cast<size_t>(width) * height;
    if (cams_out) std::memcpy(cams_out, s.cams.data(), V * sizeof(lfdg_camera));
    if (range_out) {
        range_out[0] = s.dmin;
        range_out[1] = s.dmax;
    }
    if (!lab_out && !rgb_out && !gt_out) return LFDG_OK;  // rig and range only
    std::vector<float> rgb_tmp;
    float* rgb = rgb_out;
    if (!rgb) {
        rgb_tmp.resize(hw * 3 * V);
        rgb = rgb_tmp.data();
    }
    parallel_rows(V * height, threads, [&](int lo, int hi) {
        for (int r = lo; r < hi;) {
            const int v = r / height, y0 = r % height;
            const int y1 = std::min(height, y0 + (hi - r));
            render_rows(s, v, y0, y1, rgb + v * hw * 3, gt_out ? gt_out + v * hw : nullptr);
            r += y1 - y0;
        }
    });
    if (lab_out) {
        parallel_rows(static_cast<int>(V * height), threads, [&](int lo, int hi) {
            for (size_t i = static_cast<size_t>(lo) * width; i < static_cast<size_t>(hi) * width; ++i)
                to_lab(rgb + 3 * i, lab_out + 3 * i);
        });
    }
    return LFDG_OK;
}

int lfdg_render_scene(int kind, int n_views, int width, int height, double f, double baseline, double extra,
                      int grid_nx, int grid_ny, int threads, float* lab_out, float* rgb_out, float* gt_out,
                      lfdg_camera* cams_out, double* range_out) {
    return render_impl(kind, n_views, width, height, f, baseline, extra, grid_nx, grid_ny, nullptr, 0, threads, lab_out,
                       rgb_out, gt_out, cams_out, range_out);
}

// The scene of (kind, n_views, W, H, f, baseline, extra) rendered through caller-given cameras
// (any calibrated rig: rotations, skew, off-plane centres) — render_scene with spec.cameras
// replaced, as tests/acceptance.cpp:398-399 does with make_grid_rig.
int lfdg_render_scene_cams(int kind, int n_views, int width, int height, double f, double baseline, double extra,
                           const lfdg_camera* cams, int n_cams, int threads, float* lab_out, float* rgb_out,
                           float* gt_out, double* range_out) {
    if (!cams || n_cams < 2) return LFDG_INVALID_PARAMS;
    return render_impl(kind, n_views, width, height, f, baseline, extra, 0, 0, cams, n_cams, threads, lab_out, rgb_out,
                       gt_out, nullptr, range_out);
}

// rgb_to_scaled_lab over n pixels (image.hpp:97-107).
int lfdg_rgb_to_scaled_lab(int64_t n_pixels, const float* rgb, float* lab) {
    for (int64_t i = 0; i < n_pixels; ++i) to_lab(rgb + 3 * i, lab + 3 * i);
    return LFDG_OK;
}

}  // extern "C"
