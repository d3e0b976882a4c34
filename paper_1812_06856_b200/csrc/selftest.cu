// Self-test entry points of the C-ABI: evaluate the device ports of glibc exp/expf
// (glibc_math.cuh) on caller-supplied inputs so tests can compare them with the host libm.
#include "context.h"
#include "glibc_math.cuh"

namespace {
__global__ void k_exp(const double* in, double* out, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = lfdg::libm::exp(in[i]);
}
__global__ void k_exp_nonpos(const double* in, double* out, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = lfdg::libm::exp_nonpos(in[i]);
}
__global__ void k_expf(const float* in, float* out, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = lfdg::libm::expf(in[i]);
}
template <typename T, typename K>
int run(int device, const T* in, T* out, size_t n, K kernel) {
    try {
        LFDG_CUDA_CHECK(cudaSetDevice(device));
        T *din = nullptr, *dout = nullptr;
        LFDG_CUDA_CHECK(cudaMalloc(&din, n * sizeof(T)));
        LFDG_CUDA_CHECK(cudaMalloc(&dout, n * sizeof(T)));
        LFDG_CUDA_CHECK(cudaMemcpy(din, in, n * sizeof(T), cudaMemcpyHostToDevice));
        kernel<<<(unsigned)((n + 255) / 256), 256>>>(din, dout, n);
        LFDG_CUDA_CHECK(cudaGetLastError());
        LFDG_CUDA_CHECK(cudaMemcpy(out, dout, n * sizeof(T), cudaMemcpyDeviceToHost));
        cudaFree(din);
        cudaFree(dout);
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        return e.code;
    }
}
}  // namespace

extern "C" {
int lfdg_selftest_exp(int device, const double* in, double* out, size_t n) { return run(device, in, out, n, k_exp); }
int lfdg_selftest_exp_nonpos(int device, const double* in, double* out, size_t n) {
    return run(device, in, out, n, k_exp_nonpos);
}
int lfdg_selftest_expf(int device, const float* in, float* out, size_t n) { return run(device, in, out, n, k_expf); }
}

// FP64 roofline denominator: dependent-free DFMA stream (8 independent chains per thread,
// grid = 148 SMs x 8 CTAs x 256 threads); returns achieved FLOP/s counting a DFMA as 2.
namespace {
__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
        x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
    }
    const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 1.2345) out[0] = s;
}
}  // namespace

namespace {
__global__ void k_ffma(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = __fmaf_rn(x0, a, b); x1 = __fmaf_rn(x1, a, b); x2 = __fmaf_rn(x2, a, b); x3 = __fmaf_rn(x3, a, b);
        x4 = __fmaf_rn(x4, a, b); x5 = __fmaf_rn(x5, a, b); x6 = __fmaf_rn(x6, a, b); x7 = __fmaf_rn(x7, a, b);
    }
    const float s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 1.2345f) out[0] = s;
}

// Best-of-5 event time of `launch` over `flop` floating-point operations -> FLOP/s.
template <typename L>
double time_flops(L launch, double flop) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return flop / (best * 1e-3);
}
}  // namespace

// FP32 roofline denominator (the sweep's bilinear / TSSD arithmetic): FFMA stream, 8 independent
// chains per thread, 148 SMs x 8 CTAs x 256 threads; an FFMA counts as 2 FLOP.
extern "C" int lfdg_selftest_fp32_peak(int device, double* flops) {
    try {
        LFDG_CUDA_CHECK(cudaSetDevice(device));
        int sms = 0;
        LFDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        lfdg::DevBuf<float> out;
        out.alloc(1);
        const int iters = 16384, blocks = sms * 8, threads = 256;
        *flops = time_flops([&] { k_ffma<<<blocks, threads>>>(out.p, iters, 0.999999f, 1e-7f); },
                            2.0 * 8.0 * iters * (double)blocks * threads);
        LFDG_CUDA_CHECK(cudaGetLastError());
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        return e.code;
    }
}

extern "C" int lfdg_selftest_fp64_peak(int device, double* flops) {
    try {
        LFDG_CUDA_CHECK(cudaSetDevice(device));
        int sms = 0;
        LFDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        double* out = nullptr;
        LFDG_CUDA_CHECK(cudaMalloc(&out, sizeof(double)));
        const int iters = 4096, blocks = sms * 8, threads = 256;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);  // warm-up
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            cudaEventRecord(e1);
            LFDG_CUDA_CHECK(cudaEventSynchronize(e1));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(out);
        *flops = 2.0 * 8.0 * iters * (double)blocks * threads / (best * 1e-3);
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        return e.code;
    }
}
