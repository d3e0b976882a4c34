// Self-test entry points of the C-ABI: evaluate the device ports of glibc exp/expf
// (glibc_math.cuh) on caller-supplied inputs so tests can compare them with the host libm.
#include "context.h"
#include "glibc_math.cuh"

namespace {
__global__ void k_exp(const double* in, double* out, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = lfdg::libm::exp(in[i]);
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
int lfdg_selftest_expf(int device, const float* in, float* out, size_t n) { return run(device, in, out, n, k_expf); }
}
