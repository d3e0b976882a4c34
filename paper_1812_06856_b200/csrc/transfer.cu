// Host <-> device transfers of the end-to-end path: LAB images in ([V][H][W][3] float, ideally
// pinned host memory), planes + depth rasters out.  Uploads go through a float3 staging
// buffer and a repack kernel into the float4 layout the kernels gather from, so a pinned
// source is one DMA per view (no host-side reformatting).
#include "context.h"
#include "glibc_math.cuh"

namespace lfdg {
namespace {
__global__ void k_repack(const float* __restrict__ src, float4* __restrict__ dst, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = make_float4(src[3 * i], src[3 * i + 1], src[3 * i + 2], 0.f);
}
// rgb_to_scaled_lab (image.hpp:97-107) fused with the repack: sRGB [n][3] -> scaled LAB float4,
// bit-identical to the reference through the glibc powf / cbrtf ports (glibc_math.cuh).
__global__ void k_rgb_to_lab(const float* __restrict__ src, float4* __restrict__ dst, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float L, A, B;
    libm::rgb_to_scaled_lab(src[3 * i], src[3 * i + 1], src[3 * i + 2], L, A, B);
    dst[i] = make_float4(L, A, B, 0.f);
}
// 8-bit sRGB (read_image, io.hpp:136-146: channel / 255.f) -> rgb_to_scaled_lab -> float4, so
// decoded 8-bit views cross PCIe at a quarter of the float bytes.
__global__ void k_rgb8_to_lab(const unsigned char* __restrict__ src, float4* __restrict__ dst, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float r = (float)src[3 * i] / 255.f, g = (float)src[3 * i + 1] / 255.f, b = (float)src[3 * i + 2] / 255.f;
    float L, A, B;
    libm::rgb_to_scaled_lab(r, g, b, L, A, B);
    dst[i] = make_float4(L, A, B, 0.f);
}
}  // namespace

// The float staging buffer (stage_s.buf) is shared by the serial uploads (upload_images /
// upload_rgb, compute stream) and the pipelined prefetch (copy stream).  A serial upload while a
// prefetch is uncommitted would be overwritten by (or overwrite) the staged views, so it is
// refused; after a serial repack the buffer is marked consumed on the compute stream, so the
// next prefetch's copy waits for the repack instead of racing it.
static void staging_acquire(Ctx& c) {
    if (c.pipe.has_staged) throw Error(LFDG_STATE, "a prefetched upload is still uncommitted");
}
static void staging_release(Ctx& c) {
    if (c.pipe.stream) LFDG_CUDA_CHECK(cudaEventRecord(c.pipe.consumed, c.stream));
}

// 8-bit sRGB images in ([n][H][W][3] bytes, R G B order), converted like read_image +
// rgb_to_scaled_lab on the device.
void upload_rgb8(Ctx& c, int v0, int n, const unsigned char* host) {
    c.require_views();
    if (v0 < 0 || n < 0 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    if (n == 0) return;
    if (!host) throw Error(LFDG_STATE, "null images");
    const size_t hw = c.hw();
    StagingScratch& s = c.stage_s;
    s.buf8.alloc((size_t)c.V * hw * 3);
    LFDG_CUDA_CHECK(cudaMemcpyAsync(s.buf8.p, host, (size_t)n * hw * 3, cudaMemcpyHostToDevice, c.stream));
    const size_t m = (size_t)n * hw;
    k_rgb8_to_lab<<<(unsigned)((m + 255) / 256), 256, 0, c.stream>>>(s.buf8.p, c.lab.p + (size_t)v0 * hw, m);
    LFDG_LAUNCHED(&c);
}

// sRGB images in ([n][H][W][3] floats in [0, 1]), converted to the scaled LAB the hot path reads
// on the device (the reference converts on the host before the path, pipeline.hpp:245).
void upload_rgb(Ctx& c, int v0, int n, const float* host) {
    c.require_views();
    if (v0 < 0 || n < 0 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    if (n == 0) return;
    if (!host) throw Error(LFDG_STATE, "null images");
    staging_acquire(c);
    const size_t hw = c.hw();
    StagingScratch& s = c.stage_s;
    s.buf.alloc((size_t)c.V * hw * 3);
    LFDG_CUDA_CHECK(cudaMemcpyAsync(s.buf.p, host, (size_t)n * hw * 3 * sizeof(float), cudaMemcpyHostToDevice, c.stream));
    const size_t m = (size_t)n * hw;
    k_rgb_to_lab<<<(unsigned)((m + 255) / 256), 256, 0, c.stream>>>(s.buf.p, c.lab.p + (size_t)v0 * hw, m);
    LFDG_LAUNCHED(&c);
    staging_release(c);
}

void upload_images(Ctx& c, int v0, int n, const float* host) {
    c.require_views();
    if (v0 < 0 || n < 0 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    if (n == 0) return;
    if (!host) throw Error(LFDG_STATE, "null images");
    staging_acquire(c);
    const size_t hw = c.hw();
    StagingScratch& s = c.stage_s;
    s.buf.alloc((size_t)c.V * hw * 3);
    LFDG_CUDA_CHECK(cudaMemcpyAsync(s.buf.p, host, (size_t)n * hw * 3 * sizeof(float), cudaMemcpyHostToDevice, c.stream));
    const size_t m = (size_t)n * hw;
    k_repack<<<(unsigned)((m + 255) / 256), 256, 0, c.stream>>>(s.buf.p, c.lab.p + (size_t)v0 * hw, m);
    LFDG_LAUNCHED(&c);
    staging_release(c);
}

// ---- pipelined transfers ---------------------------------------------------------------------
static void ensure_pipe(Ctx& c) {
    CopyPipe& q = c.pipe;
    if (q.stream) return;
    LFDG_CUDA_CHECK(cudaStreamCreateWithFlags(&q.stream, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&q.staged, &q.consumed, &q.computed, &q.downloaded})
        LFDG_CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    LFDG_CUDA_CHECK(cudaEventRecord(q.consumed, c.stream));  // the staging buffer starts free
}

// H2D of views [v0, v0+n) (scaled LAB floats) into the staging buffer on the copy stream, after
// the previous commit has consumed it; overlaps whatever the compute stream is doing.
void prefetch_images(Ctx& c, int v0, int n, const float* host) {
    c.require_views();
    if (v0 < 0 || n < 1 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    if (!host) throw Error(LFDG_STATE, "null images");
    ensure_pipe(c);
    CopyPipe& q = c.pipe;
    if (q.has_staged) throw Error(LFDG_STATE, "a prefetched upload is still uncommitted");
    const size_t hw = c.hw();
    c.stage_s.buf.alloc((size_t)c.V * hw * 3);
    LFDG_CUDA_CHECK(cudaStreamWaitEvent(q.stream, q.consumed, 0));
    LFDG_CUDA_CHECK(cudaMemcpyAsync(c.stage_s.buf.p, host, (size_t)n * hw * 3 * sizeof(float), cudaMemcpyHostToDevice,
                                    q.stream));
    LFDG_CUDA_CHECK(cudaEventRecord(q.staged, q.stream));
    q.v0 = v0;
    q.n = n;
    q.has_staged = true;
}

// On the compute stream: wait for the staged copy and repack it into the LAB the kernels read.
void commit_images(Ctx& c) {
    CopyPipe& q = c.pipe;
    if (!q.has_staged) throw Error(LFDG_STATE, "no prefetched upload to commit");
    const size_t hw = c.hw();
    LFDG_CUDA_CHECK(cudaStreamWaitEvent(c.stream, q.staged, 0));
    const size_t m = (size_t)q.n * hw;
    k_repack<<<(unsigned)((m + 255) / 256), 256, 0, c.stream>>>(c.stage_s.buf.p, c.lab.p + (size_t)q.v0 * hw, m);
    LFDG_LAUNCHED(&c);
    LFDG_CUDA_CHECK(cudaEventRecord(q.consumed, c.stream));
    q.has_staged = false;
}

// D2H of the current planes / depth of views [v0, v0+n) on the copy stream, ordered after the
// work enqueued so far on the compute stream.  Call wait_downloads before anything overwrites
// planes or depth (the next sweep).
void download_results_async(Ctx& c, int v0, int n, lfdg_plane* planes, float* depth) {
    c.require_views();
    if (v0 < 0 || n < 0 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    ensure_pipe(c);
    CopyPipe& q = c.pipe;
    LFDG_CUDA_CHECK(cudaEventRecord(q.computed, c.stream));
    LFDG_CUDA_CHECK(cudaStreamWaitEvent(q.stream, q.computed, 0));
    if (planes)
        LFDG_CUDA_CHECK(cudaMemcpyAsync(planes, c.planes.p + (size_t)v0 * c.nsp, (size_t)n * c.nsp * sizeof(lfdg_plane),
                                        cudaMemcpyDeviceToHost, q.stream));
    if (depth)
        LFDG_CUDA_CHECK(cudaMemcpyAsync(depth, c.depth.p + (size_t)v0 * c.hw(), (size_t)n * c.hw() * sizeof(float),
                                        cudaMemcpyDeviceToHost, q.stream));
    LFDG_CUDA_CHECK(cudaEventRecord(q.downloaded, q.stream));
    q.has_download = true;
}

void wait_downloads(Ctx& c) {
    CopyPipe& q = c.pipe;
    if (!q.has_download) return;
    LFDG_CUDA_CHECK(cudaStreamWaitEvent(c.stream, q.downloaded, 0));
    q.has_download = false;
}

void download_results(Ctx& c, int v0, int n, lfdg_plane* planes, float* depth) {
    c.require_views();
    if (v0 < 0 || n < 0 || v0 + n > c.V) throw Error(LFDG_STATE, "view range out of bounds");
    if (planes)
        LFDG_CUDA_CHECK(cudaMemcpyAsync(planes, c.planes.p + (size_t)v0 * c.nsp, (size_t)n * c.nsp * sizeof(lfdg_plane),
                                        cudaMemcpyDeviceToHost, c.stream));
    if (depth)
        LFDG_CUDA_CHECK(cudaMemcpyAsync(depth, c.depth.p + (size_t)v0 * c.hw(), (size_t)n * c.hw() * sizeof(float),
                                        cudaMemcpyDeviceToHost, c.stream));
}

}  // namespace lfdg

extern "C" {

int lfdg_upload_images(lfdg_ctx* p, int v0, int n, const float* images) {
    const lfdg::NvtxRange range_("upload_images");
    try {
        auto* c = reinterpret_cast<lfdg::Ctx*>(p);
        if (!c) throw lfdg::Error(LFDG_STATE, "null context");
        LFDG_CUDA_CHECK(cudaSetDevice(c->device));
        lfdg::upload_images(*c, v0, n, images);
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        lfdg::set_last_error(e.what());
        return e.code;
    }
}

int lfdg_upload_rgb(lfdg_ctx* p, int v0, int n, const float* rgb) {
    const lfdg::NvtxRange range_("upload_rgb");
    try {
        auto* c = reinterpret_cast<lfdg::Ctx*>(p);
        if (!c) throw lfdg::Error(LFDG_STATE, "null context");
        LFDG_CUDA_CHECK(cudaSetDevice(c->device));
        lfdg::upload_rgb(*c, v0, n, rgb);
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        lfdg::set_last_error(e.what());
        return e.code;
    }
}

#define LFDG_TRANSFER_ENTRY(body)                                   \
    try {                                                           \
        auto* c = reinterpret_cast<lfdg::Ctx*>(p);                  \
        if (!c) throw lfdg::Error(LFDG_STATE, "null context");     \
        LFDG_CUDA_CHECK(cudaSetDevice(c->device));                  \
        body;                                                       \
        return LFDG_OK;                                             \
    } catch (const lfdg::Error& e) {                                \
        lfdg::set_last_error(e.what());                             \
        return e.code;                                              \
    }

int lfdg_prefetch_images(lfdg_ctx* p, int v0, int n, const float* images) {
    const lfdg::NvtxRange range_("prefetch_images");
    LFDG_TRANSFER_ENTRY(lfdg::prefetch_images(*c, v0, n, images))
}

int lfdg_commit_images(lfdg_ctx* p) {
    const lfdg::NvtxRange range_("commit_images");
    LFDG_TRANSFER_ENTRY(lfdg::commit_images(*c))
}

int lfdg_download_results_async(lfdg_ctx* p, int v0, int n, lfdg_plane* planes, float* depth) {
    const lfdg::NvtxRange range_("download_results_async");
    LFDG_TRANSFER_ENTRY(lfdg::download_results_async(*c, v0, n, planes, depth))
}

int lfdg_wait_downloads(lfdg_ctx* p) { LFDG_TRANSFER_ENTRY(lfdg::wait_downloads(*c)) }

int lfdg_upload_rgb8(lfdg_ctx* p, int v0, int n, const unsigned char* rgb8) {
    const lfdg::NvtxRange range_("upload_rgb8");
    try {
        auto* c = reinterpret_cast<lfdg::Ctx*>(p);
        if (!c) throw lfdg::Error(LFDG_STATE, "null context");
        LFDG_CUDA_CHECK(cudaSetDevice(c->device));
        lfdg::upload_rgb8(*c, v0, n, rgb8);
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        lfdg::set_last_error(e.what());
        return e.code;
    }
}

int lfdg_rgb_to_scaled_lab_gpu(int device, const float* rgb, float* lab, size_t n) {
    try {
        if (!rgb || !lab) throw lfdg::Error(LFDG_STATE, "null buffer");
        LFDG_CUDA_CHECK(cudaSetDevice(device));
        if (n == 0) return LFDG_OK;
        cudaStream_t st = nullptr;
        LFDG_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{st};
        lfdg::DevBuf<float> din;   // RAII: freed on every exit path
        lfdg::DevBuf<float4> dout;
        din.alloc(n * 3);
        dout.alloc(n);
        LFDG_CUDA_CHECK(cudaMemcpyAsync(din.p, rgb, n * 3 * sizeof(float), cudaMemcpyHostToDevice, st));
        lfdg::k_rgb_to_lab<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(din.p, dout.p, n);
        LFDG_CUDA_CHECK(cudaGetLastError());
        LFDG_CUDA_CHECK(cudaMemcpy2DAsync(lab, 3 * sizeof(float), dout.p, sizeof(float4), 3 * sizeof(float), n,
                                          cudaMemcpyDeviceToHost, st));
        LFDG_CUDA_CHECK(cudaStreamSynchronize(st));
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        lfdg::set_last_error(e.what());
        return e.code;
    }
}

int lfdg_download_results(lfdg_ctx* p, int v0, int n, lfdg_plane* planes, float* depth, int sync) {
    const lfdg::NvtxRange range_("download_results");
    try {
        auto* c = reinterpret_cast<lfdg::Ctx*>(p);
        if (!c) throw lfdg::Error(LFDG_STATE, "null context");
        LFDG_CUDA_CHECK(cudaSetDevice(c->device));
        lfdg::download_results(*c, v0, n, planes, depth);
        if (sync) LFDG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        lfdg::set_last_error(e.what());
        return e.code;
    }
}

}  // extern "C"
