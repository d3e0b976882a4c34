// Device allocator behind DevBuf (context.h) with an optional out-of-bounds-write detector.
//
// LFDG_GUARD=1 (read once, at the first allocation): each buffer is allocated as
// [64 KiB guard | payload | 64 KiB guard], both guards filled with 0xA5, and registered;
// lfdg_debug_check_guards() copies every live buffer's guards back and counts the corrupted
// ones.  Payload addresses stay 256-byte aligned (the guard is a multiple of 256 B).
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "context.h"

namespace lfdg {
namespace {
constexpr size_t kGuard = 64 * 1024;
constexpr unsigned char kPattern = 0xA5;
std::mutex g_mu;
std::unordered_map<void*, size_t>& registry() {
    static std::unordered_map<void*, size_t> r;  // payload pointer -> payload bytes
    return r;
}
}  // namespace

bool guard_mode() {
    static const bool on = [] {
        const char* e = std::getenv("LFDG_GUARD");
        return e && e[0] == '1';
    }();
    return on;
}

void* dev_alloc(size_t bytes) {
    if (!guard_mode()) {
        void* p = nullptr;
        LFDG_CUDA_CHECK(cudaMalloc(&p, bytes));
        return p;
    }
    unsigned char* base = nullptr;
    LFDG_CUDA_CHECK(cudaMalloc(&base, bytes + 2 * kGuard));
    LFDG_CUDA_CHECK(cudaMemset(base, kPattern, kGuard));
    LFDG_CUDA_CHECK(cudaMemset(base + kGuard + bytes, kPattern, kGuard));
    void* p = base + kGuard;
    std::lock_guard<std::mutex> lk(g_mu);
    registry()[p] = bytes;
    return p;
}

void dev_free(void* p) {
    if (!p) return;
    if (!guard_mode()) {
        cudaFree(p);
        return;
    }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        registry().erase(p);
    }
    cudaFree(static_cast<unsigned char*>(p) - kGuard);
}

namespace {
bool guards_intact(void* p, size_t bytes, std::vector<unsigned char>& tmp) {
    tmp.resize(kGuard);
    const unsigned char* base = static_cast<unsigned char*>(p) - kGuard;
    for (const unsigned char* g : {base, base + kGuard + bytes}) {
        LFDG_CUDA_CHECK(cudaMemcpy(tmp.data(), g, kGuard, cudaMemcpyDeviceToHost));
        for (unsigned char b : tmp)
            if (b != kPattern) return false;
    }
    return true;
}
}  // namespace
}  // namespace lfdg

extern "C" {

int lfdg_debug_guard_enabled(void) { return lfdg::guard_mode() ? 1 : 0; }

int lfdg_debug_check_guards(uint64_t* n_buffers, uint64_t* n_corrupt) {
    try {
        LFDG_CUDA_CHECK(cudaDeviceSynchronize());
        std::lock_guard<std::mutex> lk(lfdg::g_mu);
        std::vector<unsigned char> tmp;
        uint64_t nb = 0, nc = 0;
        for (const auto& kv : lfdg::registry()) {
            ++nb;
            if (!lfdg::guards_intact(kv.first, kv.second, tmp)) ++nc;
        }
        if (n_buffers) *n_buffers = nb;
        if (n_corrupt) *n_corrupt = nc;
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        return e.code;
    }
}

int lfdg_debug_guard_selftest(int device, uint64_t* detected) {
    try {
        if (!lfdg::guard_mode()) return LFDG_STATE;
        LFDG_CUDA_CHECK(cudaSetDevice(device));
        uint64_t before = 0, after = 0;
        {
            lfdg::DevBuf<int> b;
            b.alloc(1000);
            LFDG_CUDA_CHECK(cudaMemset(b.p, 0, 1000 * sizeof(int)));  // in bounds: no report
            if (lfdg_debug_check_guards(nullptr, &before) != LFDG_OK) return LFDG_CUDA;
            LFDG_CUDA_CHECK(cudaMemset(b.p + 1000, 0, sizeof(int)));  // one element past the end
            if (lfdg_debug_check_guards(nullptr, &after) != LFDG_OK) return LFDG_CUDA;
        }
        if (detected) *detected = (before == 0 && after == 1) ? 1 : 0;
        return LFDG_OK;
    } catch (const lfdg::Error& e) {
        return e.code;
    }
}

}  // extern "C"
