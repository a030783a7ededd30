// Shared plumbing for the B200 frPCA hot path: status codes, error capture,
// device buffers. All panels on the device are ROW-MAJOR r x l (ld = l), so a
// CSR nonzero gathers one contiguous l*8-byte row of the dense operand.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/frpca_b200.h"
#include "errors.hpp"

namespace fb {

// Exceptions carried to the C-ABI boundary: errors.hpp (plain C++, shared
// with the host-only sources).
// detail::require of types.hpp:45-47: std::invalid_argument with the message.
inline void require(bool cond, const char* msg) {
    if (!cond) throw InvalidArgument(msg);
}

#define FB_CUDA(expr)                                                                    \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            throw ::fb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) +   \
                                  " (" __FILE__ ":" + std::to_string(__LINE__) + ")");   \
    } while (0)

// Every kernel launch in this library is followed by FB_LAUNCH_CHECK(), which
// also counts it (frpca_launch_count, reported by bench.py as gpu_launches).
void count_launch();
#define FB_LAUNCH_CHECK()        \
    do {                         \
        ::fb::count_launch();    \
        FB_CUDA(cudaGetLastError()); \
    } while (0)

// Minimal owning device buffer (stream-ordered allocation).
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count, cudaStream_t stream) {
        release();
        s = stream;
        n = count;
        if (count) FB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), stream));
    }
    void release() noexcept {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
    size_t bytes() const { return n * sizeof(T); }
};

// Opt-in of `fn` to `bytes` of dynamic shared memory on the CURRENT device.
// The attribute is per device, so it is tracked per (kernel, device) and raised
// when a later call needs more; calls from several host threads are serialised.
inline void smem_optin(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    FB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = done[{fn, dev}];
    if (cur >= bytes) return;
    FB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    cur = bytes;
}
template <class K>
inline void smem_optin(K* fn, size_t bytes) { smem_optin(reinterpret_cast<const void*>(fn), bytes); }

inline int ceil_div(int64_t a, int64_t b) { return int((a + b - 1) / b); }

}  // namespace fb
