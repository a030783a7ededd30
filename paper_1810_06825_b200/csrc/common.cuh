// Shared plumbing for the B200 frPCA hot path: status codes, error capture,
// device buffers. All panels on the device are ROW-MAJOR r x l (ld = l), so a
// CSR nonzero gathers one contiguous l*8-byte row of the dense operand.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <chrono>
#include <cstdlib>
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

// Large device buffers are recycled per device instead of going back to the
// stream-ordered pool. Measured at C3 (tools/e2e_ab.py, FRPCA_DEBUG_ALLOC):
// re-taking a multi-GB block from the pool cost 10-600 ms of host time per
// cudaMallocAsync while copies and kernels were in flight, although every
// call of a repeated run asks for the same sizes. A released buffer of at
// least kCacheMin bytes is parked with an event recorded on its last stream;
// a later request of the same device takes the smallest parked buffer that
// fits within 1/8 slack, after making its stream wait on that event (the
// ordering the pool itself would provide). Parked buffers go back to the
// pool when an allocation fails (then retried), beyond kCacheMax bytes, or
// when the device has less than kMinFree bytes free.
// current device switched for a scope (restored on exit)
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

struct BufCache {
    struct Entry {
        void* p;
        size_t bytes;
        int dev;
        cudaEvent_t ev;
    };
    static constexpr size_t kCacheMin = size_t(32) << 20;
    static constexpr size_t kCacheMax = size_t(128) << 30;
    static constexpr size_t kMinFree = size_t(20) << 30;  // device headroom kept for other allocators
    std::mutex mu;
    std::vector<Entry> parked;
    size_t held = 0;
    std::chrono::steady_clock::time_point last_check{};
    static BufCache& get() {
        static BufCache* c = new BufCache;  // never destroyed (process exit order)
        return *c;
    }
    // back to the stream-ordered pool (no unmap: the pool keeps its memory)
    static void drop(Entry& e) {
        DeviceScope ds(e.dev);  // (the buffer's device, whatever the caller's)
        cudaEventSynchronize(e.ev);
        cudaEventDestroy(e.ev);
        cudaFreeAsync(e.p, cudaStreamPerThread);
    }
    // a parked buffer of [bytes, bytes + bytes/8] on this device, or nullptr
    void* take(size_t bytes, cudaStream_t s, size_t& cap) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
        std::lock_guard<std::mutex> lk(mu);
        size_t best = parked.size();
        for (size_t k = 0; k < parked.size(); ++k) {
            const Entry& e = parked[k];
            if (e.dev == dev && e.bytes >= bytes && e.bytes - bytes <= bytes / 8 &&
                (best == parked.size() || e.bytes < parked[best].bytes))
                best = k;
        }
        if (best == parked.size()) return nullptr;
        Entry e = parked[best];
        parked.erase(parked.begin() + long(best));
        held -= e.bytes;
        cudaStreamWaitEvent(s, e.ev, 0);
        cudaEventDestroy(e.ev);
        cap = e.bytes;
        return e.p;
    }
    bool give(void* p, size_t bytes, cudaStream_t s, int dev) {
        static const bool dbg = std::getenv("FRPCA_DEBUG_E2E") != nullptr;
        const auto g0 = std::chrono::steady_clock::now();
        struct Report {
            bool on;
            std::chrono::steady_clock::time_point t0;
            size_t bytes;
            int drops = 0;
            bool checked = false;
            ~Report() {
                if (!on) return;
                const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                if (ms > 2.0)
                    std::fprintf(stderr, "[e2e] park %.1f MB took %.1f ms (mem check %d, drops %d)\n", bytes / 1e6, ms,
                                 int(checked), drops);
            }
        } rep{dbg, g0, bytes};
        DeviceScope ds(dev);  // the event belongs to the buffer's device (its last stream's)
        cudaEvent_t ev;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (cudaEventRecord(ev, s) != cudaSuccess) {
            cudaGetLastError();  // (not left for a later launch check)
            cudaEventDestroy(ev);
            return false;
        }
        std::lock_guard<std::mutex> lk(mu);
        parked.push_back({p, bytes, dev, ev});
        held += bytes;
        // device headroom, checked at most every 2 s (cudaMemGetInfo stalled a
        // release for ~40 ms now and then, measured inside frpca_run_csr)
        bool low = false;
        const auto now = std::chrono::steady_clock::now();
        if (now - last_check > std::chrono::seconds(2)) {
            last_check = now;
            size_t fr = 0, tot = 0;
            low = cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr < kMinFree;
            rep.checked = true;
        }
        // oldest first: beyond the cap any device's, when this device is short
        // of memory this device's
        for (size_t k = 0; k + 1 < parked.size();) {
            const bool over = held > kCacheMax;
            const bool mine_low = low && parked[k].dev == dev && held > bytes;
            if (!over && !(low && held > bytes)) break;
            if (over || mine_low) {
                held -= parked[k].bytes;
                drop(parked[k]);
                parked.erase(parked.begin() + long(k));
                ++rep.drops;
            } else {
                ++k;
            }
        }
        return true;
    }
    void flush() {
        std::lock_guard<std::mutex> lk(mu);
        for (auto& e : parked) drop(e);
        parked.clear();
        held = 0;
        cudaStreamSynchronize(cudaStreamPerThread);  // the pool can hand the memory out again
    }
};

// Minimal owning device buffer (stream-ordered allocation; large buffers
// recycled through BufCache).
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    size_t cap = 0;  // bytes actually held (>= n * sizeof(T))
    int dev = 0;     // device of the allocation
    DBuf() = default;
    DBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), cap(o.cap), dev(o.dev) { o.p = nullptr; o.n = 0; o.cap = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; s = o.s; cap = o.cap; dev = o.dev;
            o.p = nullptr; o.n = 0; o.cap = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count, cudaStream_t stream) {
        release();
        s = stream;
        n = count;
        if (!count) return;
        cudaGetDevice(&dev);
        const size_t bytes = count * sizeof(T);
        if (bytes >= BufCache::kCacheMin) {
            if (void* q = BufCache::get().take(bytes, stream, cap)) {
                p = static_cast<T*>(q);
                return;
            }
        }
        cap = bytes;
        static const bool dbg = std::getenv("FRPCA_DEBUG_E2E") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, stream);
        if (dbg) {
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (ms > 2.0) std::fprintf(stderr, "[e2e] cudaMallocAsync %.1f MB took %.1f ms\n", bytes / 1e6, ms);
        }
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            BufCache::get().flush();
            e = cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, stream);
        }
        if (e != cudaSuccess) {
            p = nullptr;
            n = cap = 0;
            FB_CUDA(e);
        }
    }
    void release() noexcept {
        if (p && !(cap >= BufCache::kCacheMin && BufCache::get().give(p, cap, s, dev))) cudaFreeAsync(p, s);
        p = nullptr;
        n = cap = 0;
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
