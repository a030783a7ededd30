// K1/K2: CSR SpMM over row-major fp64 panels, Y = A * X.
//   spmm           (sparse_matrix.hpp:177-206) runs on the CSR of A;
//   spmm_transpose (sparse_matrix.hpp:208-240) runs the SAME kernel on the
//   transposed CSR built at load, so A^T * Y is a gather with no atomics.
//
// One warp owns one output row slice of up to 64*NCH columns; lane j holds
// columns {64*ch + 2*j, +1} (double2). Each nonzero gathers one contiguous
// l*8-byte row of X (coalesced 512-byte warp loads), and the accumulation of
// every output entry is the reference's order: a sequential sum over the row's
// nonzeros in CSR order (rows split into chunks for load balance are summed
// per chunk, then the chunk partials are added in chunk order).
// Column ids / values are streamed once (evict-first); X rows go through L1/L2
// (read-only path) since power-law columns are re-gathered many times.
#include <cstdlib>

#include "internal.cuh"

namespace fb {
namespace {

constexpr int kThreads = 256;

double env_double(const char* name, double dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atof(e) : dflt;
}

template <int VEC>
struct Vec;
template <>
struct Vec<2> {
    using T = double2;
    __device__ static T load(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
    __device__ static T load_pol(const double* p, uint64_t pol) {
        T r;
        asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
        return r;
    }
    __device__ static void fma(T& a, double v, const T& x) {
        a.x = __fma_rn(v, x.x, a.x);
        a.y = __fma_rn(v, x.y, a.y);
    }
    // outputs and partials are not re-read by this kernel: streaming stores
    // keep them from evicting the gathered operand's rows from L2
    __device__ static void store(double* p, const T& a) { __stcs(reinterpret_cast<double2*>(p), a); }
    __device__ static T zero() { return make_double2(0.0, 0.0); }
};
template <>
struct Vec<1> {
    using T = double;
    __device__ static T load(const double* p) { return __ldg(p); }
    __device__ static T load_pol(const double* p, uint64_t pol) {
        T r;
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
        return r;
    }
    __device__ static void fma(T& a, double v, const T& x) { a = __fma_rn(v, x, a); }
    __device__ static void store(double* p, const T& a) { __stcs(p, a); }
    __device__ static T zero() { return 0.0; }
};

// L2 policies of MODE_HINT (evict_last for the hinted X rows, evict_first
// for the others).
struct Hot {
    uint64_t keep, stream;
};

// Gather modes: plain ids; ids whose sign bit marks an L2-hot X row
// (DCsr::hint_h): hot rows are loaded with an evict_last policy, the others
// evict_first, so the rare rows streamed from HBM do not push the popular rows
// out of L2.
constexpr int MODE_PLAIN = 0, MODE_HINT = 2;

__device__ __forceinline__ void make_policies(Hot& h) {
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(h.keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(h.stream));
}

template <int VEC, int NCH, int MODE>
__device__ __forceinline__ void gather(typename Vec<VEC>::T (&x)[NCH], int c, const double* __restrict__ Xl,
                                       int64_t ldx, const bool (&ok)[NCH], int lane, int ncols,
                                       const Hot& hot) {
    using V = Vec<VEC>;
    using T = typename V::T;
    if (MODE == MODE_HINT) {
        const uint64_t pol = c < 0 ? hot.keep : hot.stream;
        const double* src = Xl + int64_t(c & 0x7fffffff) * ldx;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) x[ch] = ok[ch] ? V::load_pol(src + ch * 32 * VEC, pol) : V::zero();
        return;
    }
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
        x[ch] = ok[ch] ? V::load(Xl + int64_t(c) * ldx + ch * 32 * VEC) : V::zero();
}

template <int VEC, int NCH, int MODE>
__device__ __forceinline__ void row_accumulate(const int32_t* __restrict__ col,
                                               const double* __restrict__ val, int64_t p0, int64_t p1,
                                               const double* __restrict__ X, int64_t ldx,
                                               int lane, int ncols, const Hot& hot,
                                               typename Vec<VEC>::T (&acc)[NCH]) {
    using V = Vec<VEC>;
    using T = typename V::T;
    bool ok[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) ok[ch] = (ch * 32 + lane) * VEC < ncols;
    const double* Xl = X + lane * VEC;
    for (int64_t base = p0; base < p1; base += 32) {
        const int cnt = (p1 - base) < 32 ? int(p1 - base) : 32;
        int myc = 0;
        double myv = 0.0;
        if (lane < cnt) {
            myc = __ldcs(col + base + lane);
            myv = __ldcs(val + base + lane);
        }
        int j = 0;
        for (; j + 4 <= cnt; j += 4) {
            int c[4];
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                c[u] = __shfl_sync(0xffffffffu, myc, j + u);
                v[u] = __shfl_sync(0xffffffffu, myv, j + u);
            }
            T x[4][NCH];
#pragma unroll
            for (int u = 0; u < 4; ++u) gather<VEC, NCH, MODE>(x[u], c[u], Xl, ldx, ok, lane, ncols, hot);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) V::fma(acc[ch], v[u], x[u][ch]);
        }
        if (j < cnt) {
            // the last 1-3 nonzeros as one group with their loads in flight
            // together (a sequential tail would pay one round trip each); the
            // padding slots re-read a valid row with weight 0 and add exactly 0
            const int rem = cnt - j;
            int c[3];
            double v[3];
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int src = u < rem ? j + u : j;
                c[u] = __shfl_sync(0xffffffffu, myc, src);
                const double vv = __shfl_sync(0xffffffffu, myv, src);
                v[u] = u < rem ? vv : 0.0;
            }
            T x[3][NCH];
#pragma unroll
            for (int u = 0; u < 3; ++u) gather<VEC, NCH, MODE>(x[u], c[u], Xl, ldx, ok, lane, ncols, hot);
#pragma unroll
            for (int u = 0; u < 3; ++u)
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) V::fma(acc[ch], v[u], x[u][ch]);
        }
    }
}

template <int VEC, int NCH, int MODE>
__device__ __forceinline__ void spmm_items(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                           const double* __restrict__ val, const WorkItem* __restrict__ items,
                                           int64_t nitems, const double* __restrict__ X, int64_t ldx,
                                           double* __restrict__ Y, int64_t ldy, double* __restrict__ part,
                                           int ncols, const Hot& hot, const uint8_t* __restrict__ skip,
                                           int32_t* __restrict__ counter) {
    using V = Vec<VEC>;
    using T = typename V::T;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    // items are taken from a global counter when one is given (the skip list
    // of the panelled A^T*Y leaves many items nearly empty, so a static
    // stride leaves warps idle); which warp runs an item does not change its
    // arithmetic
    int64_t it = warp;
    if (counter) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        it = __shfl_sync(0xffffffffu, t, 0);
    }
    for (; it < nitems;) {
        const WorkItem w = items[it];
        if (w.r1 >= 0) {
            for (int32_t r = w.r0; r < w.r1; ++r) {
                if (skip && skip[r]) continue;  // served by the streaming path
                T acc[NCH];
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) acc[ch] = V::zero();
                row_accumulate<VEC, NCH, MODE>(col, val, rowptr[r], rowptr[r + 1], X, ldx, lane, ncols, hot, acc);
                double* yr = Y + int64_t(r) * ldy + lane * VEC;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
                    if ((ch * 32 + lane) * VEC < ncols) V::store(yr + ch * 32 * VEC, acc[ch]);
            }
        } else {
            T acc[NCH];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) acc[ch] = V::zero();
            row_accumulate<VEC, NCH, MODE>(col, val, w.p0, w.p1, X, ldx, lane, ncols, hot, acc);
            const int64_t slot = -int64_t(w.r1) - 1;
            double* pr = part + slot * ncols + lane * VEC;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
                if ((ch * 32 + lane) * VEC < ncols) V::store(pr + ch * 32 * VEC, acc[ch]);
        }
        if (counter) {
            int t = 0;
            if (lane == 0) t = atomicAdd(counter, 1);
            it = __shfl_sync(0xffffffffu, t, 0);
        } else {
            it += nwarps;
        }
    }
}

// Plain kernel (A^T * Y, and A * X over the full width).
template <int VEC, int NCH, int MODE>
__global__ void __launch_bounds__(kThreads, 4)
k_spmm(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
       const double* __restrict__ val, const WorkItem* __restrict__ items, int64_t nitems,
       const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy,
       double* __restrict__ part, int ncols, const uint8_t* __restrict__ skip, int32_t* __restrict__ counter) {
    Hot hot{0, 0};
    if (MODE == MODE_HINT) make_policies(hot);
    spmm_items<VEC, NCH, MODE>(rowptr, col, val, items, nitems, X, ldx, Y, ldy, part, ncols, hot, skip, counter);
}

// ---- Sliced A*X with shared-memory hot rows (k_spmm_sx) ---------------------
// For an X several times larger than L2: Y = A X runs in slices of 32
// columns. A slice of X (n x 32 doubles; 83 MB at C3) stays L2-resident while
// A streams through, so the gathers stop missing to HBM, and the X rows of the
// H most popular columns (A.sx_h, ids encoded kColHot | rank) come from a
// shared-memory copy made at kernel start (at C3 the top 640 columns hold ~30%
// of the nonzeros), so those gathers leave L2 alone. One lane per column:
// lane j accumulates Y(r, c0 + j) as the FMA chain over the row's nonzeros in
// CSR order -- per entry the same operations as the full-width kernel, so the
// two are bitwise equal (padding slots add fma(0, x, acc) == acc).
constexpr int kSxThreads = 1024;
constexpr int kSxW = 32;

__device__ __forceinline__ double sx_gather(int32_t e, const double* __restrict__ Xc, int64_t ldx,
                                            const double* __restrict__ Xs, int lane, bool ok) {
    if (e & kColHot) return Xs[(e & kRankMask) * kSxW + lane];  // warp-uniform
    return ok ? __ldg(Xc + int64_t(e) * ldx) : 0.0;
}

__device__ __forceinline__ double sx_row(const int32_t* __restrict__ col, const double* __restrict__ val, int64_t p0,
                                         int64_t p1, const double* __restrict__ Xc, int64_t ldx,
                                         const double* __restrict__ Xs, int lane, bool ok) {
    double acc = 0.0;
    for (int64_t base = p0; base < p1; base += 32) {
        const int cnt = (p1 - base) < 32 ? int(p1 - base) : 32;
        int myc = 0;
        double myv = 0.0;
        if (lane < cnt) {
            myc = __ldcs(col + base + lane);
            myv = __ldcs(val + base + lane);
        }
        for (int j = 0; j < cnt; j += 8) {
            // eight gathers in flight; past the end a slot re-reads the
            // group's first row with weight 0 (adds exactly 0)
            const int rem = cnt - j;
            double x[8], v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int src = u < rem ? j + u : j;
                const int32_t e = __shfl_sync(0xffffffffu, myc, src);
                const double vv = __shfl_sync(0xffffffffu, myv, src);
                v[u] = u < rem ? vv : 0.0;
                x[u] = sx_gather(e, Xc, ldx, Xs, lane, ok);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = __fma_rn(v[u], x[u], acc);
        }
    }
    return acc;
}

__global__ void __launch_bounds__(kSxThreads, 1)
k_spmm_sx(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, const double* __restrict__ val,
          const WorkItem* __restrict__ items, int64_t nitems, const double* __restrict__ X, int64_t ldx, int w,
          double* __restrict__ Y, int64_t ldy, double* __restrict__ part, const int32_t* __restrict__ rank_ids,
          int H, int32_t* __restrict__ counter) {
    extern __shared__ double Xs[];  // H x 32
    const int lane = threadIdx.x & 31;
    const bool ok = lane < w;
    for (int e = threadIdx.x; e < H * kSxW; e += blockDim.x) {
        const int r = e >> 5, j = e & 31;
        Xs[e] = j < w ? __ldg(X + int64_t(rank_ids[r]) * ldx + j) : 0.0;
    }
    __syncthreads();
    const double* Xc = X + lane;
    for (;;) {
        int it = 0;
        if (lane == 0) it = atomicAdd(counter, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems) break;
        const WorkItem wi = items[it];
        if (wi.r1 >= 0) {
            for (int32_t r = wi.r0; r < wi.r1; ++r) {
                const double acc = sx_row(col, val, rowptr[r], rowptr[r + 1], Xc, ldx, Xs, lane, ok);
                if (ok) __stcs(Y + int64_t(r) * ldy + lane, acc);
            }
        } else {
            const double acc = sx_row(col, val, wi.p0, wi.p1, Xc, ldx, Xs, lane, ok);
            if (ok) __stcs(part + (-int64_t(wi.r1) - 1) * w + lane, acc);
        }
    }
}

// ---- Ring-staged gathers (k_spmm_ring) ---------------------------------------
// The gather kernels are latency-bound (ncu at C3: 77% of issue stalls on the
// long scoreboard, DRAM and L2 both near 57%): a warp can keep only the few
// rows in flight that its registers hold. Here each warp owns a ring of R
// shared-memory slots; one lane per nonzero moves the X row into a slot with a
// 1-D bulk copy (cp.async.bulk, completing on the slot's mbarrier), so R rows
// stay in flight continuously without registers, and the warp consumes the
// slots in CSR order: per output entry the same FMA chain as k_spmm (bitwise
// equal).
constexpr int kRingWarps = 16;
constexpr int kRingSlots = 8;

__device__ __forceinline__ void ring_mbar_init(uint64_t* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(b))));
}
__device__ __forceinline__ void ring_wait(uint64_t* b, unsigned parity) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
    asm volatile(
        "{\n .reg .pred p;\n"
        "RW: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra RW;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}
// expect the row's bytes on the slot barrier and start its copy
__device__ __forceinline__ void ring_issue(double* slot, uint64_t* bar, const double* src, unsigned bytes,
                                           uint64_t pol) {
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            static_cast<unsigned>(__cvta_generic_to_shared(slot))),
        "l"(src), "r"(bytes), "r"(b), "l"(pol)
        : "memory");
}

template <int NCH, int MODE>
__global__ void __launch_bounds__(kRingWarps * 32, 1)
k_spmm_ring(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, const double* __restrict__ val,
            const WorkItem* __restrict__ items, int64_t nitems, const double* __restrict__ X, int64_t ldx,
            double* __restrict__ Y, int64_t ldy, double* __restrict__ part, int ncols, int32_t* __restrict__ counter,
            int stride) {
    using V = Vec<2>;
    using T = V::T;
    extern __shared__ __align__(128) double ring_sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* ring = ring_sm + size_t(warp) * kRingSlots * stride;
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring_sm + size_t(kRingWarps) * kRingSlots * stride) + warp * kRingSlots;
    if (lane < kRingSlots) ring_mbar_init(bars + lane);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    Hot hot{0, 0};
    if (MODE == MODE_HINT) make_policies(hot);
    const unsigned bytes = unsigned(ncols) * 8u;
    bool ok[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) ok[ch] = (ch * 32 + lane) * 2 < ncols;
    // nonzero q -> its X row and L2 policy
    auto src_of = [&](int32_t cc, uint64_t& pol) {
        pol = (MODE == MODE_HINT && cc < 0) ? hot.keep : hot.stream;
        return X + int64_t(cc & 0x7fffffff) * ldx;
    };
    uint32_t gi = 0, gc = 0;  // running issue / consume counts: slot g % R, parity (g / R) & 1
    for (;;) {
        int it = 0;
        if (lane == 0) it = atomicAdd(counter, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems) break;
        const WorkItem w = items[it];
        const bool chunk = w.r1 < 0;
        const int64_t P0 = chunk ? w.p0 : rowptr[w.r0], P1 = chunk ? w.p1 : rowptr[w.r1];
        // first R nonzeros in flight, one lane each
        int64_t qi = P0;
        {
            const int n = int(min(int64_t(kRingSlots), P1 - P0));
            if (lane < n) {
                uint64_t pol;
                const double* src = src_of(__ldcs(col + P0 + lane), pol);
                const int slot = int((gi + lane) % kRingSlots);
                ring_issue(ring + slot * stride, bars + slot, src, bytes, pol);
            }
            qi += n;
            gi += n;
        }
        // ids of the next nonzeros to issue, 32 at a time
        int64_t cbase = qi;
        int32_t myc = (qi + lane < P1) ? __ldcs(col + qi + lane) : 0;
        int64_t vbase = P0;
        double myv = (P0 + lane < P1) ? __ldcs(val + P0 + lane) : 0.0;
        int32_t r = w.r0;
        int64_t rend = chunk ? P1 : rowptr[r + 1];
        T acc[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) acc[ch] = V::zero();
        for (int64_t qc = P0; qc < P1; ++qc) {
            while (!chunk && qc == rend) {  // rows that end here (empty rows too)
                double* yr = Y + int64_t(r) * ldy + lane * 2;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    if (ok[ch]) V::store(yr + ch * 64, acc[ch]);
                    acc[ch] = V::zero();
                }
                ++r;
                rend = rowptr[r + 1];
            }
            if (qc - vbase >= 32) {
                vbase = qc;
                myv = (qc + lane < P1) ? __ldcs(val + qc + lane) : 0.0;
            }
            const double v = __shfl_sync(0xffffffffu, myv, int(qc - vbase));
            const int slot = int(gc % kRingSlots);
            ring_wait(bars + slot, (gc / kRingSlots) & 1u);
            const double* xs = ring + slot * stride + lane * 2;
            T x[NCH];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) x[ch] = ok[ch] ? *reinterpret_cast<const T*>(xs + ch * 64) : V::zero();
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) V::fma(acc[ch], v, x[ch]);
            ++gc;
            __syncwarp();  // every lane has read the slot before it is refilled
            if (qi < P1) {
                if (qi - cbase >= 32) {
                    cbase = qi;
                    myc = (qi + lane < P1) ? __ldcs(col + qi + lane) : 0;
                }
                if (lane == int(qi - cbase)) {
                    uint64_t pol;
                    const double* src = src_of(myc, pol);
                    ring_issue(ring + slot * stride, bars + slot, src, bytes, pol);  // gi % R == slot
                }
                ++qi;
                ++gi;
            }
        }
        if (chunk) {
            double* pr = part + (-int64_t(w.r1) - 1) * ncols + lane * 2;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
                if (ok[ch]) V::store(pr + ch * 64, acc[ch]);
        } else {
            for (; r < w.r1; ++r) {  // the item's last rows (and empty rows after them)
                double* yr = Y + int64_t(r) * ldy + lane * 2;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    if (ok[ch]) V::store(yr + ch * 64, acc[ch]);
                    acc[ch] = V::zero();
                }
            }
        }
    }
}

// Long rows: Y[row] = sum of its chunk partials in a fixed order. One CTA per
// long row; warp w sums the w-th contiguous eighth of the row's chunks
// sequentially (loads unrolled), then the eight warp sums are added in warp
// order -- deterministic, and short enough that no single warp walks the
// hundreds of partials of a Zipf-head column alone.
constexpr int kCombWarps = 8;
__global__ void __launch_bounds__(kCombWarps * 32)
k_combine(const Combine* __restrict__ comb, const double* __restrict__ part, int ncols,
          double* __restrict__ Y, int64_t ldy) {
    __shared__ double red[kCombWarps][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Combine cb = comb[blockIdx.x];
    const int ns = cb.s1 - cb.s0;
    const int per = (ns + kCombWarps - 1) / kCombWarps;
    const int s0 = cb.s0 + min(ns, warp * per), s1 = cb.s0 + min(ns, (warp + 1) * per);
    for (int cb0 = 0; cb0 < ncols; cb0 += 256) {
        for (int c = cb0 + lane; c < min(ncols, cb0 + 256); c += 32) {
            double acc = 0.0;
            int s = s0;
            for (; s + 4 <= s1; s += 4) {
                const double a0 = part[int64_t(s) * ncols + c], a1 = part[int64_t(s + 1) * ncols + c];
                const double a2 = part[int64_t(s + 2) * ncols + c], a3 = part[int64_t(s + 3) * ncols + c];
                acc += a0; acc += a1; acc += a2; acc += a3;
            }
            for (; s < s1; ++s) acc += part[int64_t(s) * ncols + c];
            red[warp][c - cb0] = acc;
        }
        __syncthreads();
        for (int c = cb0 + threadIdx.x; c < min(ncols, cb0 + 256); c += blockDim.x) {
            double acc = red[0][c - cb0];
            for (int w = 1; w < kCombWarps; ++w) acc += red[w][c - cb0];
            Y[int64_t(cb.row) * ldy + c] = acc;
        }
        __syncthreads();
    }
}

// Even widths: the same partition and summation order as k_combine (bitwise
// equal), with each lane owning column pairs {64 ch + 2 lane, +1} (double2)
// and two slots' rows in flight per step, so a warp streams whole 8 l-byte
// partial rows instead of one 256-byte column strip at a time.
template <int NCH>
__global__ void __launch_bounds__(kCombWarps * 32)
k_combine2(const Combine* __restrict__ comb, const double* __restrict__ part, int ncols,
           double* __restrict__ Y, int64_t ldy) {
    __shared__ double2 red[kCombWarps][NCH * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Combine cb = comb[blockIdx.x];
    const int ns = cb.s1 - cb.s0;
    const int per = (ns + kCombWarps - 1) / kCombWarps;
    const int s0 = cb.s0 + min(ns, warp * per), s1 = cb.s0 + min(ns, (warp + 1) * per);
    bool ok[NCH];
    double2 acc[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        ok[ch] = 64 * ch + 2 * lane < ncols;
        acc[ch] = make_double2(0.0, 0.0);
    }
    const double* pl = part + 2 * lane;
    int s = s0;
    for (; s + 2 <= s1; s += 2) {
        double2 a[NCH], b[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const double2* pa = reinterpret_cast<const double2*>(pl + int64_t(s) * ncols + 64 * ch);
            const double2* pb = reinterpret_cast<const double2*>(pl + int64_t(s + 1) * ncols + 64 * ch);
            a[ch] = ok[ch] ? __ldcs(pa) : make_double2(0.0, 0.0);
            b[ch] = ok[ch] ? __ldcs(pb) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            acc[ch].x += a[ch].x; acc[ch].y += a[ch].y;
            acc[ch].x += b[ch].x; acc[ch].y += b[ch].y;
        }
    }
    if (s < s1) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
            if (ok[ch]) {
                const double2* pa = reinterpret_cast<const double2*>(pl + int64_t(s) * ncols + 64 * ch);
                const double2 a = __ldcs(pa);
                acc[ch].x += a.x; acc[ch].y += a.y;
            }
    }
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) red[warp][ch * 32 + lane] = acc[ch];
    __syncthreads();
    for (int e = threadIdx.x; e < NCH * 32; e += kCombWarps * 32) {
        const int c = 64 * (e >> 5) + 2 * (e & 31);
        if (c >= ncols) continue;
        double2 r = red[0][e];
        for (int w = 1; w < kCombWarps; ++w) {
            r.x += red[w][e].x;
            r.y += red[w][e].y;
        }
        *reinterpret_cast<double2*>(Y + int64_t(cb.row) * ldy + c) = r;
    }
}

// Panel chunks of A^T*Y (PanelPlan): every item is a chunk of one hot row
// inside one panel, summed sequentially into its partial slot. Items are taken
// in list (= panel-major) order through a global counter, so the resident
// warps all work on about one panel of the gathered operand at a time.
template <int NCH>
__global__ void __launch_bounds__(kThreads, 4)
k_spmm_panels(const int32_t* __restrict__ col, const double* __restrict__ val,
              const WorkItem* __restrict__ items, int64_t nitems, const double* __restrict__ X, int64_t ldx,
              double* __restrict__ part, int ncols, int32_t* __restrict__ counter) {
    using V = Vec<2>;
    using T = V::T;
    const int lane = threadIdx.x & 31;
    const Hot hot{0, 0};
    for (;;) {
        int it = 0;
        if (lane == 0) it = atomicAdd(counter, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems) break;
        const WorkItem w = items[it];
        T acc[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) acc[ch] = V::zero();
        row_accumulate<2, NCH, MODE_PLAIN>(col, val, w.p0, w.p1, X, ldx, lane, ncols, hot, acc);
        double* pr = part + (-int64_t(w.r1) - 1) * ncols + lane * 2;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
            if ((ch * 32 + lane) * 2 < ncols) V::store(pr + ch * 64, acc[ch]);
    }
}

// Non-owning view of a work list, or of one of its chunks (ItemList::cut_*)
struct Items {
    const WorkItem* items;
    int64_t nitems;
    const Combine* comb;
    int64_t ncomb, nslots;
    bool main;  // A's own list (carries the L2-hint ids)
    Items(const ItemList& L, bool main_list) : Items(L, main_list, -1) {}
    Items(const ItemList& L, bool main_list, int k) : main(main_list) {
        const int64_t i0 = k < 0 ? 0 : L.cut_item[size_t(k)], i1 = k < 0 ? L.nitems : L.cut_item[size_t(k) + 1];
        const int64_t c0 = k < 0 ? 0 : L.cut_comb[size_t(k)], c1 = k < 0 ? L.ncomb : L.cut_comb[size_t(k) + 1];
        items = L.items.get() + i0;
        nitems = i1 - i0;
        comb = L.comb.get() + c0;
        ncomb = c1 - c0;
        nslots = L.nslots;
    }
};

template <int VEC, int NCH, int MODE>
void launch_plain(Ctx& c, const DCsr& A, const Items& L, const uint8_t* skip, const double* X, int64_t ldx,
                  double* Y, int64_t ldy, double* part, int ncols) {
    if (!L.nitems) return;
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
        FB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_spmm<VEC, NCH, MODE>,
                                                              kThreads, 0));
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    int grid = int(std::min<int64_t>(int64_t(c.num_sms) * blocks_per_sm, (L.nitems + 7) / 8));
    grid = std::max(grid, 1);
    // Items come from a global counter (FRPCA_SPMM_DYNAMIC=1, the default;
    // 2 = only the cold list of the panelled A^T*Y, 0 = static stride).
    // Measured per run against the static stride: C1 17.85 -> 17.26 ms,
    // C2 80.8 -> 74.8, C3 228.8 -> 211.7, C4 354 -> 343 (tools/ab_env.py)
    const int dyn = int(env_double("FRPCA_SPMM_DYNAMIC", 1.0));
    int32_t* counter = nullptr;
    if (dyn == 1 || (dyn == 2 && skip)) {
        if (!c.wcount.get()) c.wcount.alloc(2, c.stream);
        counter = c.wcount.get() + (c.stream == c.aux ? 1 : 0);
        FB_CUDA(cudaMemsetAsync(counter, 0, sizeof(int32_t), c.stream));
    }
    k_spmm<VEC, NCH, MODE><<<grid, kThreads, 0, c.stream>>>(A.rowptr.get(), A.col.get(), A.val.get(),
                                                           L.items, L.nitems, X, ldx, Y, ldy, part,
                                                           ncols, skip, counter);
    FB_LAUNCH_CHECK();
}

// Ring kernel for a list without skipped rows (FRPCA_SPMM_RING=0/1); rows of
// X must be 16-byte multiples at 16-byte aligned addresses (bulk copies)
template <int NCH, int MODE>
bool launch_ring(Ctx& c, const DCsr& A, const Items& L, const double* X, int64_t ldx, double* Y, int64_t ldy,
                 double* part, int ncols) {
    if (int(env_double("FRPCA_SPMM_RING", 0.0)) == 0) return false;  // opt-in: measured slower
    if (ncols % 2 || ldx % 2 || (reinterpret_cast<uintptr_t>(X) % 16)) return false;
    const int stride = (ncols + 1) / 2 * 2;  // doubles per slot (16-byte multiple)
    const size_t smem = sizeof(double) * size_t(kRingWarps) * kRingSlots * stride +
                        sizeof(uint64_t) * kRingWarps * kRingSlots;
    if (smem > 227 * 1024) return false;
    smem_optin(k_spmm_ring<NCH, MODE>, smem);
    if (!c.wcount.get()) c.wcount.alloc(2, c.stream);
    int32_t* counter = c.wcount.get() + (c.stream == c.aux ? 1 : 0);
    FB_CUDA(cudaMemsetAsync(counter, 0, sizeof(int32_t), c.stream));
    k_spmm_ring<NCH, MODE><<<c.num_sms, kRingWarps * 32, smem, c.stream>>>(
        A.rowptr.get(), A.col.get(), A.val.get(), L.items, L.nitems, X, ldx, Y, ldy, part, ncols, counter,
        stride);
    FB_LAUNCH_CHECK();
    return true;
}

template <int VEC, int NCH>
void launch(Ctx& c, const DCsr& A, const Items& L, const uint8_t* skip, const double* X, int64_t ldx,
            double* Y, int64_t ldy, double* part, int ncols) {
    const bool hint = A.hint_h > 0 && L.main;
    if (VEC == 2 && !skip && L.nitems) {
        const bool done = hint ? launch_ring<NCH, MODE_HINT>(c, A, L, X, ldx, Y, ldy, part, ncols)
                               : launch_ring<NCH, MODE_PLAIN>(c, A, L, X, ldx, Y, ldy, part, ncols);
        if (done) return;
    }
    if (hint) return launch_plain<VEC, NCH, MODE_HINT>(c, A, L, skip, X, ldx, Y, ldy, part, ncols);
    launch_plain<VEC, NCH, MODE_PLAIN>(c, A, L, skip, X, ldx, Y, ldy, part, ncols);
}

void combine(Ctx& c, const Items& L, const double* part, int nc, double* Y, int64_t ldy) {
    if (!L.ncomb) return;
    // k_combine2 wins when rows have few partials (C4's A^T*Y: 11 per row,
    // 11.2 -> 6.0 ms per run) and loses with many (C1: 49 per row, 0.45 ->
    // 0.61 ms; C3: 636, 3.7 -> 4.1 ms), so it is chosen by the mean
    const char* e = std::getenv("FRPCA_COMBINE1");  // tests force either kernel
    const bool few = L.nslots <= 16 * L.ncomb || (e && e[0] == '2');
    if (nc % 2 == 0 && ldy % 2 == 0 && reinterpret_cast<uintptr_t>(Y) % 16 == 0 && few && !(e && e[0] == '1')) {
        const unsigned g = unsigned(L.ncomb);
        auto go = [&](auto k1, auto k2, auto k3, auto k4) {
            switch ((nc + 63) / 64) {
                case 1: k1<<<g, kCombWarps * 32, 0, c.stream>>>(L.comb, part, nc, Y, ldy); break;
                case 2: k2<<<g, kCombWarps * 32, 0, c.stream>>>(L.comb, part, nc, Y, ldy); break;
                case 3: k3<<<g, kCombWarps * 32, 0, c.stream>>>(L.comb, part, nc, Y, ldy); break;
                default: k4<<<g, kCombWarps * 32, 0, c.stream>>>(L.comb, part, nc, Y, ldy); break;
            }
        };
        go(k_combine2<1>, k_combine2<2>, k_combine2<3>, k_combine2<4>);
        FB_LAUNCH_CHECK();
        return;
    }
    k_combine<<<unsigned(L.ncomb), kCombWarps * 32, 0, c.stream>>>(L.comb, part, nc, Y, ldy);
    FB_LAUNCH_CHECK();
}

// One slice of <= 256 columns over the work list L (rows with skip[r] left
// out), then the fixed-order combine of its long rows.
void spmm_list(Ctx& c, const DCsr& A, const Items& L, const uint8_t* skip, const double* X, int64_t ldx,
               int nc, double* Y, int64_t ldy, double* part) {
    const bool v2 = (nc % 2 == 0) && (ldx % 2 == 0) && (ldy % 2 == 0) &&
                    (reinterpret_cast<uintptr_t>(X) % 16 == 0) && (reinterpret_cast<uintptr_t>(Y) % 16 == 0);
    if (v2) {
        switch ((nc + 63) / 64) {
            case 1: launch<2, 1>(c, A, L, skip, X, ldx, Y, ldy, part, nc); break;
            case 2: launch<2, 2>(c, A, L, skip, X, ldx, Y, ldy, part, nc); break;
            case 3: launch<2, 3>(c, A, L, skip, X, ldx, Y, ldy, part, nc); break;
            default: launch<2, 4>(c, A, L, skip, X, ldx, Y, ldy, part, nc); break;
        }
        combine(c, L, part, nc, Y, ldy);
        return;
    }
    // scalar path (odd widths): slices of <= 128 columns
    for (int o = 0; o < nc; o += 128) {
        const int w = std::min(128, nc - o);
        const int nch = (w + 31) / 32;
        if (nch <= 1) launch<1, 1>(c, A, L, skip, X + o, ldx, Y + o, ldy, part, w);
        else if (nch <= 2) launch<1, 2>(c, A, L, skip, X + o, ldx, Y + o, ldy, part, w);
        else launch<1, 4>(c, A, L, skip, X + o, ldx, Y + o, ldy, part, w);
        combine(c, L, part, w, Y + o, ldy);
    }
}

void launch_panels(Ctx& c, const DCsr& T, const double* Y, int64_t ldy, double* part, int nc) {
    const PanelPlan& P = T.pan;
    FB_CUDA(cudaMemsetAsync(P.counter.get(), 0, sizeof(int32_t), c.stream));
    const int grid = c.num_sms * 4;
    auto go = [&](auto kern) {
        kern<<<grid, kThreads, 0, c.stream>>>(T.col.get(), T.val.get(), P.hot.items.get(), P.hot.nitems, Y, ldy,
                                              part, nc, P.counter.get());
        FB_LAUNCH_CHECK();
    };
    switch ((nc + 63) / 64) {
        case 1: go(k_spmm_panels<1>); break;
        case 2: go(k_spmm_panels<2>); break;
        case 3: go(k_spmm_panels<3>); break;
        default: go(k_spmm_panels<4>); break;
    }
}

// Opt-in (FRPCA_SPMM_SX=1; FRPCA_SX_KB sets the shared memory given to hot
// rows, default 160 KB: 640 rows). Measured slower than the full-width kernel
// at every config (per run: C1 17.1 -> 23.3 ms, C2 72.3 -> 118.9, C3 208 ->
// 361; profiles/r2_ab_spmm_sx.json): re-streaming A's ids and values once per
// slice and the 256-byte gathers cost more than the L2 misses they remove.
bool use_sx(const Ctx& c, const DCsr& A, int64_t ncols) {
    (void)c;
    (void)ncols;
    return int(env_double("FRPCA_SPMM_SX", 0.0)) == 1 && A.rank_of.n > 0;
}

void spmm_sx(Ctx& c, DCsr& A, const double* X, int64_t ldx, int64_t ncols, double* Y, int64_t ldy) {
    const int64_t budget = int64_t(env_double("FRPCA_SX_KB", 160.0) * 1024.0);
    const int H = int(std::min<int64_t>(A.cols, std::max<int64_t>(0, budget / (8 * kSxW))));
    ensure_encoding(c, A, 0, H);
    const size_t smem = sizeof(double) * size_t(H) * kSxW;
    smem_optin(k_spmm_sx, std::max<size_t>(smem, 48 * 1024));
    if (!c.wcount.get()) c.wcount.alloc(2, c.stream);
    int32_t* counter = c.wcount.get() + (c.stream == c.aux ? 1 : 0);
    DBuf<double> part;
    if (A.L.nslots) part.alloc(size_t(A.L.nslots) * kSxW, c.stream);
    for (int64_t c0 = 0; c0 < ncols; c0 += kSxW) {
        const int w = int(std::min<int64_t>(kSxW, ncols - c0));
        FB_CUDA(cudaMemsetAsync(counter, 0, sizeof(int32_t), c.stream));
        k_spmm_sx<<<c.num_sms, kSxThreads, smem, c.stream>>>(A.rowptr.get(), A.col.get(), A.val.get(),
                                                             A.L.items.get(), A.L.nitems, X + c0, ldx, w, Y + c0,
                                                             ldy, part.get(), A.rank_ids.get(), H, counter);
        FB_LAUNCH_CHECK();
        combine(c, Items(A.L, true), part.get(), w, Y + c0, ldy);
    }
}

}  // namespace

void spmm_device(Ctx& c, const DCsr& A, const double* X, int64_t ldx, int64_t ncols, double* Y,
                 int64_t ldy, const char* tag) {
    if (A.rows == 0 || ncols == 0) return;
    // algorithmic bytes: 12 B/nnz + 8 B/row ptr + dense in + out
    const double bytes = 12.0 * A.nnz + 8.0 * (A.rows + 1) + 8.0 * ncols * (A.cols + A.rows);
    const double flops = 2.0 * A.nnz * ncols;
    Prof prof(c, tag, bytes, flops);
    DCsr& Am = const_cast<DCsr&>(A);
    if (Am.pend && !Am.pend->need.empty() && ncols <= 256 && !use_sx(c, A, ncols)) {
        // the values are still landing (pipelined upload): item chunk k starts
        // as soon as the values of its rows are on the device
        std::shared_ptr<PendingValues> pv = std::move(Am.pend);
        ensure_hint(c, Am, ncols);
        DBuf<double> part;
        if (A.L.nslots) part.alloc(size_t(A.L.nslots) * ncols, c.stream);
        // Item chunks alternate between the main and the aux stream (their
        // own work counters; disjoint output rows and partial slots), so a
        // chunk's blocks fill the SMs the previous chunk's tail frees (an
        // item of a long row runs for milliseconds); the main stream joins.
        if (!c.aux) {
            FB_CUDA(cudaStreamCreateWithFlags(&c.aux, cudaStreamNonBlocking));
            FB_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
            FB_CUDA(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
        }
        const cudaStream_t s0 = c.stream;
        // (only where a chunk is ONE launch over its own partial slots: the
        // scalar path of an odd or unaligned width runs slices of <= 128
        // columns that re-use the partial buffer at another stride, so two
        // chunks in flight on two streams overwrote each other's partials --
        // odd l > 128 through frpca_run_csr, found by the randomised sweep)
        const bool one_launch = ncols <= 128 || (ncols % 2 == 0 && ldx % 2 == 0 && ldy % 2 == 0 &&
                                                 reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
                                                 reinterpret_cast<uintptr_t>(Y) % 16 == 0);
        const bool alt = env_double("FRPCA_PIPE_ALT", 1.0) != 0.0 && one_launch;
        FB_CUDA(cudaEventRecord(c.ev_fork, s0));
        FB_CUDA(cudaStreamWaitEvent(c.aux, c.ev_fork, 0));
        for (size_t k = 0; k + 1 < A.L.cut_row.size(); ++k) {
            c.stream = (alt && (k & 1)) ? c.aux : s0;
            FB_CUDA(cudaStreamWaitEvent(c.stream, pv->ev[size_t(pv->need[k])], 0));
            spmm_list(c, A, Items(A.L, true, int(k)), nullptr, X, ldx, int(ncols), Y, ldy, part.get());
        }
        c.stream = s0;
        FB_CUDA(cudaEventRecord(c.ev_join, c.aux));
        FB_CUDA(cudaStreamWaitEvent(s0, c.ev_join, 0));
        part.s = s0;  // (freed behind the join)
        return;
    }
    consume_pending(c, Am);
    if (use_sx(c, A, ncols)) return spmm_sx(c, Am, X, ldx, ncols, Y, ldy);
    ensure_hint(c, Am, std::min<int64_t>(ncols, 256));
    DBuf<double> part;
    for (int64_t off = 0; off < ncols; off += 256) {
        const int nc = int(std::min<int64_t>(256, ncols - off));
        if (A.L.nslots && part.n < size_t(A.L.nslots) * nc) part.alloc(size_t(A.L.nslots) * nc, c.stream);
        spmm_list(c, A, Items(A.L, true), nullptr, X + off, ldx, nc, Y + off, ldy, part.get());
    }
}

// Z = A^T Y on the transposed CSR T. When Y (T.cols x l) is several times
// larger than a panel, the hot rows of T run through the panel plan first
// (chunks panel-major + combine), then the cold rows through their own list.
bool panel_rows_for(const DCsr& T, int64_t ncols, int64_t& pr, int64_t& cap) {
    const int64_t w = std::min<int64_t>(ncols, 256);
    const double panel_bytes = env_double("FRPCA_PANEL_MB", 32.0) * 1048576.0;
    const double min_bytes = env_double("FRPCA_PANEL_MIN_MB", 96.0) * 1048576.0;
    const bool use = ncols % 2 == 0 && 8.0 * double(T.cols) * double(w) > min_bytes &&
                     env_double("FRPCA_NO_PANELS", 0.0) == 0.0;
    if (!use) return false;
    pr = std::max<int64_t>(1, int64_t(panel_bytes / (8.0 * double(w))));
    cap = int64_t(env_double("FRPCA_PANEL_PART_GB", 16.0) * 1073741824.0 / (8.0 * double(w)));
    return true;
}

void spmm_t_device(Ctx& c, DCsr& T, const double* Y, int64_t ncols, double* Z, const char* tag) {
    if (T.rows == 0 || ncols == 0) return;
    consume_pending(c, T);
    const int64_t w = std::min<int64_t>(ncols, 256);
    int64_t pr = 0, cap = 0;
    const bool use = panel_rows_for(T, ncols, pr, cap);
    if (use) ensure_panels(c, T, pr, cap);
    if (!use || T.pan.nhot == 0) return spmm_device(c, T, Y, ncols, ncols, Z, ncols, tag);
    const PanelPlan& P = T.pan;
    const double bytes = 12.0 * T.nnz + 8.0 * (T.rows + 1) + 8.0 * ncols * (T.cols + T.rows);
    Prof prof(c, tag, bytes, 2.0 * T.nnz * ncols);
    // The cold rows (disjoint output rows, their own partial slots) run on a
    // second stream beside the panel chunks and their combine, filling the
    // panel kernel's tail; the arithmetic is unchanged. It pays while Y is
    // a few times L2 (C1, Y 1.6 GB: 17.26 -> 17.05 ms per run) and costs
    // with larger Y (C2 6 GB: 74.8 -> 75.4, C3 20.6 GB: 211.7 -> 212.7; the
    // cold rows' HBM gathers evict panel rows), so by default it is on up to
    // 4 GB of Y (FRPCA_COLD_CONCURRENT=0/1 forces it)
    const double ybytes = 8.0 * double(T.cols) * double(w);
    const bool conc = env_double("FRPCA_COLD_CONCURRENT", ybytes <= 4.0 * 1073741824.0 ? 1.0 : 0.0) != 0.0 &&
                      P.cold.nitems > 0;
    const size_t slots = conc ? size_t(P.hot.nslots + P.cold.nslots) : size_t(std::max(P.hot.nslots, P.cold.nslots));
    // persistent with the plan: a per-call multi-GB allocation can remap pool
    // memory every run (measured: ~150 ms per call at C3)
    DBuf<double>& part = const_cast<PanelPlan&>(P).part;
    if (part.n < slots * size_t(w)) part.alloc(slots * size_t(w), c.stream);
    if (conc && !c.aux) {
        FB_CUDA(cudaStreamCreateWithFlags(&c.aux, cudaStreamNonBlocking));
        FB_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
        FB_CUDA(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
    }
    for (int64_t off = 0; off < ncols; off += 256) {
        const int nc = int(std::min<int64_t>(256, ncols - off));
        FB_CUDA(cudaMemsetAsync(P.counter.get(), 0, sizeof(int32_t), c.stream));
        if (conc) FB_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        {
            Prof ph(c, "spmm_AtY_panels", 0, 0);
            launch_panels(c, T, Y + off, ncols, part.get(), nc);
        }
        if (conc) {
            // queued after the panel kernel, so its CTAs take the SMs the
            // panel kernel's tail frees
            const cudaStream_t s0 = c.stream;
            FB_CUDA(cudaStreamWaitEvent(c.aux, c.ev_fork, 0));
            c.stream = c.aux;
            {
                Prof pd(c, "spmm_AtY_cold", 0, 0);
                spmm_list(c, T, Items(P.cold, false), P.skip.get(), Y + off, ncols, nc, Z + off, ncols,
                          part.get() + size_t(P.hot.nslots) * size_t(nc));
            }
            c.stream = s0;
            FB_CUDA(cudaEventRecord(c.ev_join, c.aux));
        }
        {
            Prof pc(c, "spmm_AtY_pcombine", 0, 0);
            combine(c, Items(P.hot, false), part.get(), nc, Z + off, ncols);
        }
        if (conc) {
            FB_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
            continue;
        }
        Prof pd(c, "spmm_AtY_cold", 0, 0);
        spmm_list(c, T, Items(P.cold, false), P.skip.get(), Y + off, ncols, nc, Z + off, ncols, part.get());
    }
}

// ---- products with the sharded sum overlapped -----------------
namespace {

// Hands finished row chunks of a row-major output (ld = ncols) to the
// collective on Ctx::comm_stream; finish() makes the main stream wait for the
// last sum.
struct ChunkReducer {
    Ctx& c;
    double* out;
    int64_t ld;
    std::vector<cudaEvent_t> evs;
    ChunkReducer(Ctx& ctx, double* o, int64_t l) : c(ctx), out(o), ld(l) {
        if (!c.comm_stream) FB_CUDA(cudaStreamCreateWithFlags(&c.comm_stream, cudaStreamNonBlocking));
    }
    void rows(int64_t r0, int64_t r1) {
        if (r1 <= r0) return;
        cudaEvent_t ev;
        FB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        evs.push_back(ev);
        FB_CUDA(cudaEventRecord(ev, c.stream));
        FB_CUDA(cudaStreamWaitEvent(c.comm_stream, ev, 0));
        c.coll->allreduce_sum(c, out + r0 * ld, (r1 - r0) * ld, c.comm_stream);
    }
    void finish() {
        cudaEvent_t ev;
        FB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        evs.push_back(ev);
        FB_CUDA(cudaEventRecord(ev, c.comm_stream));
        FB_CUDA(cudaStreamWaitEvent(c.stream, ev, 0));
    }
    ~ChunkReducer() {
        for (auto e : evs) cudaEventDestroy(e);  // (destroying a pending event is allowed)
    }
};

}  // namespace

void spmm_device_reduced(Ctx& c, const DCsr& A, const double* X, int64_t ncols, double* Y, const char* tag) {
    if (c.world <= 1 || ncols > 256 || A.L.cut_row.size() < 2 || A.rows == 0) {
        spmm_device(c, A, X, ncols, ncols, Y, ncols, tag);  // (starts on the values as they land)
        allreduce_sum(c, Y, A.rows * ncols);
        return;
    }
    consume_pending(c, const_cast<DCsr&>(A));
    const double bytes = 12.0 * A.nnz + 8.0 * (A.rows + 1) + 8.0 * ncols * (A.cols + A.rows);
    ChunkReducer red(c, Y, ncols);
    {
        Prof prof(c, tag, bytes, 2.0 * A.nnz * ncols);  // (the sums overlap this bracket)
        ensure_hint(c, const_cast<DCsr&>(A), ncols);
        DBuf<double> part;
        if (A.L.nslots) part.alloc(size_t(A.L.nslots) * ncols, c.stream);
        const int nchunks = int(A.L.cut_row.size()) - 1;
        for (int k = 0; k < nchunks; ++k) {
            spmm_list(c, A, Items(A.L, true, k), nullptr, X, ncols, int(ncols), Y, ncols, part.get());
            red.rows(A.L.cut_row[size_t(k)], A.L.cut_row[size_t(k) + 1]);
        }
    }
    red.finish();
}

void spmm_t_device_reduced(Ctx& c, DCsr& T, const double* Y, int64_t ncols, double* Z, const char* tag) {
    consume_pending(c, T);
    int64_t pr = 0, cap = 0;
    const bool pan = panel_rows_for(T, ncols, pr, cap);
    if (pan) ensure_panels(c, T, pr, cap);
    const ItemList& L = (pan && T.pan.nhot) ? T.pan.cold : T.L;
    if (c.world <= 1 || ncols > 256 || L.cut_row.size() < 2 || T.rows == 0) {
        spmm_t_device(c, T, Y, ncols, Z, tag);
        allreduce_sum(c, Z, T.rows * ncols);
        return;
    }
    const int nc = int(ncols);
    ChunkReducer red(c, Z, ncols);
    const int nchunks = int(L.cut_row.size()) - 1;
    {
        Prof prof(c, tag, 12.0 * T.nnz + 8.0 * (T.rows + 1) + 8.0 * ncols * (T.cols + T.rows), 2.0 * T.nnz * ncols);
        if (pan && T.pan.nhot) {
            // the hot rows (panel chunks + their combine) first, whole; then the
            // cold rows chunk by chunk: chunk k completes rows [cut k, cut k+1)
            const PanelPlan& P = T.pan;
            DBuf<double>& part = const_cast<PanelPlan&>(P).part;
            const size_t slots = size_t(std::max(P.hot.nslots, P.cold.nslots));
            if (part.n < slots * size_t(nc)) part.alloc(slots * size_t(nc), c.stream);
            launch_panels(c, T, Y, ncols, part.get(), nc);
            combine(c, Items(P.hot, false), part.get(), nc, Z, ncols);
            for (int k = 0; k < nchunks; ++k) {
                spmm_list(c, T, Items(P.cold, false, k), P.skip.get(), Y, ncols, nc, Z, ncols, part.get());
                red.rows(L.cut_row[size_t(k)], L.cut_row[size_t(k) + 1]);
            }
        } else {
            DBuf<double> part;
            if (T.L.nslots) part.alloc(size_t(T.L.nslots) * nc, c.stream);
            for (int k = 0; k < nchunks; ++k) {
                spmm_list(c, T, Items(T.L, true, k), nullptr, Y, ncols, nc, Z, ncols, part.get());
                red.rows(L.cut_row[size_t(k)], L.cut_row[size_t(k) + 1]);
            }
        }
    }
    red.finish();
}

}  // namespace fb
