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

template <int VEC>
struct Vec;
template <>
struct Vec<2> {
    using T = double2;
    __device__ static T load(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
    __device__ static void fma(T& a, double v, const T& x) {
        a.x = __fma_rn(v, x.x, a.x);
        a.y = __fma_rn(v, x.y, a.y);
    }
    __device__ static void store(double* p, const T& a) { *reinterpret_cast<double2*>(p) = a; }
    __device__ static T zero() { return make_double2(0.0, 0.0); }
};
template <>
struct Vec<1> {
    using T = double;
    __device__ static T load(const double* p) { return __ldg(p); }
    __device__ static void fma(T& a, double v, const T& x) { a = __fma_rn(v, x, a); }
    __device__ static void store(double* p, const T& a) { *p = a; }
    __device__ static T zero() { return 0.0; }
};

// Hot-column staging (A * X only): the most popular columns of A are encoded
// as -(rank+1); ranks below H are served from the CTA's shared copy Xs of
// those X rows, higher ranks are decoded through hot_cols and gathered from
// global memory like any other column.
struct Hot {
    const double* Xs;        // H x ncols in shared memory (nullptr when H == 0)
    int H;
    const int32_t* cols;     // rank -> original column id
};

template <int VEC, int NCH, bool HOT>
__device__ __forceinline__ void gather(typename Vec<VEC>::T (&x)[NCH], int c, const double* __restrict__ Xl,
                                       int64_t ldx, const bool (&ok)[NCH], int lane, int ncols,
                                       const Hot& hot) {
    using V = Vec<VEC>;
    using T = typename V::T;
    if (HOT) {
        // one generic pointer for both sources: shared copy or global row
        const double* src;
        if (c < 0) {
            const int slot = -c - 1;
            src = slot < hot.H ? hot.Xs + size_t(slot) * ncols + lane * VEC
                               : Xl + int64_t(__ldg(hot.cols + slot)) * ldx;
        } else {
            src = Xl + int64_t(c) * ldx;
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
            x[ch] = ok[ch] ? *reinterpret_cast<const T*>(src + ch * 32 * VEC) : V::zero();
        return;
    }
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
        x[ch] = ok[ch] ? V::load(Xl + int64_t(c) * ldx + ch * 32 * VEC) : V::zero();
}

template <int VEC, int NCH, bool HOT>
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
            for (int u = 0; u < 4; ++u) gather<VEC, NCH, HOT>(x[u], c[u], Xl, ldx, ok, lane, ncols, hot);
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
            for (int u = 0; u < 3; ++u) gather<VEC, NCH, HOT>(x[u], c[u], Xl, ldx, ok, lane, ncols, hot);
#pragma unroll
            for (int u = 0; u < 3; ++u)
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) V::fma(acc[ch], v[u], x[u][ch]);
        }
    }
}

template <int VEC, int NCH, bool HOT>
__device__ __forceinline__ void spmm_items(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                           const double* __restrict__ val, const WorkItem* __restrict__ items,
                                           int64_t nitems, const double* __restrict__ X, int64_t ldx,
                                           double* __restrict__ Y, int64_t ldy, double* __restrict__ part,
                                           int ncols, const Hot& hot, const uint8_t* __restrict__ skip) {
    using V = Vec<VEC>;
    using T = typename V::T;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t it = warp; it < nitems; it += nwarps) {
        const WorkItem w = items[it];
        if (w.r1 >= 0) {
            for (int32_t r = w.r0; r < w.r1; ++r) {
                if (skip && skip[r]) continue;  // served by the streaming path
                T acc[NCH];
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) acc[ch] = V::zero();
                row_accumulate<VEC, NCH, HOT>(col, val, rowptr[r], rowptr[r + 1], X, ldx, lane, ncols, hot, acc);
                double* yr = Y + int64_t(r) * ldy + lane * VEC;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
                    if ((ch * 32 + lane) * VEC < ncols) V::store(yr + ch * 32 * VEC, acc[ch]);
            }
        } else {
            T acc[NCH];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) acc[ch] = V::zero();
            row_accumulate<VEC, NCH, HOT>(col, val, w.p0, w.p1, X, ldx, lane, ncols, hot, acc);
            const int64_t slot = -int64_t(w.r1) - 1;
            double* pr = part + slot * ncols + lane * VEC;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
                if ((ch * 32 + lane) * VEC < ncols) V::store(pr + ch * 32 * VEC, acc[ch]);
        }
    }
}

// Plain kernel (A^T * Y, and A * X when no column is hot enough to stage).
// HOT = true here only decodes hot ids through the rank table (H = 0).
template <int VEC, int NCH, bool HOT>
__global__ void __launch_bounds__(kThreads, 4)
k_spmm(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
       const double* __restrict__ val, const WorkItem* __restrict__ items, int64_t nitems,
       const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy,
       double* __restrict__ part, int ncols, const int32_t* __restrict__ hot_cols,
       const uint8_t* __restrict__ skip) {
    const Hot hot{nullptr, 0, HOT ? hot_cols : nullptr};
    spmm_items<VEC, NCH, HOT>(rowptr, col, val, items, nitems, X, ldx, Y, ldy, part, ncols, hot, skip);
}

// A * X with the H most popular columns' X rows staged in shared memory: one
// 512-thread CTA per SM (16 resident warps; 128 registers keep the four
// in-flight nonzeros of every warp unspilled).
constexpr int kHotThreads = 512;
template <int NCH>
__global__ void __launch_bounds__(kHotThreads, 1)
k_spmm_hot(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
           const double* __restrict__ val, const WorkItem* __restrict__ items, int64_t nitems,
           const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy,
           double* __restrict__ part, int ncols, const int32_t* __restrict__ hot_cols, int H) {
    extern __shared__ __align__(16) double Xs[];
    const int half = ncols / 2;
    for (int e = threadIdx.x; e < H * half; e += blockDim.x) {
        const int r = e / half, c2 = e % half;
        reinterpret_cast<double2*>(Xs)[e] =
            __ldg(reinterpret_cast<const double2*>(X + int64_t(hot_cols[r]) * ldx) + c2);
    }
    __syncthreads();
    const Hot hot{Xs, H, hot_cols};
    spmm_items<2, NCH, true>(rowptr, col, val, items, nitems, X, ldx, Y, ldy, part, ncols, hot, nullptr);
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

template <int VEC, int NCH, bool HOT>
void launch_plain(Ctx& c, const DCsr& A, const double* X, int64_t ldx, double* Y, int64_t ldy,
                  double* part, int ncols) {
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
        FB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_spmm<VEC, NCH, HOT>,
                                                              kThreads, 0));
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    int grid = int(std::min<int64_t>(int64_t(c.num_sms) * blocks_per_sm, (A.nitems + 7) / 8));
    grid = std::max(grid, 1);
    k_spmm<VEC, NCH, HOT><<<grid, kThreads, 0, c.stream>>>(A.rowptr.get(), A.col.get(), A.val.get(),
                                                           A.items.get(), A.nitems, X, ldx, Y, ldy, part,
                                                           ncols, A.hot_cols.get(), A.skip.get());
    FB_LAUNCH_CHECK();
}

constexpr size_t kHotSmem = 200 * 1024;

template <int NCH>
void launch_hot(Ctx& c, const DCsr& A, const double* X, int64_t ldx, double* Y, int64_t ldy,
                double* part, int ncols) {
    const int H = int(std::min<int64_t>(A.nhot, int64_t(kHotSmem / (sizeof(double) * ncols))));
    static bool attr = false;
    if (!attr) {
        FB_CUDA(cudaFuncSetAttribute(k_spmm_hot<NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kHotSmem)));
        attr = true;
    }
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(c.num_sms, (A.nitems + 31) / 32)));
    k_spmm_hot<NCH><<<grid, kHotThreads, sizeof(double) * size_t(H) * ncols, c.stream>>>(
        A.rowptr.get(), A.col.get(), A.val.get(), A.items.get(), A.nitems, X, ldx, Y, ldy, part, ncols,
        A.hot_cols.get(), H);
    FB_LAUNCH_CHECK();
}

template <int VEC, int NCH>
void launch(Ctx& c, const DCsr& A, const double* X, int64_t ldx, double* Y, int64_t ldy,
            double* part, int ncols) {
    if (A.nhot == 0) return launch_plain<VEC, NCH, false>(c, A, X, ldx, Y, ldy, part, ncols);
    static const bool use_hot = [] {
        const char* e = std::getenv("FRPCA_HOT_STAGING");
        return e && e[0] == '1';
    }();
    if (use_hot && VEC == 2 && ncols % 2 == 0 && A.nitems >= 32 * c.num_sms)
        return launch_hot<NCH>(c, A, X, ldx, Y, ldy, part, ncols);
    launch_plain<VEC, NCH, true>(c, A, X, ldx, Y, ldy, part, ncols);
}

// ---------------------------------------------------------------------------
// A^T*Y for the kTop most popular columns of A by STREAMING Y: one CTA per SM
// walks a contiguous row range of A, stages Y's rows through shared memory
// (coalesced, each row read once) and accumulates, for every top entry
// (i, rank, v) of those rows, v * Y[i] into the rank's accumulator. Warp w
// owns ranks {w, w+16, w+32, w+48} in registers, so the accumulation of every
// output entry is in ascending row order within the CTA; the per-CTA partials
// are then added in CTA order (deterministic). This replaces nnz_top random
// 8*l-byte gathers of Y by one coalesced pass over Y.
constexpr int TOP_WARPS = 16;
constexpr int TOP_RB = 16;   // rows staged per batch

template <int NCH>
__global__ void __launch_bounds__(TOP_WARPS * 32, 1)
k_aty_top(const double* __restrict__ Y, int64_t ldy, int ncols, const int64_t* __restrict__ top_rp,
          const uint8_t* __restrict__ top_rank, const double* __restrict__ top_val,
          const int64_t* __restrict__ cuts, double* __restrict__ part) {
    extern __shared__ __align__(16) double Ys[];  // [2][TOP_RB][ncols]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = cuts[blockIdx.x], r1 = cuts[blockIdx.x + 1];
    double2 acc[4][NCH];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) acc[k][ch] = make_double2(0.0, 0.0);
    const int half = ncols / 2;
    auto stage_rows = [&](int buf, int64_t b0) {
        double* dst = Ys + size_t(buf) * TOP_RB * ncols;
        const int nrows = (r1 - b0) < TOP_RB ? int(r1 - b0) : TOP_RB;
        for (int e = tid; e < nrows * half; e += blockDim.x) {
            const int rr = e / half, c2 = e % half;
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + rr * ncols + 2 * c2));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                         "l"(Y + (b0 + rr) * ldy + 2 * c2));
        }
        asm volatile("cp.async.commit_group;\n");
    };
    if (r0 < r1) stage_rows(0, r0);
    int buf = 0;
    for (int64_t b0 = r0; b0 < r1; b0 += TOP_RB, buf ^= 1) {
        if (b0 + TOP_RB < r1) {
            stage_rows(buf ^ 1, b0 + TOP_RB);
            asm volatile("cp.async.wait_group 1;\n");
        } else {
            asm volatile("cp.async.wait_group 0;\n");
        }
        __syncthreads();
        const double* ys = Ys + size_t(buf) * TOP_RB * ncols + lane * 2;
        const int nrows = (r1 - b0) < TOP_RB ? int(r1 - b0) : TOP_RB;
        for (int rr = 0; rr < nrows; ++rr) {
            const int64_t p0 = top_rp[b0 + rr], p1 = top_rp[b0 + rr + 1];
            for (int64_t p = p0; p < p1; ++p) {
                const int rk = top_rank[p];
                if ((rk & (TOP_WARPS - 1)) != warp) continue;
                const double v = top_val[p];
                double2 y[NCH];
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
                    y[ch] = (ch * 32 + lane) * 2 < ncols
                                ? *reinterpret_cast<const double2*>(ys + rr * ncols + ch * 64)
                                : make_double2(0.0, 0.0);
                const int k = rk >> 4;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    if (kk == k)
#pragma unroll
                        for (int ch = 0; ch < NCH; ++ch) {
                            acc[kk][ch].x = __fma_rn(v, y[ch].x, acc[kk][ch].x);
                            acc[kk][ch].y = __fma_rn(v, y[ch].y, acc[kk][ch].y);
                        }
            }
        }
        __syncthreads();
    }
    // partial [cta][rank][ncols]
    double* out = part + size_t(blockIdx.x) * kTop * ncols;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        const int rk = kk * TOP_WARPS + warp;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
            if ((ch * 32 + lane) * 2 < ncols)
                *reinterpret_cast<double2*>(out + size_t(rk) * ncols + ch * 64 + lane * 2) = acc[kk][ch];
    }
}

// Z[top_cols[r]] = sum over CTAs (in order) of the partials
__global__ void k_top_combine(const double* __restrict__ part, int nparts, int ncols,
                              const int32_t* __restrict__ top_cols, double* __restrict__ Z, int64_t ldz) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kTop * ncols; e += gridDim.x * blockDim.x) {
        const int rk = e / ncols, c = e % ncols;
        double acc = 0.0;
        for (int g = 0; g < nparts; ++g) acc += part[size_t(g) * kTop * ncols + e];
        Z[int64_t(top_cols[rk]) * ldz + c] = acc;
    }
}

template <int NCH>
void launch_top(Ctx& c, const DCsr& A, const double* Y, int64_t ldy, int ncols, double* part) {
    const size_t smem = sizeof(double) * 2 * TOP_RB * size_t(ncols);
    static bool attr = false;
    if (!attr) {
        FB_CUDA(cudaFuncSetAttribute(k_aty_top<NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
        attr = true;
    }
    k_aty_top<NCH><<<A.ntop_cuts, TOP_WARPS * 32, smem, c.stream>>>(
        Y, ldy, ncols, A.top_rp.get(), A.top_rank.get(), A.top_val.get(), A.top_cuts.get(), part);
    FB_LAUNCH_CHECK();
}

}  // namespace

void combine(Ctx& c, const DCsr& A, const double* part, int nc, double* Y, int64_t ldy) {
    if (!A.ncombine) return;
    k_combine<<<unsigned(A.ncombine), kCombWarps * 32, 0, c.stream>>>(A.combine.get(), part, nc, Y, ldy);
    FB_LAUNCH_CHECK();
}

void spmm_device(Ctx& c, const DCsr& A, const double* X, int64_t ldx, int64_t ncols, double* Y,
                 int64_t ldy, const char* tag) {
    if (A.rows == 0 || ncols == 0) return;
    // algorithmic bytes: 12 B/nnz + 8 B/row ptr + dense in + out
    const double bytes = 12.0 * A.nnz + 8.0 * (A.rows + 1) + 8.0 * ncols * (A.cols + A.rows);
    const double flops = 2.0 * A.nnz * ncols;
    Prof prof(c, tag, bytes, flops);
    // L2-aware column slicing: when the gathered operand X (A.cols x ncols) is
    // only a few times larger than L2, gather it in column slices that fit
    // (each slice re-reads A's 12 B/nnz, but the 8*w-byte row gathers then hit
    // L2 instead of HBM). Slices are multiples of 64 columns.
    int64_t slice_max = 256;
    {
        const char* eb = std::getenv("FRPCA_SLICE_BUDGET_MB");
        const double budget = (eb ? std::atof(eb) : 80.0) * 1024 * 1024;
        const double xbytes = 8.0 * double(A.cols) * double(ncols);
        if (xbytes > budget && A.nnz > 8 * A.cols && std::getenv("FRPCA_SLICE")) {
            const int64_t w = int64_t(budget / (8.0 * double(A.cols))) / 64 * 64;
            if (w >= 64) slice_max = std::min<int64_t>(256, w);
        }
    }
    static const bool no_slice = [] {
        const char* e = std::getenv("FRPCA_NO_SLICE");
        return e && e[0] == '1';
    }();
    if (no_slice) slice_max = 256;
    DBuf<double> part;
    for (int64_t off = 0; off < ncols; off += slice_max) {
        const int nc = int(std::min<int64_t>(slice_max, ncols - off));
        if (A.nslots && part.n < size_t(A.nslots) * nc) part.alloc(size_t(A.nslots) * nc, c.stream);
        const bool v2 = (nc % 2 == 0) && (ldx % 2 == 0) && (ldy % 2 == 0) && (off % 2 == 0);
        const double* Xo = X + off;
        double* Yo = Y + off;
        if (v2) {
            const int nch = (nc + 63) / 64;
            switch (nch) {
                case 1: launch<2, 1>(c, A, Xo, ldx, Yo, ldy, part.get(), nc); break;
                case 2: launch<2, 2>(c, A, Xo, ldx, Yo, ldy, part.get(), nc); break;
                case 3: launch<2, 3>(c, A, Xo, ldx, Yo, ldy, part.get(), nc); break;
                default: launch<2, 4>(c, A, Xo, ldx, Yo, ldy, part.get(), nc); break;
            }
            combine(c, A, part.get(), nc, Yo, ldy);
        } else {
            // scalar path (odd widths): slices of <= 128 columns
            for (int o = 0; o < nc; o += 128) {
                const int w = std::min(128, nc - o);
                const int nch = (w + 31) / 32;
                if (nch <= 1) launch<1, 1>(c, A, Xo + o, ldx, Yo + o, ldy, part.get(), w);
                else if (nch <= 2) launch<1, 2>(c, A, Xo + o, ldx, Yo + o, ldy, part.get(), w);
                else launch<1, 4>(c, A, Xo + o, ldx, Yo + o, ldy, part.get(), w);
                combine(c, A, part.get(), w, Yo + o, ldy);
            }
        }
    }
}

void spmm_t_device(Ctx& c, const DCsr& A, const DCsr& T, const double* Y, int64_t ncols, double* Z,
                   const char* tag) {
    const bool stream = A.ntop > 0 && ncols % 2 == 0 && ncols <= 256 && ncols > 0;
    if (!stream) {
        // the gather kernel must not skip the top rows: run it on a view without the mask
        if (A.ntop > 0) {
            DCsr& Tm = const_cast<DCsr&>(T);
            DBuf<uint8_t> keep = std::move(Tm.skip);
            try {
                spmm_device(c, T, Y, ncols, ncols, Z, ncols, tag);
            } catch (...) {
                Tm.skip = std::move(keep);
                throw;
            }
            Tm.skip = std::move(keep);
            return;
        }
        return spmm_device(c, T, Y, ncols, ncols, Z, ncols, tag);
    }
    // the gather kernel handles every row except the top columns, whose rows of
    // Z are written by the streaming kernel + combine
    spmm_device(c, T, Y, ncols, ncols, Z, ncols, tag);
    Prof prof(c, "spmm_AtY_top", 8.0 * double(A.rows) * ncols, 2.0 * double(A.top_val.n) * ncols);
    DBuf<double> part(size_t(A.ntop_cuts) * kTop * ncols, c.stream);
    const int nch = int((ncols + 63) / 64);
    switch (nch) {
        case 1: launch_top<1>(c, A, Y, ncols, int(ncols), part.get()); break;
        case 2: launch_top<2>(c, A, Y, ncols, int(ncols), part.get()); break;
        case 3: launch_top<3>(c, A, Y, ncols, int(ncols), part.get()); break;
        default: launch_top<4>(c, A, Y, ncols, int(ncols), part.get()); break;
    }
    k_top_combine<<<(kTop * int(ncols) + 255) / 256, 256, 0, c.stream>>>(part.get(), A.ntop_cuts, int(ncols),
                                                                          A.top_cols.get(), Z, ncols);
    FB_LAUNCH_CHECK();
}

}  // namespace fb
