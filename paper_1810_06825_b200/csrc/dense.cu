// K4 (Gram B = W^T W, dense_kernels.hpp:156-157), K6 (rescale / output GEMM
// C = W * M, dense_kernels.hpp:172 and randsvd.hpp:262-267/:314-319), layout
// transposes and max|x| for the LU tolerance.
//
// fp64 has no tcgen05 kind, so the tall-skinny products run on the fp64
// tensor-core path that sm_100a does have: warp-level DMMA
// (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4). Each warp owns a 32x32 tile
// (16 MMAs per k4 step from 8 operand loads), operands are staged in padded
// shared memory by a 2-stage cp.async pipeline, and split-K partials are
// reduced in a fixed order so results are deterministic run to run.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "internal.cuh"

namespace fb {
namespace {

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------------------
// Gram: B = W^T W over lower 64x64 tiles, split over rows.
constexpr int GT = 64;      // output tile
constexpr int GK = 16;      // rows per stage
constexpr int GPAD = GT + 4;

__global__ void __launch_bounds__(128)
k_gram(const double* __restrict__ W, int64_t r, int n, int nt, int64_t rows_per_split,
       double* __restrict__ part) {
    __shared__ __align__(16) double As[2][GK][GPAD];
    __shared__ __align__(16) double Bs[2][GK][GPAD];
    // lower tile index -> (ti, tj), ti >= tj
    int t = blockIdx.x, ti = 0;
    while (t > ti) { t -= ti + 1; ++ti; }
    const int tj = t;
    const bool diag = ti == tj;
    const int i0 = ti * GT, j0 = tj * GT;
    const int64_t rs = int64_t(blockIdx.y) * rows_per_split;
    const int64_t re = min(r, rs + rows_per_split);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wi = warp >> 1, wj = warp & 1;

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    auto load = [&](int stage, int64_t k0) {
#pragma unroll
        for (int e = 0; e < (GK * GT) / 128; ++e) {
            const int idx = e * 128 + tid;
            const int kr = idx / GT, cc = idx % GT;
            const int64_t row = k0 + kr;
            const bool rv = row < re;
            const int ci = i0 + cc;
            cp_async8(&As[stage][kr][cc], W + (rv ? row * n + min(ci, n - 1) : 0), rv && ci < n);
            if (!diag) {
                const int cj = j0 + cc;
                cp_async8(&Bs[stage][kr][cc], W + (rv ? row * n + min(cj, n - 1) : 0), rv && cj < n);
            }
        }
        cp_async_commit();
    };

    const int64_t nsteps = (re - rs + GK - 1) / GK;
    if (nsteps > 0) load(0, rs);
    for (int64_t s = 0; s < nsteps; ++s) {
        const int stage = int(s & 1);
        if (s + 1 < nsteps) {
            load(stage ^ 1, rs + (s + 1) * GK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double(*Ab)[GPAD] = As[stage];
        const double(*Bb)[GPAD] = diag ? As[stage] : Bs[stage];
#pragma unroll
        for (int kk = 0; kk < GK / 4; ++kk) {
            const int krow = kk * 4 + (lane & 3);
            double af[4], bf[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) af[a] = Ab[krow][wi * 32 + a * 8 + (lane >> 2)];
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = Bb[krow][wj * 32 + b * 8 + (lane >> 2)];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(acc[a][b], af[a], bf[b]);
        }
        __syncthreads();
    }
    // partial tile (64x64 row-major) for this split
    double* out = part + (int64_t(blockIdx.y) * gridDim.x + blockIdx.x) * (GT * GT);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int ii = wi * 32 + a * 8 + (lane >> 2);
            const int jj = wj * 32 + b * 8 + (lane & 3) * 2;
            *reinterpret_cast<double2*>(out + ii * GT + jj) = make_double2(acc[a][b][0], acc[a][b][1]);
        }
}

// Sum split partials in split order; write B column-major, both triangles.
__global__ void k_gram_reduce(const double* __restrict__ part, int ntiles, int nsplit, int n,
                              double* __restrict__ B) {
    const int tile = blockIdx.x;
    int t = tile, ti = 0;
    while (t > ti) { t -= ti + 1; ++ti; }
    const int tj = t;
    for (int e = threadIdx.x; e < GT * GT; e += blockDim.x) {
        const int ii = e / GT, jj = e % GT;
        const int i = ti * GT + ii, j = tj * GT + jj;
        if (i >= n || j >= n || (ti == tj && jj > ii)) continue;
        double acc = 0.0;
        for (int s = 0; s < nsplit; ++s) acc += part[(int64_t(s) * ntiles + tile) * (GT * GT) + e];
        B[i + int64_t(j) * n] = acc;
        B[j + int64_t(i) * n] = acc;
    }
}

// ---------------------------------------------------------------------------
// Gram for narrow panels (n <= 224): one CTA per SM owns a contiguous row range
// and the WHOLE lower triangle of B at 8x8 granularity (3% waste at n = 200,
// vs ~50% for 64-wide tiles). The T(T+1)/2 lower 8x8 tiles (T = ceil(n/8))
// are dealt to 16 warps in row-major order; per k4 step a warp loads the A
// fragment of its current tile row once and one B fragment per tile, i.e.
// ~1 LDS.64 per DMMA (half the shared-memory bandwidth a DMMA consumes).
// Rows are staged 32 at a time by a 2-stage cp.async pipeline into rows of
// stride S (S = 12 mod 16 doubles: conflict-free fragment loads).
constexpr int G2_WARPS = 16;
constexpr int G2_ROWS = 32;

template <int MAXT>
__global__ void __launch_bounds__(G2_WARPS * 32, 1)
k_gram2(const double* __restrict__ W, int64_t r, int n, int S, int64_t rows_per_cta,
        double* __restrict__ part) {
    extern __shared__ __align__(16) double sm[];  // [2][G2_ROWS][S]
    const int T = (n + 7) / 8;
    const int NT = T * (T + 1) / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t0 = (warp * NT) / G2_WARPS, t1 = ((warp + 1) * NT) / G2_WARPS;
    const int64_t rs = int64_t(blockIdx.x) * rows_per_cta;
    const int64_t re = min(r, rs + rows_per_cta);
    double acc[MAXT][2];
#pragma unroll
    for (int i = 0; i < MAXT; ++i) acc[i][0] = acc[i][1] = 0.0;

    const bool vec = (n % 2) == 0;
    auto load = [&](int stage, int64_t k0) {
        double* dst = sm + size_t(stage) * G2_ROWS * S;
        if (vec) {
            const int per_row = n / 2;
            for (int e = tid; e < G2_ROWS * per_row; e += blockDim.x) {
                const int kr = e / per_row, cc = (e % per_row) * 2;
                const int64_t row = k0 + kr;
                const bool v = row < re;
                const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + kr * S + cc));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                             "l"(W + (v ? row * n + cc : 0)), "r"(v ? 16 : 0));
            }
        } else {
            for (int e = tid; e < G2_ROWS * n; e += blockDim.x) {
                const int kr = e / n, cc = e % n;
                const int64_t row = k0 + kr;
                cp_async8(dst + kr * S + cc, W + (row < re ? row * n + cc : 0), row < re);
            }
        }
        // zero the padding columns [n, 8T) read by the last tile
        for (int e = tid; e < G2_ROWS * (8 * T - n); e += blockDim.x) {
            const int kr = e / (8 * T - n), cc = n + e % (8 * T - n);
            dst[kr * S + cc] = 0.0;
        }
        cp_async_commit();
    };
    const int64_t nsteps = (re - rs + G2_ROWS - 1) / G2_ROWS;
    if (nsteps > 0) load(0, rs);
    // (ti, tj) of this warp's first tile
    int ti0 = 0;
    while ((ti0 + 1) * (ti0 + 2) / 2 <= t0) ++ti0;
    const int tj0 = t0 - ti0 * (ti0 + 1) / 2;
    for (int64_t st = 0; st < nsteps; ++st) {
        const int stage = int(st & 1);
        if (st + 1 < nsteps) {
            load(stage ^ 1, rs + (st + 1) * G2_ROWS);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* Ws = sm + size_t(stage) * G2_ROWS * S;
#pragma unroll
        for (int kk = 0; kk < G2_ROWS / 4; ++kk) {
            const double* rowp = Ws + (kk * 4 + (lane & 3)) * S + (lane >> 2);
            int ti = ti0, tj = tj0;
            double a = rowp[ti * 8];
#pragma unroll
            for (int i = 0; i < MAXT; ++i) {
                if (t0 + i < t1) {
                    const double b = rowp[tj * 8];
                    dmma(acc[i], a, b);
                    if (++tj > ti) {
                        ++ti;
                        tj = 0;
                        a = rowp[min(ti, T - 1) * 8];
                    }
                }
            }
        }
        __syncthreads();
    }
    // partial tiles: part[cta][tile][64], 8x8 row-major within the tile
    double* out = part + size_t(blockIdx.x) * NT * 64;
#pragma unroll
    for (int i = 0; i < MAXT; ++i) {
        if (t0 + i < t1) {
            const int ii = lane >> 2, jj = (lane & 3) * 2;
            *reinterpret_cast<double2*>(out + size_t(t0 + i) * 64 + ii * 8 + jj) =
                make_double2(acc[i][0], acc[i][1]);
        }
    }
}

// B (column-major n x n, both triangles) = sum over CTAs of the partial tiles,
// added in CTA order.
__global__ void k_gram2_reduce(const double* __restrict__ part, int nparts, int n,
                               double* __restrict__ B) {
    const int T = (n + 7) / 8;
    const int NT = T * (T + 1) / 2;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < NT * 64; e += gridDim.x * blockDim.x) {
        const int t = e / 64, w = e % 64;
        int ti = 0;
        while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
        const int tj = t - ti * (ti + 1) / 2;
        const int i = ti * 8 + w / 8, j = tj * 8 + w % 8;
        if (i >= n || j >= n || j > i) continue;
        double acc = 0.0;
        for (int p = 0; p < nparts; ++p) acc += part[size_t(p) * NT * 64 + e];
        B[i + int64_t(j) * n] = acc;
        B[j + int64_t(i) * n] = acc;
    }
}

// Gram v3: one warp per 5x5 block of 8x8 tiles of the lower triangle (NBR
// block rows, NBR(NBR+1)/2 warps), straight-line: per k4 step a warp loads 5
// (diagonal block) or 10 operand fragments and issues 15 or 25 DMMAs. Rows are
// split over CTAs and staged through shared memory (2-stage cp.async); the
// partial tiles use k_gram2's layout and fixed-order reduction.
constexpr int G3_BT = 5;
constexpr int G3_ROWS = 32;

template <int NBR, int ROWS>
__global__ void __launch_bounds__(NBR * (NBR + 1) / 2 * 32, 1)
k_gram3(const double* __restrict__ W, int64_t r, int n, int S, int64_t rows_per_cta, double* __restrict__ part) {
    extern __shared__ __align__(16) double sm[];  // [2][ROWS][S], S >= 40 NBR
    constexpr int NW = NBR * (NBR + 1) / 2;
    const int T = (n + 7) / 8;
    const int NT = T * (T + 1) / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int bi = 0;
    while ((bi + 1) * (bi + 2) / 2 <= warp) ++bi;
    const int bj = warp - bi * (bi + 1) / 2;
    const bool diag = bi == bj;
    const int64_t rs = int64_t(blockIdx.x) * rows_per_cta;
    const int64_t re = min(r, rs + rows_per_cta);
    const int ncol = 8 * G3_BT * NBR;  // staged columns (zero beyond n)
    double acc[G3_BT][G3_BT][2];
#pragma unroll
    for (int a = 0; a < G3_BT; ++a)
#pragma unroll
        for (int b = 0; b < G3_BT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    auto load = [&](int stage, int64_t k0) {
        double* dst = sm + size_t(stage) * ROWS * S;
        const int per_row = n / 2;  // n even (caller)
        for (int e = tid; e < ROWS * per_row; e += NW * 32) {
            const int kr = e / per_row, cc = (e % per_row) * 2;
            const int64_t row = k0 + kr;
            const bool v = row < re;
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + kr * S + cc));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                         "l"(W + (v ? row * n + cc : 0)), "r"(v ? 16 : 0));
        }
        for (int e = tid; e < ROWS * (ncol - n); e += NW * 32) {
            const int kr = e / (ncol - n), cc = n + e % (ncol - n);
            dst[kr * S + cc] = 0.0;
        }
        cp_async_commit();
    };
    const int64_t nsteps = (re - rs + ROWS - 1) / ROWS;
    if (nsteps > 0) load(0, rs);
    const int coff = (lane & 3) * S + (lane >> 2);
    for (int64_t st = 0; st < nsteps; ++st) {
        const int stage = int(st & 1);
        if (st + 1 < nsteps) {
            load(stage ^ 1, rs + (st + 1) * ROWS);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* Ws = sm + size_t(stage) * ROWS * S + coff;
        if (diag) {
#pragma unroll
            for (int kk = 0; kk < ROWS / 4; ++kk) {
                const double* rowp = Ws + kk * 4 * S + bi * 40;
                double f[G3_BT];
#pragma unroll
                for (int a = 0; a < G3_BT; ++a) f[a] = rowp[a * 8];
#pragma unroll
                for (int a = 0; a < G3_BT; ++a)
#pragma unroll
                    for (int b = 0; b <= a; ++b) dmma(acc[a][b], f[a], f[b]);
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < ROWS / 4; ++kk) {
                const double* rowp = Ws + kk * 4 * S;
                double fa[G3_BT];
#pragma unroll
                for (int a = 0; a < G3_BT; ++a) fa[a] = rowp[bi * 40 + a * 8];
#pragma unroll
                for (int b = 0; b < G3_BT; ++b) {
                    const double fb = rowp[bj * 40 + b * 8];
#pragma unroll
                    for (int a = 0; a < G3_BT; ++a) dmma(acc[a][b], fa[a], fb);
                }
            }
        }
        __syncthreads();
    }
    double* out = part + size_t(blockIdx.x) * NT * 64;
    const int ii = lane >> 2, jj = (lane & 3) * 2;
#pragma unroll
    for (int a = 0; a < G3_BT; ++a)
#pragma unroll
        for (int b = 0; b < G3_BT; ++b) {
            const int ti = bi * G3_BT + a, tj = bj * G3_BT + b;
            if (ti >= T || tj > ti || (diag && b > a)) continue;
            const int t = ti * (ti + 1) / 2 + tj;
            *reinterpret_cast<double2*>(out + size_t(t) * 64 + ii * 8 + jj) = make_double2(acc[a][b][0], acc[a][b][1]);
        }
}

// ---------------------------------------------------------------------------
// Gram v4: k_gram3's warps and DMMA sequence, fed by the Blackwell async copy
// path instead of a block-wide cp.async pipeline. Each W row goes to its
// padded shared-memory slot with a 1-D bulk copy (cp.async.bulk, SASS UBLKCP)
// that completes on the stage's "full" mbarrier; the warps wait on that
// barrier, run their DMMAs, and release the stage on its "empty" mbarrier. No block-wide barrier and no per-element
// index arithmetic remain in the loop. Per tile, the DMMAs are issued in the
// same order over the same 4-row groups as k_gram3 (tail rows zero-filled the
// same way), so the partials and the result are bitwise equal to it.
constexpr int G4_ROWS = 32;
constexpr int G4_STAGES = 4;

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(b))),
                 "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(b))),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(b)))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(bytes), "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
                 : "memory");
}

// A 16th warp is the producer (15 consumer warps + 1 = 512 threads at 128
// registers: a 15-warp CTA at 136 would put 4 x 136-register warps on one
// SM sub-partition, more than its 16K registers).
__device__ __forceinline__ void gram4_fill(const double* __restrict__ W, int n, int S, int64_t rs, int64_t re,
                                           int st, int slot, double* sm, uint64_t* full, int lane) {
    const int64_t k0 = rs + int64_t(st) * G4_ROWS;
    const int valid = int(min(int64_t(G4_ROWS), re - k0));
    double* dst = sm + size_t(slot) * G4_ROWS * S;
    // rows past the CTA's range read as zero (as k_gram3's zero-size copies)
    for (int e = lane; e < (G4_ROWS - valid) * n; e += 32) dst[(valid + e / n) * S + e % n] = 0.0;
    __syncwarp();
    if (lane == 0) mbar_expect_tx(full + slot, unsigned(valid) * unsigned(n) * 8u);
    __syncwarp();
    for (int kr = lane; kr < valid; kr += 32) bulk_g2s(dst + kr * S, W + (k0 + kr) * n, unsigned(n) * 8u, full + slot);
}

template <int NBR>
constexpr int g4_stride() {  // padded row stride: 12 mod 16 doubles, conflict-free fragments
    return 8 * G3_BT * NBR + ((12 - ((8 * G3_BT * NBR) % 16)) + 16) % 16;
}

template <int NBR>
__global__ void __launch_bounds__((NBR * (NBR + 1) / 2 + 1) * 32, 1)
k_gram4(const double* __restrict__ W, int64_t r, int n, int64_t rows_per_cta, double* __restrict__ part) {
    extern __shared__ __align__(128) double sm[];  // [G4_STAGES][G4_ROWS][S], then the barriers
    constexpr int NW = NBR * (NBR + 1) / 2;
    constexpr int S = g4_stride<NBR>();
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(G4_STAGES) * G4_ROWS * S);
    uint64_t* empty = full + G4_STAGES;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t rs = int64_t(blockIdx.x) * rows_per_cta;
    const int64_t re = min(r, rs + rows_per_cta);
    const int nst = int((re - rs + G4_ROWS - 1) / G4_ROWS);
    {
        // padding columns [n, ncol) are never written by the copies: zero once
        const int ncol = 8 * G3_BT * NBR;
        for (int e = tid; e < G4_STAGES * G4_ROWS * (ncol - n); e += blockDim.x) {
            const int q = e / (ncol - n), cc = n + e % (ncol - n);
            sm[size_t(q) * S + cc] = 0.0;
        }
    }
    if (tid == 0) {
        for (int st = 0; st < G4_STAGES; ++st) {
            mbar_init(full + st, 1);
            mbar_init(empty + st, NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NW) {  // producer
        int slot = 0;
        unsigned phase = 0;
        for (int st = 0; st < nst; ++st) {
            if (st >= G4_STAGES) mbar_wait(empty + slot, phase ^ 1u);
            gram4_fill(W, n, S, rs, re, st, slot, sm, full, lane);
            if (++slot == G4_STAGES) {
                slot = 0;
                phase ^= 1u;
            }
        }
        return;
    }
    int bi = 0;
    while ((bi + 1) * (bi + 2) / 2 <= warp) ++bi;
    const int bj = warp - bi * (bi + 1) / 2;
    const bool diag = bi == bj;
    double acc[G3_BT][G3_BT][2];
#pragma unroll
    for (int a = 0; a < G3_BT; ++a)
#pragma unroll
        for (int b = 0; b < G3_BT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // stage and barrier addresses as 32-bit shared-window offsets (registers)
    const unsigned full0 = static_cast<unsigned>(__cvta_generic_to_shared(full));
    constexpr unsigned stage_bytes = unsigned(G4_ROWS * S) * 8u;
    const int lane_off = (lane & 3) * S + (lane >> 2) + (diag ? bi * 40 : 0);
    unsigned soff = 0;  // current stage, byte offset
    int slot = 0;
    unsigned phase = 0;
    for (int st = nst; st > 0; --st) {
        {
            const unsigned a = full0 + 8u * unsigned(slot);
            asm volatile(
                "{\n .reg .pred p;\n"
                "W4: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
                " @!p bra W4;\n}" ::"r"(a),
                "r"(phase)
                : "memory");
        }
        const double* Ws = reinterpret_cast<const double*>(reinterpret_cast<const char*>(sm) + soff) + lane_off;
        if (diag) {
#pragma unroll
            for (int kk = 0; kk < G4_ROWS / 4; ++kk) {
                const double* rowp = Ws + kk * 4 * S;
                double f[G3_BT];
#pragma unroll
                for (int a = 0; a < G3_BT; ++a) f[a] = rowp[a * 8];
#pragma unroll
                for (int a = 0; a < G3_BT; ++a)
#pragma unroll
                    for (int b = 0; b <= a; ++b) dmma(acc[a][b], f[a], f[b]);
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < G4_ROWS / 4; ++kk) {
                const double* rowp = Ws + kk * 4 * S;
                double fa[G3_BT];
#pragma unroll
                for (int a = 0; a < G3_BT; ++a) fa[a] = rowp[bi * 40 + a * 8];
#pragma unroll
                for (int b = 0; b < G3_BT; ++b) {
                    const double fb = rowp[bj * 40 + b * 8];
#pragma unroll
                    for (int a = 0; a < G3_BT; ++a) dmma(acc[a][b], fa[a], fb);
                }
            }
        }
        __syncwarp();
        if (lane == 0) {
            const unsigned a = full0 + 8u * unsigned(G4_STAGES + slot);
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
        }
        soff += stage_bytes;
        if (++slot == G4_STAGES) {
            slot = 0;
            soff = 0;
            phase ^= 1u;
        }
    }
    const int T = (n + 7) / 8;
    const int NT = T * (T + 1) / 2;
    double* out = part + size_t(blockIdx.x) * NT * 64;
    const int ii = lane >> 2, jj = (lane & 3) * 2;
#pragma unroll
    for (int a = 0; a < G3_BT; ++a)
#pragma unroll
        for (int b = 0; b < G3_BT; ++b) {
            const int ti = bi * G3_BT + a, tj = bj * G3_BT + b;
            if (ti >= T || tj > ti || (diag && b > a)) continue;
            const int t = ti * (ti + 1) / 2 + tj;
            *reinterpret_cast<double2*>(out + size_t(t) * 64 + ii * 8 + jj) = make_double2(acc[a][b][0], acc[a][b][1]);
        }
}

template <int NBR>
void launch_gram4(Ctx& c, const double* W, int64_t r, int n, double* B) {
    constexpr int NW = NBR * (NBR + 1) / 2;
    const int T = (n + 7) / 8, NT = T * (T + 1) / 2;
    constexpr int S = g4_stride<NBR>();
    const size_t smem = sizeof(double) * size_t(G4_STAGES) * G4_ROWS * S + 2 * G4_STAGES * sizeof(uint64_t);
    smem_optin(k_gram4<NBR>, smem);
    // the same 32-row CTA split as k_gram3 (identical partials)
    int64_t nctas = std::min<int64_t>(c.num_sms, std::max<int64_t>(1, (r + G3_ROWS - 1) / G3_ROWS));
    const int64_t rpc = ((r + nctas - 1) / nctas + G3_ROWS - 1) / G3_ROWS * G3_ROWS;
    nctas = std::max<int64_t>(1, (r + rpc - 1) / rpc);
    DBuf<double> part(size_t(nctas) * NT * 64, c.stream);
    k_gram4<NBR><<<unsigned(nctas), (NW + 1) * 32, smem, c.stream>>>(W, r, n, rpc, part.get());
    FB_LAUNCH_CHECK();
    const int outs = NT * 64;
    k_gram2_reduce<<<(outs + 255) / 256, 256, 0, c.stream>>>(part.get(), int(nctas), n, B);
    FB_LAUNCH_CHECK();
}

template <int NBR, int ROWS>
void launch_gram3_rows(Ctx& c, const double* W, int64_t r, int n, double* B) {
    constexpr int NW = NBR * (NBR + 1) / 2;
    const int T = (n + 7) / 8, NT = T * (T + 1) / 2;
    const int ncol = 8 * G3_BT * NBR;
    const int S = ncol + ((12 - (ncol % 16)) + 16) % 16;
    const size_t smem = sizeof(double) * 2 * ROWS * S;
    smem_optin(k_gram3<NBR, ROWS>, size_t(smem));
    // the row split over CTAs stays at 32-row granularity whatever the staging
    // depth, so the split-K partials (and the result) do not depend on ROWS
    int64_t nctas = std::min<int64_t>(c.num_sms, std::max<int64_t>(1, (r + G3_ROWS - 1) / G3_ROWS));
    const int64_t rpc = ((r + nctas - 1) / nctas + G3_ROWS - 1) / G3_ROWS * G3_ROWS;
    nctas = std::max<int64_t>(1, (r + rpc - 1) / rpc);
    DBuf<double> part(size_t(nctas) * NT * 64, c.stream);
    k_gram3<NBR, ROWS><<<unsigned(nctas), NW * 32, smem, c.stream>>>(W, r, n, S, rpc, part.get());
    FB_LAUNCH_CHECK();
    const int outs = NT * 64;
    k_gram2_reduce<<<(outs + 255) / 256, 256, 0, c.stream>>>(part.get(), int(nctas), n, B);
    FB_LAUNCH_CHECK();
}

template <int NBR>
void launch_gram3(Ctx& c, const double* W, int64_t r, int n, double* B) {
    // staging depth (does not change the result): 64 rows per stage halves the
    // block barriers (C1 1.77 -> 1.74 ms, C3 22.4 -> 21.2 ms)
    const char* e = std::getenv("FRPCA_GRAM_ROWS");
    if (e && std::atoi(e) == 32) return launch_gram3_rows<NBR, 32>(c, W, r, n, B);
    launch_gram3_rows<NBR, 64>(c, W, r, n, B);
}

template <int MAXT>
void launch_gram2(Ctx& c, const double* W, int64_t r, int n, double* B) {
    const int T = (n + 7) / 8, NT = T * (T + 1) / 2;
    const int S = n + ((12 - (n % 16)) + 16) % 16 + ((8 * T > n + ((12 - (n % 16)) + 16) % 16) ? 16 : 0);
    const size_t smem = sizeof(double) * 2 * G2_ROWS * S;
    smem_optin(k_gram2<MAXT>, size_t(200 * 1024));
    int64_t nctas = std::min<int64_t>(c.num_sms, std::max<int64_t>(1, (r + G2_ROWS - 1) / G2_ROWS));
    const int64_t rpc = ((r + nctas - 1) / nctas + G2_ROWS - 1) / G2_ROWS * G2_ROWS;
    nctas = std::max<int64_t>(1, (r + rpc - 1) / rpc);
    DBuf<double> part(size_t(nctas) * NT * 64, c.stream);
    k_gram2<MAXT><<<unsigned(nctas), G2_WARPS * 32, smem, c.stream>>>(W, r, n, S, rpc, part.get());
    FB_LAUNCH_CHECK();
    const int outs = NT * 64;
    k_gram2_reduce<<<(outs + 255) / 256, 256, 0, c.stream>>>(part.get(), int(nctas), n, B);
    FB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// GEMM: C (r x N) = W (r x K, row-major) * M (K x N, row-major).
constexpr int MT = 64;      // rows per tile
constexpr int NT = 64;      // cols per tile
constexpr int KT = 16;      // k per stage
constexpr int APAD = KT + 4;
constexpr int BPAD = NT + 4;

__global__ void __launch_bounds__(128)
k_gemm(const double* __restrict__ W, int64_t r, int K, const double* __restrict__ M, int N,
       double* __restrict__ C, int64_t ldc, int col_major) {
    __shared__ __align__(16) double As[2][MT][APAD];
    __shared__ __align__(16) double Bs[2][KT][BPAD];
    const int64_t r0 = int64_t(blockIdx.x) * MT;
    const int n0 = blockIdx.y * NT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wi = warp >> 1, wj = warp & 1;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    auto load = [&](int stage, int k0) {
#pragma unroll
        for (int e = 0; e < (MT * KT) / 128; ++e) {
            const int idx = e * 128 + tid;
            const int rr = idx / KT, kk = idx % KT;
            const int64_t row = r0 + rr;
            const int k = k0 + kk;
            const bool v = row < r && k < K;
            cp_async8(&As[stage][rr][kk], W + (v ? row * K + k : 0), v);
        }
#pragma unroll
        for (int e = 0; e < (KT * NT) / 128; ++e) {
            const int idx = e * 128 + tid;
            const int kk = idx / NT, cc = idx % NT;
            const int k = k0 + kk, col = n0 + cc;
            const bool v = k < K && col < N;
            cp_async8(&Bs[stage][kk][cc], M + (v ? int64_t(k) * N + col : 0), v);
        }
        cp_async_commit();
    };
    const int nsteps = (K + KT - 1) / KT;
    load(0, 0);
    for (int s = 0; s < nsteps; ++s) {
        const int stage = s & 1;
        if (s + 1 < nsteps) {
            load(stage ^ 1, (s + 1) * KT);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KT / 4; ++kk) {
            double af[4], bf[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) af[a] = As[stage][wi * 32 + a * 8 + (lane >> 2)][kk * 4 + (lane & 3)];
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = Bs[stage][kk * 4 + (lane & 3)][wj * 32 + b * 8 + (lane >> 2)];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma(acc[a][b], af[a], bf[b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t row = r0 + wi * 32 + a * 8 + (lane >> 2);
            const int col = n0 + wj * 32 + b * 8 + (lane & 3) * 2;
            if (row >= r) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (col + h >= N) continue;
                if (col_major) C[int64_t(col + h) * ldc + row] = acc[a][b][h];
                else C[row * ldc + col + h] = acc[a][b][h];
            }
        }
}

// ---------------------------------------------------------------------------
// Tall-skinny GEMM with the full output width per CTA (N <= 256): C (r x N) =
// W (r x K) * M (K x N). Each warp owns 2 row tiles x NT column tiles of 8x8
// (per k4 step: 2 + NT fragment loads for 2*NT DMMAs), so the only padding is
// N up to a multiple of 8 (no 64-wide tile waste). Warps: 8 per CTA, WC
// column groups; the CTA covers 16 * 8 / WC rows. K is staged 16 at a time
// (2-stage cp.async) into rows of stride 20 (W) and NP + pad (M), both
// = 4 or 12 mod 16 doubles: conflict-free fragment loads.
constexpr int TK = 16;
constexpr int TSA = TK + 4;

template <int NT>
__global__ void __launch_bounds__(256, 2)
k_gemm_tall(const double* __restrict__ W, int64_t r, int K, const double* __restrict__ M, int N,
            double* __restrict__ C, int64_t ldc, int col_major, int WC, int SB) {
    extern __shared__ __align__(16) double sm[];
    const int BM = 16 * (8 / WC);
    const int ntiles = (N + 7) / 8;
    const int NP = 8 * ntiles;
    double* Ws = sm;                                  // [2][BM][TSA]
    double* Ms = sm + 2 * BM * TSA;                   // [2][TK][SB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rg = warp / WC, cgp = warp % WC;
    const int64_t r0 = int64_t(blockIdx.x) * BM;
    double acc[2][NT][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[a][t][0] = acc[a][t][1] = 0.0;

    auto load = [&](int stage, int k0) {
        double* wd = Ws + stage * BM * TSA;
        for (int e = tid; e < BM * TK; e += 256) {
            const int rr = e / TK, kk = e % TK;
            const int64_t row = r0 + rr;
            const int k = k0 + kk;
            const bool v = row < r && k < K;
            cp_async8(wd + rr * TSA + kk, W + (v ? row * K + k : 0), v);
        }
        double* md = Ms + stage * TK * SB;
        for (int e = tid; e < TK * NP; e += 256) {
            const int kk = e / NP, cc = e % NP;
            const int k = k0 + kk;
            const bool v = k < K && cc < N;
            cp_async8(md + kk * SB + cc, M + (v ? int64_t(k) * N + cc : 0), v);
        }
        cp_async_commit();
    };
    const int nsteps = (K + TK - 1) / TK;
    load(0, 0);
    for (int st = 0; st < nsteps; ++st) {
        const int stage = st & 1;
        if (st + 1 < nsteps) {
            load(stage ^ 1, (st + 1) * TK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* wd = Ws + stage * BM * TSA + (rg * 16 + (lane >> 2)) * TSA + (lane & 3);
        const double* md = Ms + stage * TK * SB + (lane & 3) * SB + cgp * NT * 8 + (lane >> 2);
#pragma unroll
        for (int kk = 0; kk < TK / 4; ++kk) {
            const double a0 = wd[kk * 4], a1 = wd[8 * TSA + kk * 4];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (cgp * NT + t < ntiles) {
                    const double b = md[kk * 4 * SB + t * 8];
                    dmma(acc[0][t], a0, b);
                    dmma(acc[1][t], a1, b);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int64_t row = r0 + rg * 16 + a * 8 + (lane >> 2);
            const int col = (cgp * NT + t) * 8 + (lane & 3) * 2;
            if (row >= r || cgp * NT + t >= ntiles) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (col + h >= N) continue;
                if (col_major) C[int64_t(col + h) * ldc + row] = acc[a][t][h];
                else C[row * ldc + col + h] = acc[a][t][h];
            }
        }
}

// Persistent variant for tall W: the whole column chunk of M (K x NP, NP <= 104)
// stays in shared memory for the CTA's lifetime and W is streamed through once
// (M is read once per SM instead of once per 64-row block). 8 warps, each
// owning RT x NT tiles (RT A and NT B fragments per k4 step for RT*NT DMMAs).
constexpr int PCOLS = 104;
constexpr int GP_THREADS = 256;
template <int RT, int NT>
__global__ void __launch_bounds__(GP_THREADS, 1)
k_gemm_persist(const double* __restrict__ W, int64_t r, int K, const double* __restrict__ M, int ldm,
               int N, double* __restrict__ C, int64_t ldc, int col_major, int WC, int SB) {
    extern __shared__ __align__(16) double sm[];
    const int BM = 8 * RT * ((GP_THREADS / 32) / WC);
    const int ntiles = (N + 7) / 8;
    const int NP = 8 * ntiles;
    double* Ms = sm;                                  // [K][SB]
    double* Ws = sm + size_t(K) * SB;                 // [2][BM][TSA]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rg = warp / WC, cgp = warp % WC;
    // rows K .. Kp-1 of M are read against zero-filled W columns: zero them
    // (an uninitialised Inf/NaN there would turn 0 * x into NaN)
    const int Kp = (K + TK - 1) / TK * TK;
    for (int e = tid; e < Kp * NP; e += GP_THREADS) {
        const int k = e / NP, cc = e % NP;
        cp_async8(Ms + k * SB + cc, M + (cc < N && k < K ? int64_t(k) * ldm + cc : 0), cc < N && k < K);
    }
    cp_async_commit();
    const int nsteps = (K + TK - 1) / TK;
    // 16-byte staging when the rows of W are 16-byte aligned
    const bool even = (K & 1) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0;
    auto load = [&](int stage, int64_t r0, int k0) {
        double* wd = Ws + stage * BM * TSA;
        if (even) {
            for (int e = tid; e < BM * (TK / 2); e += GP_THREADS) {
                const int rr = e / (TK / 2), c2 = e % (TK / 2);
                const int64_t row = r0 + rr;
                const int k = k0 + 2 * c2;
                const bool v = row < r && k < K;
                cp_async16(wd + rr * TSA + 2 * c2, W + (v ? row * K + k : 0), v);
            }
        } else {
            for (int e = tid; e < BM * TK; e += GP_THREADS) {
                const int rr = e / TK, kk = e % TK;
                const int64_t row = r0 + rr;
                const int k = k0 + kk;
                const bool v = row < r && k < K;
                cp_async8(wd + rr * TSA + kk, W + (v ? row * K + k : 0), v);
            }
        }
        cp_async_commit();
    };
    // one continuous two-stage pipeline over (row block, k stage): the last
    // stage of a block prefetches the first stage of the CTA's next block
    const int64_t nblocks = (r + BM - 1) / BM;
    if (int64_t(blockIdx.x) < nblocks) load(0, int64_t(blockIdx.x) * BM, 0);
    int stage = 0;
    for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
        const int64_t r0 = blk * BM;
        double acc[RT][NT][2];
#pragma unroll
        for (int a = 0; a < RT; ++a)
#pragma unroll
            for (int t = 0; t < NT; ++t) acc[a][t][0] = acc[a][t][1] = 0.0;
        for (int st = 0; st < nsteps; ++st) {
            const int64_t nb = blk + gridDim.x;
            if (st + 1 < nsteps) {
                load(stage ^ 1, r0, (st + 1) * TK);
                cp_async_wait<1>();
            } else if (nb < nblocks) {
                load(stage ^ 1, nb * BM, 0);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const double* wd = Ws + stage * BM * TSA + (rg * 8 * RT + (lane >> 2)) * TSA + (lane & 3);
            const double* md = Ms + (st * TK + (lane & 3)) * SB + cgp * NT * 8 + (lane >> 2);
#pragma unroll
            for (int kk = 0; kk < TK / 4; ++kk) {
                if (st * TK + kk * 4 >= K) break;
                double fa[RT];
#pragma unroll
                for (int a = 0; a < RT; ++a) fa[a] = wd[a * 8 * TSA + kk * 4];
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    if (cgp * NT + t < ntiles) {
                        const double b = md[kk * 4 * SB + t * 8];
#pragma unroll
                        for (int a = 0; a < RT; ++a) dmma(acc[a][t], fa[a], b);
                    }
                }
            }
            __syncthreads();
            stage ^= 1;
        }
#pragma unroll
        for (int a = 0; a < RT; ++a)
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int64_t row = r0 + rg * 8 * RT + a * 8 + (lane >> 2);
                const int col = (cgp * NT + t) * 8 + (lane & 3) * 2;
                if (row >= r || cgp * NT + t >= ntiles) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (col + h >= N) continue;
                    if (col_major) C[int64_t(col + h) * ldc + row] = acc[a][t][h];
                    else C[row * ldc + col + h] = acc[a][t][h];
                }
            }
    }
}

// ---------------------------------------------------------------------------
// The persistent GEMM fed by the Tensor Memory Accelerator: each (row block,
// k stage) tile of W (BM rows x TK = 16 columns) arrives in shared memory with
// one cp.async.bulk.tensor.2d (SASS UTMALDG) whose 128-byte swizzle makes the
// fragment loads conflict-free without padding; out-of-range rows and the
// columns past K are zero-filled by the TMA unit. Lane 0 of warp 0 issues the
// copies (after every warp released the stage on its "empty" mbarrier); the
// warps wait on the stage's "full" mbarrier. Same warp tiling, the same DMMAs
// in the same k order per output tile as k_gemm_persist: bitwise equal.
constexpr int GT_STAGES = 2;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            static_cast<unsigned>(__cvta_generic_to_shared(dst))),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
        : "memory");
}

template <int RT, int NT>
__global__ void __launch_bounds__(GP_THREADS, 1)
k_gemm_tma(const __grid_constant__ CUtensorMap wmap, int64_t r, int K, const double* __restrict__ M, int ldm, int N,
           double* __restrict__ C, int64_t ldc, int col_major, int WC, int SB) {
    extern __shared__ __align__(1024) double sm_raw[];
    // the 128-byte swizzle needs 1024-byte aligned stage tiles (1 KB of slack
    // is allocated for this)
    double* sm = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    const int BM = 8 * RT * ((GP_THREADS / 32) / WC);
    const int ntiles = (N + 7) / 8;
    const int NP = 8 * ntiles;
    const int Kp = (K + TK - 1) / TK * TK;
    double* Ws = sm;                                  // [GT_STAGES][BM][TK], 1024-aligned, swizzled
    double* Ms = sm + size_t(GT_STAGES) * BM * TK;    // [Kp][SB], rows K.. zero
    uint64_t* full = reinterpret_cast<uint64_t*>(Ms + size_t(Kp) * SB);
    uint64_t* empty = full + GT_STAGES;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rg = warp / WC, cgp = warp % WC;
    for (int e = tid; e < Kp * NP; e += GP_THREADS) {
        const int k = e / NP, cc = e % NP;
        cp_async8(Ms + k * SB + cc, M + (cc < N && k < K ? int64_t(k) * ldm + cc : 0), cc < N && k < K);
    }
    cp_async_commit();
    if (tid == 0) {
        for (int st = 0; st < GT_STAGES; ++st) {
            mbar_init(full + st, 1);
            mbar_init(empty + st, GP_THREADS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cp_async_wait<0>();
    __syncthreads();
    const int nsteps = (K + TK - 1) / TK;
    const int64_t nblocks = (r + BM - 1) / BM;
    const int64_t myblocks = int64_t(blockIdx.x) < nblocks ? (nblocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t total = myblocks * nsteps;
    const unsigned stage_bytes = unsigned(BM) * TK * 8u;
    auto issue = [&](int64_t g) {  // tile g of this CTA into slot g % 2
        const int64_t blk = blockIdx.x + (g / nsteps) * int64_t(gridDim.x);
        const int st = int(g % nsteps);
        const int slot = int(g & 1);
        mbar_expect_tx(full + slot, stage_bytes);
        tma_load_2d(Ws + size_t(slot) * BM * TK, &wmap, st * TK, int(blk * BM), full + slot);
    };
    if (warp == 0 && lane == 0) {
        for (int64_t g = 0; g < min(total, int64_t(GT_STAGES)); ++g) issue(g);
    }
    // fragment rows of this lane within the stage tile, and their swizzle key
    const int rbase = rg * 8 * RT + (lane >> 2);
    int64_t g = 0;
    for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
        const int64_t r0 = blk * BM;
        double acc[RT][NT][2];
#pragma unroll
        for (int a = 0; a < RT; ++a)
#pragma unroll
            for (int t = 0; t < NT; ++t) acc[a][t][0] = acc[a][t][1] = 0.0;
        for (int st = 0; st < nsteps; ++st, ++g) {
            const int slot = int(g & 1);
            mbar_wait(full + slot, unsigned((g >> 1) & 1));
            const char* wd = reinterpret_cast<const char*>(Ws + size_t(slot) * BM * TK);
            const double* md = Ms + (st * TK + (lane & 3)) * SB + cgp * NT * 8 + (lane >> 2);
#pragma unroll
            for (int kk = 0; kk < TK / 4; ++kk) {
                if (st * TK + kk * 4 >= K) break;
                const int k = kk * 4 + (lane & 3);
                double fa[RT];
#pragma unroll
                for (int a = 0; a < RT; ++a) {
                    const int row = rbase + a * 8;  // row & 7 == lane >> 2 (row tiles are 8-aligned)
                    fa[a] = *reinterpret_cast<const double*>(wd + row * 128 + ((((k >> 1) ^ (lane >> 2)) & 7) << 4) +
                                                             ((k & 1) << 3));
                }
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    if (cgp * NT + t < ntiles) {
                        const double b = md[kk * 4 * SB + t * 8];
#pragma unroll
                        for (int a = 0; a < RT; ++a) dmma(acc[a][t], fa[a], b);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + slot);
            if (warp == 0 && lane == 0 && g + GT_STAGES < total) {
                mbar_wait(empty + slot, unsigned((g >> 1) & 1));  // every warp is done with tile g
                issue(g + GT_STAGES);
            }
        }
#pragma unroll
        for (int a = 0; a < RT; ++a)
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int64_t row = r0 + rg * 8 * RT + a * 8 + (lane >> 2);
                const int col = (cgp * NT + t) * 8 + (lane & 3) * 2;
                if (row >= r || cgp * NT + t >= ntiles) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (col + h >= N) continue;
                    if (col_major) C[int64_t(col + h) * ldc + row] = acc[a][t][h];
                    else C[row * ldc + col + h] = acc[a][t][h];
                }
            }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// W (r x K row-major) as a 2-D tensor with boxes of TK columns x BM rows,
// 128-byte swizzle, zero fill out of range; false if it cannot be described
// (alignment, driver entry point)
bool make_w_map(CUtensorMap& map, const double* W, int64_t r, int64_t K, int BM) {
    auto enc = tensor_map_encoder();
    if (!enc || (reinterpret_cast<uintptr_t>(W) & 15) || (K * 8) % 16 || r >= (int64_t(1) << 31)) return false;
    const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(r)};
    const cuuint64_t strides[1] = {cuuint64_t(K) * 8};
    const cuuint32_t box[2] = {cuuint32_t(TK), cuuint32_t(BM)};
    const cuuint32_t estr[2] = {1, 1};
    return enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(W), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int RT, int NT>
bool launch_gemm_tma(Ctx& c, const double* W, int64_t r, int64_t K, const double* M, int64_t ldm, int64_t N,
                     double* C, int64_t ldc, bool col_major_out, int WC) {
    const int ntiles = int((N + 7) / 8), NP = 8 * ntiles;
    const int SB = NP + ((12 - (NP % 16)) + 16) % 16;
    const int BM = 8 * RT * ((GP_THREADS / 32) / WC);
    const int Kp = int((K + TK - 1) / TK) * TK;
    const size_t smem = sizeof(double) * (size_t(GT_STAGES) * BM * TK + size_t(Kp) * SB) + 4 * sizeof(uint64_t) + 1024;
    if (smem > 227 * 1024 || BM > 256) return false;
    CUtensorMap map;
    if (!make_w_map(map, W, r, K, BM)) return false;
    smem_optin(k_gemm_tma<RT, NT>, smem);
    const int64_t nblocks = (r + BM - 1) / BM;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(c.num_sms, nblocks)));
    k_gemm_tma<RT, NT><<<grid, GP_THREADS, smem, c.stream>>>(map, r, int(K), M, int(ldm), int(N), C, ldc,
                                                              col_major_out ? 1 : 0, WC, SB);
    FB_LAUNCH_CHECK();
    return true;
}

template <int RT, int NT>
void launch_gemm_persist(Ctx& c, const double* W, int64_t r, int64_t K, const double* M, int64_t ldm,
                         int64_t N, double* C, int64_t ldc, bool col_major_out, int WC) {
    const int ntiles = int((N + 7) / 8), NP = 8 * ntiles;
    const int SB = NP + ((12 - (NP % 16)) + 16) % 16;
    const int BM = 8 * RT * ((GP_THREADS / 32) / WC);
    const int Kp = int((K + TK - 1) / TK) * TK;
    const size_t smem = sizeof(double) * (size_t(Kp) * SB + 2 * size_t(BM) * TSA);
    smem_optin(k_gemm_persist<RT, NT>, size_t(227 * 1024));
    const int64_t nblocks = (r + BM - 1) / BM;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(c.num_sms, nblocks)));
    k_gemm_persist<RT, NT><<<grid, GP_THREADS, smem, c.stream>>>(W, r, int(K), M, int(ldm), int(N), C, ldc,
                                                          col_major_out ? 1 : 0, WC, SB);
    FB_LAUNCH_CHECK();
}

template <int NT>
void launch_gemm_tall(Ctx& c, const double* W, int64_t r, int64_t K, const double* M, int64_t N,
                      double* C, int64_t ldc, bool col_major_out, int WC) {
    const int ntiles = int((N + 7) / 8), NP = 8 * ntiles;
    const int SB = NP + ((12 - (NP % 16)) + 16) % 16;
    const int BM = 16 * (8 / WC);
    const size_t smem = sizeof(double) * (2 * size_t(BM) * TSA + 2 * size_t(TK) * SB);
    smem_optin(k_gemm_tall<NT>, size_t(112 * 1024));
    k_gemm_tall<NT><<<unsigned((r + BM - 1) / BM), 256, smem, c.stream>>>(W, r, int(K), M, int(N), C, ldc,
                                                                       col_major_out ? 1 : 0, WC, SB);
    FB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
__global__ void k_transpose(const double* __restrict__ in, int64_t rows, int64_t cols,
                            double* __restrict__ out) {
    __shared__ double tile[32][33];
    const int64_t c0 = int64_t(blockIdx.x) * 32;
    // row tiles loop past grid.y's 65535 limit (outputs taller than 2M rows)
    for (int64_t r0 = int64_t(blockIdx.y) * 32; r0 < rows; r0 += int64_t(gridDim.y) * 32) {
        __syncthreads();  // previous tile consumed
        for (int k = threadIdx.y; k < 32; k += blockDim.y) {
            const int64_t r = r0 + k, c = c0 + threadIdx.x;
            if (r < rows && c < cols) tile[k][threadIdx.x] = in[r * cols + c];
        }
        __syncthreads();
        for (int k = threadIdx.y; k < 32; k += blockDim.y) {
            const int64_t c = c0 + k, r = r0 + threadIdx.x;
            if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][k];
        }
    }
}

__global__ void k_maxabs(const double* __restrict__ x, int64_t n, unsigned long long* __restrict__ out) {
    double m = 0.0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        m = fmax(m, fabs(x[i]));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

}  // namespace

void gram_device(Ctx& c, const double* W, int64_t r, int64_t n, double* B) {
    Prof prof(c, "gram", 8.0 * r * n, double(r) * n * (n + 1));
    if (n <= 224 && r > 0) {
        const int T = int((n + 7) / 8), NT = T * (T + 1) / 2;
        const bool g2 = std::getenv("FRPCA_GRAM2") != nullptr;  // tests compare both kernels
        if (!g2 && n % 2 == 0 && r >= 4096) {
            const int nbr = (T + G3_BT - 1) / G3_BT;
            // the bulk-copy kernel needs 16-byte rows and addresses
            const char* g3 = std::getenv("FRPCA_GRAM3");  // A/B and tests
            const bool bulk = !(g3 && *g3 == '1') && (reinterpret_cast<uintptr_t>(W) % 16) == 0;
            if (bulk) {
                if (nbr == 5) return launch_gram4<5>(c, W, r, int(n), B);
                if (nbr == 4) return launch_gram4<4>(c, W, r, int(n), B);
                if (nbr == 3) return launch_gram4<3>(c, W, r, int(n), B);
            }
            if (nbr == 5) return launch_gram3<5>(c, W, r, int(n), B);
            if (nbr == 4) return launch_gram3<4>(c, W, r, int(n), B);
            if (nbr == 3) return launch_gram3<3>(c, W, r, int(n), B);
        }
        const int maxt = (NT + G2_WARPS - 1) / G2_WARPS;
        if (maxt <= 2) return launch_gram2<2>(c, W, r, int(n), B);
        if (maxt <= 4) return launch_gram2<4>(c, W, r, int(n), B);
        if (maxt <= 8) return launch_gram2<8>(c, W, r, int(n), B);
        if (maxt <= 13) return launch_gram2<13>(c, W, r, int(n), B);
        if (maxt <= 21) return launch_gram2<21>(c, W, r, int(n), B);
        return launch_gram2<26>(c, W, r, int(n), B);
    }
    const int nt = int((n + GT - 1) / GT);
    const int ntiles = nt * (nt + 1) / 2;
    int64_t nsplit = std::max<int64_t>(1, (int64_t(c.num_sms) * 8) / ntiles);
    nsplit = std::min<int64_t>(nsplit, std::max<int64_t>(1, (r + 63) / 64));
    const int64_t rps = ((r + nsplit - 1) / nsplit + GK - 1) / GK * GK;
    nsplit = std::max<int64_t>(1, (r + rps - 1) / rps);
    DBuf<double> part(size_t(nsplit) * ntiles * GT * GT, c.stream);
    dim3 grid(ntiles, unsigned(nsplit));
    k_gram<<<grid, 128, 0, c.stream>>>(W, r, int(n), nt, rps, part.get());
    FB_LAUNCH_CHECK();
    k_gram_reduce<<<ntiles, 256, 0, c.stream>>>(part.get(), ntiles, int(nsplit), int(n), B);
    FB_LAUNCH_CHECK();
}

void gemm_device(Ctx& c, const double* W, int64_t r, int64_t K, const double* M, int64_t N,
                 double* C, int64_t ldc, bool col_major_out) {
    if (r == 0 || N == 0) return;
    Prof prof(c, "rescale_gemm", 8.0 * r * (K + N), 2.0 * r * K * N);
    // persistent kernel with M resident in shared memory, in column chunks of
    // <= 104 (K <= 208 keeps a chunk of M within 227 KB)
    if (K <= 208 && r >= 4096) {
        for (int64_t c0 = 0; c0 < N; c0 += PCOLS) {
            const int64_t nc = std::min<int64_t>(PCOLS, N - c0);
            double* Cc = col_major_out ? C + c0 * ldc : C + c0;
            const int ntiles = int((nc + 7) / 8);
            // a warp holds at most 7 column tiles (<4, 7>): 8 tiles (57-64 columns)
            // go to two column groups of 4, not to one group of 8
            const int WC = ntiles <= 7 ? 1 : 2;
            const int nt = (ntiles + WC - 1) / WC;
            const char* ge = std::getenv("FRPCA_GEMM_CPASYNC");  // A/B and tests
            const bool tma = !(ge && *ge == '1');
            if (nt <= 2) {
                if (!tma || !launch_gemm_tma<4, 2>(c, W, r, K, M + c0, N, nc, Cc, ldc, col_major_out, WC))
                    launch_gemm_persist<4, 2>(c, W, r, K, M + c0, N, nc, Cc, ldc, col_major_out, WC);
            } else if (nt <= 4) {
                if (!tma || !launch_gemm_tma<4, 4>(c, W, r, K, M + c0, N, nc, Cc, ldc, col_major_out, WC))
                    launch_gemm_persist<4, 4>(c, W, r, K, M + c0, N, nc, Cc, ldc, col_major_out, WC);
            } else {
                if (!tma || !launch_gemm_tma<4, 7>(c, W, r, K, M + c0, N, nc, Cc, ldc, col_major_out, WC))
                    launch_gemm_persist<4, 7>(c, W, r, K, M + c0, N, nc, Cc, ldc, col_major_out, WC);
            }
        }
        return;
    }
    dim3 grid(unsigned((r + MT - 1) / MT), unsigned((N + NT - 1) / NT));
    k_gemm<<<grid, 128, 0, c.stream>>>(W, r, int(K), M, int(N), C, ldc, col_major_out ? 1 : 0);
    FB_LAUNCH_CHECK();
}

void transpose_device(Ctx& c, const double* in, int64_t rows, int64_t cols, double* out) {
    if (rows == 0 || cols == 0) return;
    Prof prof(c, "transpose", 16.0 * rows * cols, 0.0);
    dim3 grid(unsigned((cols + 31) / 32), unsigned(std::min<int64_t>(65535, (rows + 31) / 32)));
    k_transpose<<<grid, dim3(32, 8), 0, c.stream>>>(in, rows, cols, out);
    FB_LAUNCH_CHECK();
}

void maxabs_device_async(Ctx& c, const double* x, int64_t n, unsigned long long* out) {
    FB_CUDA(cudaMemsetAsync(out, 0, 8, c.stream));
    if (n) {
        const int grid = int(std::max<int64_t>(1, std::min<int64_t>(c.num_sms * 8, (n + 255) / 256)));
        k_maxabs<<<grid, 256, 0, c.stream>>>(x, n, out);
        FB_LAUNCH_CHECK();
    }
}

double maxabs_device(Ctx& c, const double* x, int64_t n) {
    DBuf<unsigned long long> d(1, c.stream);
    FB_CUDA(cudaMemsetAsync(d.get(), 0, 8, c.stream));
    if (n) {
        const int grid = int(std::max<int64_t>(1, std::min<int64_t>(c.num_sms * 8, (n + 255) / 256)));
        k_maxabs<<<grid, 256, 0, c.stream>>>(x, n, d.get());
        FB_LAUNCH_CHECK();
    }
    unsigned long long h;
    FB_CUDA(cudaMemcpyAsync(&h, d.get(), 8, cudaMemcpyDeviceToHost, c.stream));
    FB_CUDA(cudaStreamSynchronize(c.stream));
    double v;
    std::memcpy(&v, &h, 8);
    return v;
}

}  // namespace fb
