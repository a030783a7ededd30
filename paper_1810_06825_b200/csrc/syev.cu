// K5: the l x l symmetric eigenproblem of eig_svd (dense_kernels.hpp:159-161,
// Eigen's SelfAdjointEigenSolver in the reference) for l <= kEigMax.
//
// cuSOLVER's syevd spends ~1.9 ms on a 200 x 200 matrix, almost all of it
// launch and host round-trip overhead. This solver is three kernels (the
// default for l <= 232; latency-bound in the single-CTA tridiagonalisation):
//   E1 k_sytrd  one CTA: Householder tridiagonalisation with the packed lower
//               triangle resident in shared memory (LAPACK dsytd2 order);
//   E2 k_stedc  one CTA: divide and conquer on the tridiagonal (Cuppen's
//               rank-one tearing; leaves by implicit QL with Wilkinson shifts,
//               one warp per leaf; the merges of one level run concurrently,
//               each on its own group of warps; LAPACK-style deflation, the
//               secular equation solved per root by one warp with the
//               two-pole ("middle way") rational model under a bisection
//               bracket, and Gu-Eisenstat's recomputed z so the merged
//               eigenvectors are orthogonal to working precision);
//   E3 k_ormtr  one warp per eigenvector: V = H_0 ... H_{n-3} Z.
// Any non-convergence raises a flag and the caller falls back to cuSOLVER.
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace fb {
namespace {

constexpr int kEigMax = 232;
const int kNoConvCode = kErrEigNoConv;  // n(n+1)/2 doubles fit one CTA's shared memory
constexpr int kET = 1024;
constexpr int kLeafMax = 32;

__device__ __forceinline__ int pk(int i, int j, int n) { return j * n - (j * (j - 1)) / 2 + (i - j); }

// block-wide sum, same order on every thread (deterministic), result to all
__device__ double block_sum(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
    return s;
}

// ---------------------------------------------------------------- E1
// Packed lower triangle, row-major: A[i][k] (k <= i) at i(i+1)/2 + k.
__device__ __forceinline__ int rp(int i) { return (i * (i + 1)) >> 1; }

constexpr int kST = 512;  // k_sytrd threads: 128 registers each for the lane-resident slices
constexpr int kSW = kST / 32;

// every warp reduces the kSW per-warp partials itself (same order everywhere)
__device__ __forceinline__ double warp_total(const double* red) {
    const int lane = threadIdx.x & 31;
    double v = lane < kSW ? red[lane] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr size_t kSmemMax = 226 * 1024;  // dynamic, next to the static reduction arrays
// the kSW x n column partials of (B) fit next to the packed matrix
__host__ __device__ constexpr bool sytrd_colp(int n) {
    return sizeof(double) * (size_t(n) * (n + 1) / 2 + 2 * kEigMax + kSW * size_t(n)) <= kSmemMax;
}
__host__ __device__ constexpr size_t sytrd_smem(int n) {
    return sizeof(double) * (size_t(n) * (n + 1) / 2 + 2 * kEigMax + (sytrd_colp(n) ? kSW * size_t(n) : 0));
}
// k_sytrd_fused: packed matrix, double-buffered v and w, column partials
__host__ __device__ constexpr bool sytrd_fused_fits(int n) {
    return sizeof(double) * (size_t(n) * (n + 1) / 2 + 4 * kEigMax + kSW * size_t(n)) <= kSmemMax;
}
__host__ __device__ constexpr size_t sytrd_fused_smem(int n) {
    return sizeof(double) * (size_t(n) * (n + 1) / 2 + 4 * kEigMax + kSW * size_t(n));
}

// Per column: (A) reflector from the norm partials of the previous step,
// (B) p = tau A22 v with the partials of p^T v, (C) w, (D) A22 -= v w^T +
// w v^T with the norm partials of the next column. With the column partials
// (n <= ~215) every stored element is read once in (B) and v, w live in
// registers (lane-resident slices k = lane + 32 m).
__global__ void __launch_bounds__(kST, 1)
k_sytrd(const double* __restrict__ B, int n, double* __restrict__ Hv, double* __restrict__ tau,
        double* __restrict__ dg, double* __restrict__ eo, long long* __restrict__ clk) {
    extern __shared__ double sm[];
    double* A = sm;                    // packed lower, row-major
    double* v = A + rp(n);             // Householder vector (v[0] = 1)
    double* w = v + kEigMax;           // p, then w
    double* colp = sytrd_colp(n) ? w + kEigMax : nullptr;  // kSW x n column partials of p
    __shared__ double redA[32], redB[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = warp; i < n; i += kSW)
        for (int k = lane; k <= i; k += 32) A[rp(i) + k] = B[k + size_t(i) * n];  // B symmetric
    __syncthreads();
    {   // norm partials of column 0 below its subdiagonal entry
        double ps = 0.0;
        for (int i = 2 + warp; i < n; i += kSW) {
            const double x = A[rp(i)];
            ps = fma(x, x, ps);
        }
        if (lane == 0) redA[warp] = ps;
    }
    __syncthreads();
    for (int j = 0; j + 2 < n; ++j) {
        const int t = n - j - 1;
        const bool tim = clk && j == 20 && tid == 0;
        if (tim) clk[140] = clock64();
        // (A) reflector
        const double xnorm2 = warp_total(redA);
        const double alpha = A[rp(j + 1) + j];
        double beta = alpha, tj = 0.0, scal = 0.0;
        if (xnorm2 != 0.0) {
            beta = -copysign(sqrt(fma(alpha, alpha, xnorm2)), alpha);
            tj = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        if (tid < t) {
            const double vi = tid == 0 ? 1.0 : A[rp(j + 1 + tid) + j] * scal;
            v[tid] = vi;
            Hv[size_t(j) * n + tid] = vi;
        }
        if (tid == 0) { tau[j] = tj; eo[j] = beta; dg[j] = A[rp(j) + j]; }
        __syncthreads();
        if (tim) clk[141] = clock64();
        if (colp) {
            // (B) rows i = i0 + kSW r (r < 8) of a batch: the row part over
            // the lanes (x v[k]), the column part into lane-owned
            // accumulators (x v[i]); the 8 row sums leave the warp by a
            // transpose reduction (lane l ends with row (l >> 2) & 7)
            double vr[8], cacc[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int k = lane + 32 * m;
                vr[m] = k < t ? v[k] : 0.0;
                cacc[m] = 0.0;
            }
            for (int i0 = warp; i0 < t; i0 += 8 * kSW) {
                double a[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    a[r] = 0.0;
                    const int i = i0 + kSW * r;
                    if (i < t) {
                        const double* row = A + rp(j + 1 + i) + (j + 1);
                        const double vi = v[i];
#pragma unroll
                        for (int m = 0; m < 8; ++m) {
                            if (32 * m > i) break;
                            const int k = lane + 32 * m;
                            if (k <= i) {
                                const double x = row[k];
                                a[r] = fma(x, vr[m], a[r]);
                                if (k < i) cacc[m] = fma(x, vi, cacc[m]);
                            }
                        }
                    }
                }
                {
                    const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double snd = h4 ? a[q] : a[q + 4], keep = h4 ? a[q + 4] : a[q];
                        a[q] = keep + __shfl_xor_sync(0xffffffffu, snd, 16);
                    }
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const double snd = h3 ? a[q] : a[q + 2], keep = h3 ? a[q + 2] : a[q];
                        a[q] = keep + __shfl_xor_sync(0xffffffffu, snd, 8);
                    }
                    {
                        const double snd = h2 ? a[0] : a[1], keep = h2 ? a[1] : a[0];
                        a[0] = keep + __shfl_xor_sync(0xffffffffu, snd, 4);
                    }
                    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
                    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
                    const int i = i0 + kSW * ((lane >> 2) & 7);
                    if ((lane & 3) == 0 && i < t) w[i] = a[0];
                }
            }
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int k = lane + 32 * m;
                if (k < t) colp[warp * n + k] = cacc[m];
            }
            __syncthreads();
            double pv = 0.0;
            if (tid < t) {
                double a = w[tid];
#pragma unroll
                for (int q = 0; q < kSW; ++q) a += colp[q * n + tid];
                a *= tj;
                w[tid] = a;
                pv = a * v[tid];
            }
            for (int o = 16; o; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
            if (lane == 0) redB[warp] = pv;
            __syncthreads();
            if (tim) clk[142] = clock64();
            // (C) w = p - (tau/2)(p^T v) v, each warp its own register slice
            const double alpha2 = -0.5 * tj * warp_total(redB);
            double wr[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int k = lane + 32 * m;
                wr[m] = k < t ? fma(alpha2, vr[m], w[k]) : 0.0;
            }
            __syncthreads();  // every warp has read p before w is overwritten
            if (tid < t) w[tid] = fma(alpha2, v[tid], w[tid]);
            __syncthreads();
            if (tim) clk[143] = clock64();
            // (D) rank-2 update from the register slices
            double ps = 0.0;
            for (int i = warp; i < t; i += kSW) {
                const double vi = v[i], wi = w[i];
                double* row = A + rp(j + 1 + i) + (j + 1);
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    if (32 * m > i) break;
                    const int k = lane + 32 * m;
                    if (k <= i) {
                        const double x = row[k] - fma(vi, wr[m], wi * vr[m]);
                        row[k] = x;
                        if (m == 0 && lane == 0 && i >= 2) ps = fma(x, x, ps);
                    }
                }
            }
            if (lane == 0) redA[warp] = ps;
        } else {
            // (B) p = tau * A22 v: one warp per row (two rows in flight), lanes
            // over the row and its column
            double pv = 0.0;
            for (int i0 = warp; i0 < t; i0 += 2 * kSW) {
                const int i1 = i0 + kSW;
                double a0 = 0.0, a1 = 0.0;
                for (int k = lane; k < t; k += 32) {
                    const int K = j + 1 + k;
                    const double vk = v[k];
                    a0 = fma(k <= i0 ? A[rp(j + 1 + i0) + K] : A[rp(K) + j + 1 + i0], vk, a0);
                    if (i1 < t) a1 = fma(k <= i1 ? A[rp(j + 1 + i1) + K] : A[rp(K) + j + 1 + i1], vk, a1);
                }
                for (int o = 16; o; o >>= 1) {
                    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
                    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
                }
                a0 *= tj;
                a1 *= tj;
                if (lane == 0) {
                    w[i0] = a0;
                    if (i1 < t) w[i1] = a1;
                }
                pv = fma(a0, v[i0], pv);
                if (i1 < t) pv = fma(a1, v[i1], pv);
            }
            if (lane == 0) redB[warp] = pv;
            __syncthreads();
            if (tim) clk[142] = clock64();
            // (C) w = p - (tau/2)(p^T v) v
            {
                const double alpha2 = -0.5 * tj * warp_total(redB);
                if (tid < t) w[tid] = fma(alpha2, v[tid], w[tid]);
            }
            __syncthreads();
            if (tim) clk[143] = clock64();
            // (D) rank-2 update; lane 0 of the row's warp sees the next column
            double ps = 0.0;
            for (int i = warp; i < t; i += kSW) {
                const double vi = v[i], wi = w[i];
                double* row = A + rp(j + 1 + i) + (j + 1);
                for (int k = lane; k <= i; k += 32) {
                    const double x = row[k] - fma(vi, w[k], wi * v[k]);
                    row[k] = x;
                    if (k == 0 && i >= 2) ps = fma(x, x, ps);
                }
            }
            if (lane == 0) redA[warp] = ps;
        }
        __syncthreads();
        if (tim) clk[144] = clock64();
    }
    if (tid == 0) {
        if (n >= 2) {
            dg[n - 2] = A[rp(n - 2) + n - 2];
            dg[n - 1] = A[rp(n - 1) + n - 1];
            eo[n - 2] = A[rp(n - 1) + n - 2];
            tau[n - 2] = 0.0;
        } else {
            dg[0] = A[0];
        }
    }
}

// Fused variant (n <= ~213, the column-partial layout): the rank-2 update of
// step j and the symmetric product of step j + 1 are one pass over the
// trailing matrix, so every stored element is loaded and stored once per
// column instead of being read by (B) and read + written again by (D).
// Per column j:
//   (D1) column j + 1 updated with (v_j, w_j) and its norm partials;
//   (A)  reflector v_{j+1} (double-buffered v, w);
//   (DB) rows/columns >= j + 2: a -= v_j w_j^T + w_j v_j^T, and in the same
//        visit p += a v_{j+1} (row part over the lanes, column part into
//        lane-owned accumulators);
//   (C)  w_{j+1} = p - (tau/2)(p^T v) v.
// Same arithmetic per element as k_sytrd; the symmetric-product sums run in
// the same per-warp / per-lane order.
template <bool UPD, bool SYM>
__device__ __forceinline__ void sytrd_pass(double* __restrict__ A, int c0, int n, const double* __restrict__ vo,
                                           const double* __restrict__ wo, const double* __restrict__ vn,
                                           double* __restrict__ pw, double* __restrict__ colp) {
    // trailing block: rows / columns c0 .. n-1 (relative index i', k);
    // (vo, wo) are indexed relative to c0 - 1 (the step being applied),
    // vn relative to c0 (the step whose product is formed)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t2 = n - c0;
    double vr[8], wr[8], nr[8], cacc[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const int k = lane + 32 * m;
        vr[m] = UPD && k < t2 ? vo[k + 1] : 0.0;
        wr[m] = UPD && k < t2 ? wo[k + 1] : 0.0;
        nr[m] = SYM && k < t2 ? vn[k] : 0.0;
        cacc[m] = 0.0;
    }
    for (int i0 = warp; i0 < t2; i0 += 8 * kSW) {
        double a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            a[r] = 0.0;
            const int i = i0 + kSW * r;
            if (i < t2) {
                double* row = A + rp(c0 + i) + c0;
                const double vi = UPD ? vo[i + 1] : 0.0, wi = UPD ? wo[i + 1] : 0.0;
                const double ni = SYM ? vn[i] : 0.0;
                double x[8];
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int k = lane + 32 * m;
                    x[m] = (32 * m <= i && k <= i) ? row[k] : 0.0;
                }
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    if (32 * m > i) break;
                    const int k = lane + 32 * m;
                    if (k <= i) {
                        double y = x[m];
                        if (UPD) {
                            y = y - fma(vi, wr[m], wi * vr[m]);
                            row[k] = y;
                        }
                        if (SYM) {
                            a[r] = fma(y, nr[m], a[r]);
                            if (k < i) cacc[m] = fma(y, ni, cacc[m]);
                        }
                    }
                }
            }
        }
        if (SYM) {
            const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double snd = h4 ? a[q] : a[q + 4], keep = h4 ? a[q + 4] : a[q];
                a[q] = keep + __shfl_xor_sync(0xffffffffu, snd, 16);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const double snd = h3 ? a[q] : a[q + 2], keep = h3 ? a[q + 2] : a[q];
                a[q] = keep + __shfl_xor_sync(0xffffffffu, snd, 8);
            }
            {
                const double snd = h2 ? a[0] : a[1], keep = h2 ? a[1] : a[0];
                a[0] = keep + __shfl_xor_sync(0xffffffffu, snd, 4);
            }
            a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
            a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
            const int i = i0 + kSW * ((lane >> 2) & 7);
            if ((lane & 3) == 0 && i < t2) pw[i] = a[0];
        }
    }
    if (SYM) {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int k = lane + 32 * m;
            if (k < t2) colp[warp * n + k] = cacc[m];
        }
    }
}

__global__ void __launch_bounds__(kST, 1)
k_sytrd_fused(const double* __restrict__ B, int n, double* __restrict__ Hv, double* __restrict__ tau,
              double* __restrict__ dg, double* __restrict__ eo, long long* __restrict__ clk) {
    extern __shared__ double sm[];
    double* A = sm;                     // packed lower, row-major
    double* vb = A + rp(n);             // [2][kEigMax] Householder vectors (v[0] = 1)
    double* wb = vb + 2 * kEigMax;      // [2][kEigMax] p, then w
    double* colp = wb + 2 * kEigMax;    // kSW x n column partials of p
    __shared__ double redA[32], redB[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = warp; i < n; i += kSW)
        for (int k = lane; k <= i; k += 32) A[rp(i) + k] = B[k + size_t(i) * n];  // B symmetric
    __syncthreads();
    if (n < 3) {
        if (tid == 0) {
            if (n == 2) {
                dg[0] = A[0]; dg[1] = A[2]; eo[0] = A[1]; tau[0] = 0.0;
            } else if (n == 1) {
                dg[0] = A[0];
            }
        }
        return;
    }
    // reflector of column j into (vb + buf): norm partials in redA
    auto reflector = [&](int j, int buf, double& tj) {
        const int t = n - j - 1;
        const double xnorm2 = warp_total(redA);
        const double alpha = A[rp(j + 1) + j];
        double beta = alpha, scal = 0.0;
        tj = 0.0;
        if (xnorm2 != 0.0) {
            beta = -copysign(sqrt(fma(alpha, alpha, xnorm2)), alpha);
            tj = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        if (tid < t) {
            const double vi = tid == 0 ? 1.0 : A[rp(j + 1 + tid) + j] * scal;
            vb[buf * kEigMax + tid] = vi;
            Hv[size_t(j) * n + tid] = vi;
        }
        if (tid == 0) { tau[j] = tj; eo[j] = beta; dg[j] = A[rp(j) + j]; }
    };
    // p from the partials, p^T v, then w = p - (tau/2)(p^T v) v, in place
    auto make_w = [&](int j, int buf, double tj) {
        const int t = n - j - 1;
        double* w = wb + buf * kEigMax;
        const double* v = vb + buf * kEigMax;
        double a = 0.0, pv = 0.0;
        if (tid < t) {
            a = w[tid];
#pragma unroll
            for (int q = 0; q < kSW; ++q) a += colp[q * n + tid];
            a *= tj;
            pv = a * v[tid];
        }
        for (int o = 16; o; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
        if (lane == 0) redB[warp] = pv;
        __syncthreads();
        const double alpha2 = -0.5 * tj * warp_total(redB);
        if (tid < t) w[tid] = fma(alpha2, v[tid], a);
        __syncthreads();
    };
    {   // norm partials of column 0 below its subdiagonal entry
        double ps = 0.0;
        for (int i = 2 + warp; i < n; i += kSW) {
            const double x = A[rp(i)];
            ps = fma(x, x, ps);
        }
        if (lane == 0) redA[warp] = ps;
    }
    __syncthreads();
    double tj;
    reflector(0, 0, tj);
    __syncthreads();
    sytrd_pass<false, true>(A, 1, n, nullptr, nullptr, vb, wb, colp);
    __syncthreads();
    make_w(0, 0, tj);
    for (int j = 0; j + 2 < n; ++j) {
        const int cur = j & 1, nxt = cur ^ 1;
        const int t = n - j - 1;
        const double* vo = vb + cur * kEigMax;
        const double* wo = wb + cur * kEigMax;
        const bool tim = clk && j == 20 && tid == 0;
        if (tim) clk[140] = clock64();
        {   // (D1) column j + 1 (relative row tid, column 0) and its norm partials
            double ps = 0.0;
            if (tid < t) {
                double* e = A + rp(j + 1 + tid) + (j + 1);
                const double x = *e - fma(vo[tid], wo[0], wo[tid] * vo[0]);
                *e = x;
                if (tid >= 2) ps = x * x;
            }
            for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            if (lane == 0) redA[warp] = ps;
        }
        __syncthreads();
        if (tim) clk[141] = clock64();
        if (j + 3 < n) {
            double tn;
            reflector(j + 1, nxt, tn);
            __syncthreads();
            if (tim) clk[142] = clock64();
            sytrd_pass<true, true>(A, j + 2, n, vo, wo, vb + nxt * kEigMax, wb + nxt * kEigMax, colp);
            __syncthreads();
            if (tim) clk[143] = clock64();
            make_w(j + 1, nxt, tn);
        } else {
            sytrd_pass<true, false>(A, j + 2, n, vo, wo, nullptr, nullptr, nullptr);
            __syncthreads();
        }
        if (tim) clk[144] = clock64();
    }
    if (tid == 0) {
        dg[n - 2] = A[rp(n - 2) + n - 2];
        dg[n - 1] = A[rp(n - 1) + n - 1];
        eo[n - 2] = A[rp(n - 1) + n - 2];
        tau[n - 2] = 0.0;
    }
}

// ---------------------------------------------------------------- E2
struct LeafWs {
    double z[kLeafMax][kLeafMax + 1];  // row-major, lane = row
    double d[kLeafMax], e[kLeafMax], rc[kLeafMax], rs[kLeafMax];
    int perm[kLeafMax];
};

// Implicit QL with Wilkinson shifts on a b x b tridiagonal (b <= 32): lane 0
// runs the scalar recurrence and records the rotations of a sweep, then every
// lane applies them to its row of Z. Eigenvalues left in d (unsorted).
__device__ bool leaf_ql(int b, LeafWs& w, int lane) {
    for (int c = 0; c < b; ++c)
        if (lane < b) w.z[lane][c] = lane == c ? 1.0 : 0.0;
    if (lane == 0) w.e[b - 1] = 0.0;
    __syncwarp();
    for (int l = 0; l < b; ++l) {
        for (int iter = 0;; ++iter) {
            int m = l, rlo = l;
            if (lane == 0) {
                for (m = l; m < b - 1; ++m) {
                    const double dd = fabs(w.d[m]) + fabs(w.d[m + 1]);
                    if (fabs(w.e[m]) <= DBL_EPSILON * dd) break;
                }
                if (m != l && iter < 60) {
                    double g = (w.d[l + 1] - w.d[l]) / (2.0 * w.e[l]);
                    double r = sqrt(fma(g, g, 1.0));
                    g = w.d[m] - w.d[l] + w.e[l] / (g + copysign(r, g));
                    double s = 1.0, c = 1.0, p = 0.0;
                    int i;
                    for (i = m - 1; i >= l; --i) {
                        const double f = s * w.e[i], bb = c * w.e[i];
                        r = sqrt(fma(f, f, g * g));  // |f|, |g| ~ eigenvalue scale: no overflow
                        w.e[i + 1] = r;
                        if (r == 0.0) {
                            w.d[i + 1] -= p;
                            w.e[m] = 0.0;
                            break;
                        }
                        const double ri = 1.0 / r;
                        s = f * ri;
                        c = g * ri;
                        g = w.d[i + 1] - p;
                        r = (w.d[i] - g) * s + 2.0 * c * bb;
                        p = s * r;
                        w.d[i + 1] = g + p;
                        g = c * r - bb;
                        w.rc[i] = c;
                        w.rs[i] = s;
                    }
                    rlo = i + 1;
                    if (!(r == 0.0 && i >= l)) {
                        w.d[l] -= p;
                        w.e[l] = g;
                        w.e[m] = 0.0;
                    }
                }
            }
            m = __shfl_sync(0xffffffffu, m, 0);
            rlo = __shfl_sync(0xffffffffu, rlo, 0);
            __syncwarp();
            if (m == l) break;
            if (iter >= 60) return false;
            if (lane < b)
                for (int i = m - 1; i >= rlo; --i) {
                    const double f = w.z[lane][i + 1];
                    w.z[lane][i + 1] = w.rs[i] * w.z[lane][i] + w.rc[i] * f;
                    w.z[lane][i] = w.rc[i] * w.z[lane][i] - w.rs[i] * f;
                }
            __syncwarp();
        }
    }
    return true;
}

struct MergeWs {
    double dfull[kEigMax], zfull[kEigMax], ds[kEigMax], zs[kEigMax];
    double dk[kEigMax], zk[kEigMax], zh[kEigMax], tauk[kEigMax];
    double ddf[kEigMax], vals[kEigMax];
    double rc[kEigMax], rs[kEigMax];
    int cs[kEigMax], ck[kEigMax], cdf[kEigMax], orgk[kEigMax], ri[kEigMax], rj[kEigMax], pos[kEigMax];
    struct Scal {
        int k, ndf, nrot, sgn, ok;
        double rho, zsum2, zn2, dmax;
    } sc[16];  // per concurrent merge
};

// A group of whole warps working on one merge; `bar.sync id, nt` is its barrier.
struct Grp {
    int t, nt, id;
};
__device__ __forceinline__ void gsync(const Grp& g) { asm volatile("bar.sync %0, %1;\n" ::"r"(g.id), "r"(g.nt)); }

// The deferred top-level merge, finished by E3: output column c is
// sum_j Z[:, ck[j]] U[j][src[c]] (src[c] < k) or Z[:, cdf[src[c] - k]].
struct TopPlan {
    int k;
    int ck[kEigMax], cdf[kEigMax], src[kEigMax];
};

constexpr int kSecLanes = 8;  // lanes per secular root
constexpr int kLeaves = 16;
constexpr size_t kUsMax = kLeaves * sizeof(LeafWs) / sizeof(double);  // U staged over the leaf workspace

__device__ __forceinline__ double group_sum(double v, unsigned mask) {
    for (int o = kSecLanes / 2; o; o >>= 1) v += __shfl_xor_sync(mask, v, o);
    return v;
}

// Convergence factor of the secular solver: |f| <= c eps (1 + rho sum |terms|),
// LAPACK dlaed4's test up to its constant. (An earlier factor c = 8 k, up to
// 1600 at n = 200, left the roots loose enough that the eigenvectors, and
// through eig_svd's S^-1 the power iteration's basis, lost ~1.5x in subspace
// accuracy against the long-double arbiter at C2.) Set per launch.
__constant__ double c_sec_tol = 8.0;

// Root i of 1 + rho sum_j z_j^2 / (d_j - lambda) = 0 (d ascending, rho > 0),
// by a group of kSecLanes lanes: lambda = d_org + tau.
__device__ bool secular_root(int i, int k, const double* dk, const double* zk, double rho, double zsum2,
                             int sl, unsigned mask, int& org_out, double& tau_out) {
    const bool last = i == k - 1;
    // f and the pole-split derivatives at the bracket midpoint (relative to d_i)
    const double w = last ? rho * zsum2 : dk[i + 1] - dk[i];
    const double mid = 0.5 * w;
    double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0, eabs = 0.0;
    for (int j = sl; j < k; j += kSecLanes) {
        const double del = (dk[j] - dk[i]) - mid;
        const double inv = 1.0 / del;
        const double t = zk[j] * zk[j] * inv;
        if (j <= i) { psi += t; dpsi = fma(t, inv, dpsi); }
        else { phi += t; dphi = fma(t, inv, dphi); }
        eabs += fabs(t);
    }
    psi = group_sum(psi, mask); dpsi = group_sum(dpsi, mask);
    phi = group_sum(phi, mask); dphi = group_sum(dphi, mask);
    eabs = group_sum(eabs, mask);
    double f = 1.0 + rho * (psi + phi);
    int org;
    double lo, hi, tau;
    if (last || f >= 0.0) { org = i; lo = 0.0; hi = mid; tau = mid; }
    else { org = i + 1; lo = mid - w; hi = 0.0; tau = mid - w; }
    if (last) { hi = w; }
    const double dorg = dk[org];
    const double di = dk[i] - dorg, di1 = last ? 0.0 : dk[i + 1] - dorg;
    bool ok = false;
    for (int it = 0; it < 200; ++it) {
        if (it > 0) {
            psi = dpsi = phi = dphi = eabs = 0.0;
            for (int j = sl; j < k; j += kSecLanes) {
                const double del = (dk[j] - dorg) - tau;
                const double inv = 1.0 / del;
                const double t = zk[j] * zk[j] * inv;
                if (j <= i) { psi += t; dpsi = fma(t, inv, dpsi); }
                else { phi += t; dphi = fma(t, inv, dphi); }
                eabs += fabs(t);
            }
            psi = group_sum(psi, mask); dpsi = group_sum(dpsi, mask);
            phi = group_sum(phi, mask); dphi = group_sum(dphi, mask);
            eabs = group_sum(eabs, mask);
            f = 1.0 + rho * (psi + phi);
        }
        if (fabs(f) <= c_sec_tol * DBL_EPSILON * (1.0 + rho * eabs)) { ok = true; break; }
        if (f < 0.0) lo = tau; else hi = tau;
        if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) { ok = true; break; }
        // two-pole rational model through (f, f') at tau, solved for the step eta
        const double Di = di - tau;
        double eta = 0.0;
        bool good = false;
        if (last) {
            const double sp = rho * dpsi * Di * Di;
            const double c = f - sp / Di;
            if (c != 0.0) { eta = Di + sp / c; good = true; }
        } else {
            const double Di1 = di1 - tau;
            const double sp = rho * dpsi * Di * Di, sf = rho * dphi * Di1 * Di1;
            const double c = f - sp / Di - sf / Di1;
            const double bq = c * (Di + Di1) + sp + sf, cq = f * Di * Di1;
            if (c == 0.0) {
                if (bq != 0.0) { eta = cq / bq; good = true; }
            } else {
                const double disc = bq * bq - 4.0 * c * cq;
                if (disc >= 0.0) {
                    const double q = 0.5 * (bq + copysign(sqrt(disc), bq));
                    const double e1 = q / c, e2 = q != 0.0 ? cq / q : e1;
                    const bool in1 = tau + e1 > lo && tau + e1 < hi, in2 = tau + e2 > lo && tau + e2 < hi;
                    if (in1 && in2) eta = fabs(e1) < fabs(e2) ? e1 : e2;
                    else eta = in1 ? e1 : e2;
                    good = in1 || in2;
                }
            }
        }
        const double tn = tau + eta;
        tau = (good && tn > lo && tn < hi) ? tn : 0.5 * (lo + hi);
    }
    org_out = org;
    tau_out = tau;
    return ok;
}

__device__ __forceinline__ void stamp(long long* clk, int slot) {
    if (clk && threadIdx.x == 0) clk[slot] = clock64();
}

// merge of the adjacent blocks [s0, s0 + n1) and [s0 + n1, s0 + n1 + n2).
// top != nullptr: the last merge; its eigenvector product is left to E3.
// merge of the adjacent blocks [s0, s0 + n1) and [s0 + n1, s0 + n1 + n2) by
// the thread group G (merges of one level run concurrently on disjoint slices
// of the workspaces: arrays at [s0, s0 + sz), U and Tmp at row s0 * n).
// top != nullptr: the last merge; its eigenvector product is left to E3.
__device__ bool merge_blocks(int n, int s0, int n1, int n2, double* Dc, const double* Eo, double* Z, double* TmpAll,
                             double* UtAll, double* Us, size_t us_cap, MergeWs& MW, int gi, TopPlan* top,
                             const Grp& G) {
    const int tid = G.t, NT = G.nt;
    const int sz = n1 + n2, p = s0 + n1;
    double *dfull = MW.dfull + s0, *zfull = MW.zfull + s0, *ds = MW.ds + s0, *zs = MW.zs + s0;
    double *dk = MW.dk + s0, *zk = MW.zk + s0, *zh = MW.zh + s0, *tauk = MW.tauk + s0;
    double *ddf = MW.ddf + s0, *vals = MW.vals + s0, *rcv = MW.rc + s0, *rsv = MW.rs + s0;
    int *cs = MW.cs + s0, *ck = MW.ck + s0, *cdf = MW.cdf + s0, *orgk = MW.orgk + s0;
    int *ri = MW.ri + s0, *rj = MW.rj + s0, *pos = MW.pos + s0;
    MergeWs::Scal& sc = MW.sc[gi];
    double* Tmp = TmpAll + size_t(s0) * n;
    double* Ut = UtAll + size_t(s0) * n;
    const double rho0 = Eo[p - 1];
    const int sgn = rho0 < 0.0 ? -1 : 1;
    for (int j = tid; j < sz; j += NT) {
        zfull[j] = j < n1 ? Z[(p - 1) + size_t(s0 + j) * n] : Z[p + size_t(s0 + j) * n];
        dfull[j] = Dc[s0 + j];
    }
    gsync(G);
    // sorted order of sgn * d: position = rank in its own block + rank in the
    // other (binary search; block 1 first on ties)
    for (int j = tid; j < sz; j += NT) {
        const bool b1 = j < n1;
        const double key = sgn * dfull[j];
        const int own = b1 ? (sgn > 0 ? j : n1 - 1 - j) : (sgn > 0 ? j - n1 : sz - 1 - j);
        const int o0 = b1 ? n1 : 0, on = b1 ? n2 : n1;
        int lo = 0, hi = on;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const int idx = o0 + (sgn > 0 ? mid : on - 1 - mid);
            const double okey = sgn * dfull[idx];
            if (b1 ? okey < key : okey <= key) lo = mid + 1; else hi = mid;
        }
        const int q = own + lo;
        ds[q] = key;
        zs[q] = zfull[j];
        cs[q] = j;
    }
    if (tid < 32) {
        double z2 = 0.0, dm = 0.0;
        for (int j = tid; j < sz; j += 32) { z2 = fma(zfull[j], zfull[j], z2); dm = fmax(dm, fabs(dfull[j])); }
        for (int o = 16; o; o >>= 1) {
            z2 += __shfl_xor_sync(0xffffffffu, z2, o);
            dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
        }
        if (tid == 0) { sc.zn2 = z2; sc.dmax = dm; sc.ok = 1; }
    }
    gsync(G);
    if (tid == 0) {
        // deflation (LAPACK dlaed2 rules) over the sorted sequence; the
        // rotation test only runs for nearly equal neighbours (|cs| <= 1/2)
        const double rho = fabs(rho0) * sc.zn2;
        const double zinv = 1.0 / sqrt(sc.zn2);
        const double tol = 8.0 * DBL_EPSILON * fmax(sc.dmax, rho);
        int prev = -1;
        double dprev = 0.0, zprev = 0.0;
        int k = 0, ndf = 0, nrot = 0;
        for (int q = 0; q < sz; ++q) {
            const int j = cs[q];
            const double dj = ds[q], zj = zs[q] * zinv;
            if (rho * fabs(zj) <= tol) {
                ddf[ndf] = dj; cdf[ndf] = j; ++ndf;
                continue;
            }
            if (prev >= 0 && fabs(dj - dprev) <= 2.0 * tol) {
                const double r = sqrt(fma(zprev, zprev, zj * zj));
                const double c = zj / r, sn = zprev / r;
                if (fabs((dj - dprev) * c * sn) <= tol) {
                    ri[nrot] = prev; rj[nrot] = j; rcv[nrot] = c; rsv[nrot] = sn; ++nrot;
                    const double dp = c * c * dprev + sn * sn * dj, dn = sn * sn * dprev + c * c * dj;
                    ddf[ndf] = dp; cdf[ndf] = prev; ++ndf;
                    prev = j; dprev = dn; zprev = r;
                    continue;
                }
            }
            if (prev >= 0) { dk[k] = dprev; zk[k] = zprev; ck[k] = prev; ++k; }
            prev = j; dprev = dj; zprev = zj;
        }
        if (prev >= 0) { dk[k] = dprev; zk[k] = zprev; ck[k] = prev; ++k; }
        double zsum = 0.0;
        for (int j = 0; j < k; ++j) zsum = fma(zk[j], zk[j], zsum);
        sc.k = k; sc.ndf = ndf; sc.nrot = nrot; sc.sgn = sgn; sc.rho = rho; sc.zsum2 = zsum;
    }
    gsync(G);
    const int k = sc.k, ndf = sc.ndf, nrot = sc.nrot;
    if (nrot)
        for (int r = tid; r < sz; r += NT) {
            double* zr = Z + (s0 + r);
            for (int t = 0; t < nrot; ++t) {
                double& qi = zr[size_t(s0 + ri[t]) * n];
                double& qj = zr[size_t(s0 + rj[t]) * n];
                const double x = qi, y = qj, c = rcv[t], sn = rsv[t];
                qi = c * x - sn * y;
                qj = sn * x + c * y;
            }
        }
    {   // secular roots, kSecLanes lanes each
        const int g8 = tid / kSecLanes, sl = tid % kSecLanes;
        const unsigned mask = 0xffu << ((threadIdx.x & 31) & ~(kSecLanes - 1));
        for (int i = g8; i < k; i += NT / kSecLanes) {
            int org;
            double tau;
            const bool r = secular_root(i, k, dk, zk, sc.rho, sc.zsum2, sl, mask, org, tau);
            if (sl == 0) { orgk[i] = org; tauk[i] = tau; }
            if (!r) sc.ok = 0;
        }
    }
    gsync(G);
    if (!sc.ok) return false;
    const int lane = tid & 31, warp = tid >> 5, nw = NT >> 5;
    // Gu-Eisenstat zhat, one warp per j, lanes split the factors (fixed tree)
    for (int j = warp; j < k; j += nw) {
        const double dj = dk[j];
        double prod = 1.0;
        for (int i = lane; i < k - 1; i += 32) {
            const double lam = (dk[orgk[i]] - dj) + tauk[i];
            prod *= lam / (i < j ? (dk[i] - dj) : (dk[i + 1] - dj));
        }
        for (int o = 16; o; o >>= 1) prod *= __shfl_xor_sync(0xffffffffu, prod, o);
        prod *= ((dk[orgk[k - 1]] - dj) + tauk[k - 1]) / sc.rho;
        if (lane == 0) zh[j] = copysign(sqrt(fabs(prod)), zk[j]);
    }
    gsync(G);
    double* U = (top || size_t(k) * k > us_cap) ? Ut : Us;
    for (int i = warp; i < k; i += nw) {
        const double dorg = dk[orgk[i]], tau = tauk[i];
        double nrm = 0.0;
        for (int j = lane; j < k; j += 32) {
            const double u = zh[j] / ((dk[j] - dorg) - tau);
            nrm = fma(u, u, nrm);
        }
        for (int o = 16; o; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
        const double inv = 1.0 / sqrt(nrm);
        for (int j = lane; j < k; j += 32) U[size_t(j) * k + i] = (zh[j] / ((dk[j] - dorg) - tau)) * inv;
        if (lane == 0) vals[i] = sc.sgn * (dorg + tau);
    }
    for (int t = tid; t < ndf; t += NT) vals[k + t] = sc.sgn * ddf[t];
    gsync(G);
    for (int a = tid; a < sz; a += NT) {  // ascending order of all sz values (rank sort)
        const double va = vals[a];
        int r = 0;
        for (int b = 0; b < sz; ++b) {
            const double vb = vals[b];
            r += (vb < va) || (vb == va && b < a);
        }
        pos[a] = r;
    }
    gsync(G);
    if (top) {  // last merge: hand the product to E3
        for (int a = tid; a < sz; a += NT) {
            top->src[pos[a]] = a;
            if (a < k) top->ck[a] = ck[a];
            else top->cdf[a - k] = cdf[a - k];
            Dc[s0 + pos[a]] = vals[a];
        }
        if (tid == 0) top->k = k;
        gsync(G);
        return true;
    }
    const int ngrp = (k + 7) / 8;
    for (int e = tid; e < sz * ngrp; e += NT) {
        const int r = e % sz, a0 = (e / sz) * 8;
        double acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0;
        const double* zr = Z + (s0 + r);
        for (int j = 0; j < k; ++j) {
            const double zv = zr[size_t(s0 + ck[j]) * n];
            const double* u = U + size_t(j) * k + a0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (a0 + q < k) acc[q] = fma(zv, u[q], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (a0 + q < k) Tmp[r + size_t(pos[a0 + q]) * sz] = acc[q];
    }
    for (int e = tid; e < sz * ndf; e += NT) {
        const int r = e % sz, t = e / sz;
        Tmp[r + size_t(pos[k + t]) * sz] = Z[(s0 + r) + size_t(s0 + cdf[t]) * n];
    }
    gsync(G);
    for (int e = tid; e < sz * sz; e += NT) {
        const int r = e % sz, c = e / sz;
        Z[(s0 + r) + size_t(s0 + c) * n] = Tmp[e];
    }
    for (int a = tid; a < sz; a += NT) Dc[s0 + pos[a]] = vals[a];
    gsync(G);
    return true;
}

__global__ void __launch_bounds__(kET, 1)
k_stedc(int n, const double* __restrict__ dg, const double* __restrict__ eo, double* __restrict__ Z,
        double* __restrict__ Tmp, double* __restrict__ Ut, double* __restrict__ Dout, TopPlan* __restrict__ top,
        int* __restrict__ info, long long* __restrict__ clk) {
    extern __shared__ __align__(16) unsigned char smraw[];
    MergeWs& M = *reinterpret_cast<MergeWs*>(smraw);
    LeafWs* L = reinterpret_cast<LeafWs*>(smraw + ((sizeof(MergeWs) + 15) / 16) * 16);
    __shared__ double Dc[kEigMax], Eo[kEigMax];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    stamp(clk, 0);
    for (int i = tid; i < n; i += kET) {
        Dc[i] = dg[i];
        Eo[i] = i + 1 < n ? eo[i] : 0.0;
    }
    for (size_t e = tid; e < size_t(n) * n; e += kET) Z[e] = 0.0;
    __syncthreads();
    const int LB = (n + kLeaves - 1) / kLeaves, nleaf = (n + LB - 1) / LB;
    if (tid == 0)
        for (int b = 1; b < nleaf; ++b) {  // Cuppen tears at the leaf boundaries
            const int p = b * LB;
            Dc[p - 1] -= Eo[p - 1];
            Dc[p] -= Eo[p - 1];
        }
    __syncthreads();
    bool ok = true;
    if (warp < nleaf) {
        LeafWs& w = L[warp];
        const int s = warp * LB, b = min(LB, n - s);
        if (lane < b) {
            w.d[lane] = Dc[s + lane];
            w.e[lane] = lane + 1 < b ? Eo[s + lane] : 0.0;
        }
        __syncwarp();
        ok = leaf_ql(b, w, lane);
        if (ok) {
            if (lane == 0) {  // ascending order (insertion sort of indices)
                for (int i = 0; i < b; ++i) w.perm[i] = i;
                for (int i = 1; i < b; ++i) {
                    const int x = w.perm[i];
                    int j = i - 1;
                    while (j >= 0 && w.d[w.perm[j]] > w.d[x]) { w.perm[j + 1] = w.perm[j]; --j; }
                    w.perm[j + 1] = x;
                }
            }
            __syncwarp();
            if (lane < b) {
                for (int c = 0; c < b; ++c) Z[(s + lane) + size_t(s + c) * n] = w.z[lane][w.perm[c]];
                Dc[s + lane] = w.d[w.perm[lane]];
            }
        }
    }
    ok = __syncthreads_and(ok);
    if (!ok) {
        if (tid == 0) atomicCAS(info, 0, kErrEigNoConv);
        return;
    }
    stamp(clk, 1);
    __shared__ int fail;
    if (tid == 0) fail = 0;
    __syncthreads();
    bool merged = false;
    int level = 0;
    for (int width = LB; width < n; width *= 2, ++level) {
        int G = 0;
        for (int s0 = 0; s0 + width < n; s0 += 2 * width) ++G;
        const bool last = 2 * width >= n;
        // warps [g * 32 / G, (g + 1) * 32 / G) merge the g-th pair
        int g = 0;
        while (g + 1 < G && ((g + 1) * 32) / G <= warp) ++g;
        const int w0 = (g * 32) / G, w1 = ((g + 1) * 32) / G;
        const Grp grp{tid - w0 * 32, (w1 - w0) * 32, 1 + g};
        const int s0 = g * 2 * width;
        const int n1 = width, n2 = min(width, n - s0 - width);
        const size_t us_cap = kUsMax / size_t(G);
        if (!merge_blocks(n, s0, n1, n2, Dc, Eo, Z, Tmp, Ut, reinterpret_cast<double*>(L) + size_t(g) * us_cap, us_cap,
                          M, g, last ? top : nullptr, grp))
            if (grp.t == 0) atomicExch(&fail, 1);
        __syncthreads();
        if (fail) {
            if (tid == 0) atomicCAS(info, 0, kErrEigNoConv);
            return;
        }
        stamp(clk, 2 + level);
        merged = merged || last;
    }
    if (!merged) {  // a single leaf: identity plan
        for (int a = tid; a < n; a += kET) { top->src[a] = a; top->cdf[a] = a; }
        if (tid == 0) top->k = 0;
    }
    for (int i = tid; i < n; i += kET) Dout[i] = Dc[i];
}

// ---------------------------------------------------------------- E3
// V = H_0 H_1 ... H_{n-3} (Z U), 8 columns per CTA: first the deferred top
// merge (kept columns: Z[:, ck] times the staged columns of U; deflated:
// copies), then the reflectors, shared by the CTA's warps and staged through
// shared memory one step ahead (cp.async).
constexpr int kOrmWarps = 8;
constexpr int kRefl = 4;  // reflectors per barrier
__global__ void __launch_bounds__(kOrmWarps * 32)
k_ormtr(const double* __restrict__ Hv, const double* __restrict__ tau, int n, const double* __restrict__ Z,
        const double* __restrict__ Ut, const TopPlan* __restrict__ top, double* __restrict__ V,
        const int* __restrict__ info) {
    __shared__ double zs[kOrmWarps][kEigMax];
    __shared__ double us[kOrmWarps][kEigMax];
    __shared__ __align__(16) double hs[2][kRefl][kEigMax];
    if (*info) return;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int c0 = blockIdx.x * kOrmWarps;
    const int k = top->k;
    // stage the U columns of this CTA's kept outputs
    for (int e = tid; e < kOrmWarps * k; e += kOrmWarps * 32) {
        const int q = e / k, j = e % k;
        const int c = c0 + q;
        const int a = c < n ? top->src[c] : k;
        us[q][j] = a < k ? Ut[size_t(j) * k + a] : 0.0;
    }
    __syncthreads();
    for (int r = tid; r < n; r += kOrmWarps * 32) {
        double acc[kOrmWarps];
#pragma unroll
        for (int q = 0; q < kOrmWarps; ++q) acc[q] = 0.0;
        for (int j = 0; j < k; ++j) {
            const double zv = Z[r + size_t(top->ck[j]) * n];
#pragma unroll
            for (int q = 0; q < kOrmWarps; ++q) acc[q] = fma(zv, us[q][j], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < kOrmWarps; ++q) {
            const int c = c0 + q;
            if (c >= n) break;
            const int a = top->src[c];
            zs[q][r] = a < k ? acc[q] : Z[r + size_t(top->cdf[a - k]) * n];
        }
    }
    __syncthreads();
    const int c = c0 + w;
    double* z = zs[w];
    // reflectors n-3 .. 0 in groups of kRefl, double buffered
    auto stage = [&](int g, int buf) {
        const int jhi = n - 3 - g * kRefl;
        for (int q = 0; q < kRefl; ++q) {
            const int j = jhi - q;
            if (j < 0) break;
            const int t = n - j - 1;
            for (int i = tid; i < t; i += kOrmWarps * 32) {
                const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&hs[buf][q][i]));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(Hv + size_t(j) * n + i));
            }
        }
        asm volatile("cp.async.commit_group;\n");
    };
    const int ngroups = n >= 3 ? (n - 3) / kRefl + 1 : 0;
    if (ngroups) stage(0, 0);
    for (int g = 0; g < ngroups; ++g) {
        const int buf = g & 1;
        if (g + 1 < ngroups) {
            stage(g + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n");
        } else {
            asm volatile("cp.async.wait_group 0;\n");
        }
        __syncthreads();
        if (c < n) {
            const int jhi = n - 3 - g * kRefl;
            for (int q = 0; q < kRefl; ++q) {
                const int j = jhi - q;
                if (j < 0) break;
                const double tj = tau[j];
                if (tj == 0.0) continue;
                const double* hv = hs[buf][q];
                const int t = n - j - 1;
                double dot = 0.0;
                for (int i = lane; i < t; i += 32) dot = fma(hv[i], z[j + 1 + i], dot);
                for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
                const double f = tj * dot;
                for (int i = lane; i < t; i += 32) z[j + 1 + i] = fma(-f, hv[i], z[j + 1 + i]);
                __syncwarp();
            }
        }
        __syncthreads();  // hs[buf] is restaged two groups later
    }
    if (c < n)
        for (int i = lane; i < n; i += 32) V[i + size_t(c) * n] = z[i];
}

size_t stedc_smem() { return ((sizeof(MergeWs) + 15) / 16) * 16 + kLeaves * sizeof(LeafWs); }

}  // namespace

// Eigenvalues ascending into d_D and eigenvectors over B (column-major), as
// syevd. Returns false (B untouched) when n is too large or a stage did not
// converge; the caller then uses cuSOLVER.
bool syev_small(Ctx& c, double* B, int64_t n64, double* d_D) {
    if (n64 < 1 || n64 > kEigMax || c.force_cusolver) return false;
    const int n = int(n64);
    cudaStream_t s = c.stream;
    smem_optin(k_sytrd, size_t(kSmemMax));
    smem_optin(k_sytrd_fused, size_t(kSmemMax));
    smem_optin(k_stedc, size_t(stedc_smem()));
    const size_t nn = size_t(n) * n;
    DBuf<double> ws(nn + 3 * size_t(n) + 3 * nn, s);
    double* H = ws.get();
    double* tau = H + nn;
    double* dg = tau + n;
    double* eo = dg + n;
    double* Z = eo + n;
    double* Tmp = Z + nn;
    double* Ut = Tmp + nn;
    // non-convergence of a stage: deferred (err_check -> cuSOLVER re-run);
    // the stages after a failed one return early
    int* info = err_flag(c);
    DBuf<unsigned char> topbuf(sizeof(TopPlan), s);
    TopPlan* top = reinterpret_cast<TopPlan*>(topbuf.get());
    static const bool timing = std::getenv("FRPCA_EIG_TIMING") != nullptr;
    DBuf<long long> clk(timing ? 160 : 0, s);
    if (timing) FB_CUDA(cudaMemsetAsync(clk.get(), 0, clk.bytes(), s));
    {
        Prof p1(c, "syev_sytrd", 0, 0);
        const char* eo_ = std::getenv("FRPCA_SYTRD_UNFUSED");  // tests compare both kernels
        if (sytrd_fused_fits(n) && !(eo_ && eo_[0] == '1'))
            k_sytrd_fused<<<1, kST, sytrd_fused_smem(n), s>>>(B, n, H, tau, dg, eo, clk.get());
        else
            k_sytrd<<<1, kST, sytrd_smem(n), s>>>(B, n, H, tau, dg, eo, clk.get());
        FB_LAUNCH_CHECK();
    }
    {
        Prof p2(c, "syev_stedc", 0, 0);
        static const double sec_tol = [] {
            const char* e = std::getenv("FRPCA_SEC_TOL");  // A/B and tests
            return e && *e ? std::atof(e) : 8.0;
        }();
        const double tol = sec_tol > 0 ? sec_tol : 8.0 * double(n);  // <= 0: the old 8 k factor
        FB_CUDA(cudaMemcpyToSymbolAsync(c_sec_tol, &tol, sizeof(double), 0, cudaMemcpyHostToDevice, s));
        k_stedc<<<1, kET, stedc_smem(), s>>>(n, dg, eo, Z, Tmp, Ut, d_D, top, info, clk.get());
        FB_LAUNCH_CHECK();
    }
    if (std::getenv("FRPCA_TEST_EIG_NOCONV")) {  // tests: the non-convergence -> cuSOLVER re-run path
        FB_CUDA(cudaMemcpyAsync(info, &kNoConvCode, sizeof(int), cudaMemcpyHostToDevice, s));
    }
    {
        Prof p3(c, "syev_ormtr", 0, 0);
        k_ormtr<<<(n + kOrmWarps - 1) / kOrmWarps, kOrmWarps * 32, 0, s>>>(H, tau, n, Z, Ut, top, B, info);
        FB_LAUNCH_CHECK();
    }
    if (timing) {
        FB_CUDA(cudaStreamSynchronize(s));
        long long h[160];
        FB_CUDA(cudaMemcpy(h, clk.get(), sizeof(h), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "sytrd step 20: A %lld B %lld C %lld D %lld\n", h[141] - h[140], h[142] - h[141],
                     h[143] - h[142], h[144] - h[143]);
        std::fprintf(stderr, "stedc n=%d leaves %lld", n, h[1] - h[0]);
        long long prev = h[1];
        for (int m = 0; m < 12 && h[2 + m]; ++m) {
            std::fprintf(stderr, " | L%d %lld", m, h[2 + m] - prev);
            prev = h[2 + m];
        }
        std::fprintf(stderr, "\n");
    }
    return true;
}

}  // namespace fb
