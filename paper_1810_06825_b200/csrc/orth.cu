// orth (dense_kernels.hpp:30-48): orthonormal basis of range(M) for a tall
// row-major panel W (r x l) by Householder QR, with the reference's rank check
// (|diag R| <= r eps max|diag R| is an error, :40-44) and
// Q = householderQ() * Identity(r, l) (:46). Used by the baseline algorithms
// basic_rpca / basic_rpcat.
//
// Same reflectors as Eigen::HouseholderQR (beta = -sign(c0) ||x||,
// tau = (beta - c0) / beta, v = [1; tail / (c0 - beta)]; a tail below
// DBL_MIN gives tau = 0), so Q agrees with the reference entry by entry, not
// only as a subspace.
//
// B200 design: ONE cooperative persistent kernel, one CTA per SM, every CTA
// owns a fixed block of rows for the whole run.
//  * Panels of 16 columns. A column step is ONE pass over the CTA's rows of
//    the panel (thread per row, 16 doubles in registers) and ONE grid
//    barrier: the pass applies the previous reflector and accumulates, for
//    the current column y, the sums y^T [y, later panel columns] on the
//    unscaled column; every CTA then forms beta, tau and the products
//    d_c = a_jc + s_c / (c0 - beta) from the per-CTA partials (fixed order).
//  * After a panel, the block reflector I - V T V^T (compact WY; T from
//    V^T V, the LAPACK dlarft recurrence) is applied to the trailing columns:
//    thread per column, V tiles broadcast from shared memory, per-CTA partials
//    of V^T [V, A2] summed in CTA order by a distributed reduction. Every sum
//    has a fixed order: the result is deterministic.
//  * Q is formed the same way in a second buffer, panels in reverse order
//    applied to Identity(r, l), rows above the panel skipped.
//  * The rank check runs on the device (deferred error, driver.cu err_check):
//    no host round trip.
#include <cooperative_groups.h>

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace fb {
namespace {

constexpr int QNB = 16;           // panel width
constexpr int kTQ = 512;          // threads per CTA
constexpr int QCW = 256;          // columns per thread-per-column chunk
constexpr int QTR = 64;           // rows per staged V tile

struct QrShared {
    double Vs[QTR][QNB];         // V tile (structure applied: 0 above, 1 on the diagonal)
    double red[kTQ / 32][QNB];   // per-warp partials of a column step
    double xr[QNB][QCW];         // row-group partials of the block-reflector stages
    double T[QNB][QNB];          // block reflector factor (upper triangular)
    double s[QNB], d[QNB], tau[QNB];
    double beta, tj, inv;
};

// V tile of rows [t0, t0 + nr) of panel (jb, bw) from the factored W
__device__ __forceinline__ void stage_v(QrShared& sh, const double* W, int l, int jb, int bw, int64_t t0, int nr) {
    for (int idx = threadIdx.x; idx < nr * QNB; idx += kTQ) {
        const int rr = idx / QNB, t = idx % QNB;
        const int64_t i = t0 + rr;
        double v = 0.0;
        if (t < bw) {
            const int dc = jb + t;
            v = i < dc ? 0.0 : (i == dc ? 1.0 : W[i * l + dc]);
        }
        sh.Vs[rr][t] = v;
    }
}

// X[rows >= jb, xc0 .. xc0 + ncols) -= V op(T) V^T X for panel (jb, bw) of the
// factored W. nv = bw in the factorisation (the panel's own columns come
// first as virtual columns, giving V^T V for T, which is built here and
// stored to Tp); nv = 0 when forming Q (T is read from Tp). trans: T^T
// (Q^T applied, factorisation) or T (Q applied).
__device__ void wy_stage(cg::grid_group& grid, QrShared& sh, const double* W, double* X, int64_t r0, int64_t r1, int l,
                         int jb, int bw, int nv, int xc0, int ncols, bool trans, double* wpart, double* wm, int ldw,
                         double* Tp, long long* clk) {
    const int tid = threadIdx.x;
    const bool tim = clk && blockIdx.x == 0 && tid == 0;
    long long c0 = tim ? clock64() : 0;
    const int G = gridDim.x, b = blockIdx.x;
    const int ne = nv + ncols;
    // thread <-> (column, row group): cw columns side by side (a power of two
    // covering ne, at most QCW), the other kTQ / cw threads of a column
    // split the rows of a tile
    int cw = 32;
    while (cw < ne && cw < QCW) cw <<= 1;
    const int ng = kTQ / cw, cl = tid % cw, g = tid / cw;
    const int64_t lo = r0 > jb ? r0 : int64_t(jb);
    // per-CTA partials of V^T [V, X]
    for (int e0 = 0; e0 < ne; e0 += cw) {
        const int e = e0 + cl;
        const bool on = e < ne, virt = e < nv;
        const int64_t xoff = virt ? 0 : int64_t(xc0) + (e - nv);
        double acc[QNB];
#pragma unroll
        for (int t = 0; t < QNB; ++t) acc[t] = 0.0;
        for (int64_t t0 = lo; t0 < r1; t0 += QTR) {
            const int nr = int(r1 - t0 < QTR ? r1 - t0 : QTR);
            __syncthreads();
            stage_v(sh, W, l, jb, bw, t0, nr);
            __syncthreads();
            if (on) {
                for (int rr0 = g; rr0 < nr; rr0 += 4 * ng) {  // four rows in flight
                    double val[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int rr = rr0 + k * ng;
                        val[k] = rr < nr ? (virt ? sh.Vs[rr][e] : X[(t0 + rr) * l + xoff]) : 0.0;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int rr = rr0 + k * ng;
                        if (rr < nr) {
#pragma unroll
                            for (int t = 0; t < QNB; ++t) acc[t] = fma(sh.Vs[rr][t], val[k], acc[t]);
                        }
                    }
                }
            }
        }
        // the row groups of a column: halving tree through shared memory
        for (int h = kTQ / 2; h >= cw; h >>= 1) {
            __syncthreads();
            if (tid >= h && tid < 2 * h) {
#pragma unroll
                for (int t = 0; t < QNB; ++t) sh.xr[t][tid - h] = acc[t];
            }
            __syncthreads();
            if (tid < h) {
#pragma unroll
                for (int t = 0; t < QNB; ++t) acc[t] += sh.xr[t][tid];
            }
        }
        if (tid < cw && on) {
#pragma unroll
            for (int t = 0; t < QNB; ++t) wpart[(int64_t(b) * QNB + t) * ldw + e] = acc[t];
        }
    }
    if (tim) { const long long c1 = clock64(); clk[2] += c1 - c0; c0 = c1; }
    grid.sync();
    // distributed reduction over the CTAs: a warp per entry, lanes over the
    // CTAs (strided, then the shuffle tree): a fixed order
    {
        const volatile double* wp = wpart;
        const int nw = G * (kTQ / 32);
        for (int idx = b * (kTQ / 32) + (tid >> 5); idx < QNB * ne; idx += nw) {
            const int t = idx / ne, e = idx % ne;
            double v = 0.0;
            for (int b0 = 0; b0 < G; b0 += 128) {
                double x[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int bb = b0 + 32 * k + (tid & 31);
                    x[k] = bb < G ? wp[(int64_t(bb) * QNB + t) * ldw + e] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) v += x[k];
            }
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((tid & 31) == 0) wm[t * ldw + e] = v;
        }
    }
    grid.sync();
    const volatile double* wv = wm;
    if (nv) {
        // T (dlarft, forward columnwise): T[t][t] = tau_t,
        // T[0:t, t] = -tau_t T[0:t, 0:t] (V^T V)[0:t, t]; row a of T only
        // needs its own earlier entries: a thread per row, V^T V from shared memory
        if (tid < QNB * QNB) {
            const int k = tid / QNB, t = tid % QNB;
            sh.xr[0][tid] = (k < bw && t < bw) ? wv[k * ldw + t] : 0.0;
        }
        __syncthreads();
        if (tid < QNB) {
            const int a = tid;
            for (int t = 0; t < QNB; ++t) {
                double v = 0.0;
                if (t < bw && a <= t) {
                    const double tt = sh.tau[t];
                    if (a == t) v = tt;
                    else {
                        for (int k = a; k < t; ++k) v += sh.T[a][k] * sh.xr[0][k * QNB + t];
                        v = -tt * v;
                    }
                }
                sh.T[a][t] = v;
            }
        }
        __syncthreads();
        if (b == 0 && tid < QNB * QNB) Tp[tid] = sh.T[tid / QNB][tid % QNB];
    } else {
        __syncthreads();
        if (tid < QNB * QNB) sh.T[tid / QNB][tid % QNB] = Tp[tid];
        __syncthreads();
    }
    if (tim) { const long long c1 = clock64(); clk[3] += c1 - c0; c0 = c1; }
    if (ncols <= 0) return;
    for (int e0 = (nv / cw) * cw; e0 < ne; e0 += cw) {
        const int e = e0 + cl;
        const bool on = e >= nv && e < ne;
        const int64_t xoff = int64_t(xc0) + (e - nv);
        double Z[QNB];
#pragma unroll
        for (int a = 0; a < QNB; ++a) Z[a] = 0.0;
        if (on) {
            double w[QNB];
#pragma unroll
            for (int k = 0; k < QNB; ++k) w[k] = k < bw ? wv[k * ldw + e] : 0.0;
#pragma unroll
            for (int a = 0; a < QNB; ++a) {
                double v = 0.0;
#pragma unroll
                for (int k = 0; k < QNB; ++k) {
                    if (trans ? k <= a : k >= a) v += (trans ? sh.T[k][a] : sh.T[a][k]) * w[k];
                }
                Z[a] = v;
            }
        }
        for (int64_t t0 = lo; t0 < r1; t0 += QTR) {
            const int nr = int(r1 - t0 < QTR ? r1 - t0 : QTR);
            __syncthreads();
            stage_v(sh, W, l, jb, bw, t0, nr);
            __syncthreads();
            if (on) {
                for (int rr0 = g; rr0 < nr; rr0 += 4 * ng) {  // four rows in flight
                    double xv[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int rr = rr0 + k * ng;
                        xv[k] = rr < nr ? X[(t0 + rr) * l + xoff] : 0.0;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int rr = rr0 + k * ng;
                        if (rr < nr) {
                            double v = 0.0;
#pragma unroll
                            for (int t = 0; t < QNB; ++t) v = fma(sh.Vs[rr][t], Z[t], v);
                            X[(t0 + rr) * l + xoff] = xv[k] - v;
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
    if (tim) clk[4] += clock64() - c0;
}

__global__ void __launch_bounds__(kTQ, 1)
k_hqr(double* W, double* Qb, int64_t r, int l, int64_t R, double* part, double* rowv, double* wpart, double* wm,
      int ldw, double* Tall, double* diag, int* err, long long* clk) {
    __shared__ QrShared sh;
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    const int64_t r0 = int64_t(b) * R, r1 = r0 + R < r ? r0 + R : r;

    // Identity(r, l) for the second phase, own rows
    for (int64_t idx = tid; idx < (r1 > r0 ? (r1 - r0) * l : 0); idx += kTQ) {
        const int64_t i = r0 + idx / l;
        Qb[i * l + idx % l] = (i == idx % l) ? 1.0 : 0.0;
    }

    int step = 0;
    const bool tim = clk && b == 0 && tid == 0;
    for (int jb = 0; jb < l; jb += QNB) {
        const int bw = l - jb < QNB ? l - jb : QNB;
        for (int jj = 0; jj <= bw; ++jj, ++step) {
            const int j = jb + jj;
            const bool havep = jj > 0, form = jj < bw;
            const int tp = jj - 1, jp = j - 1;
            const int buf = step & 1;
            // half a warp per row: lane hl holds column jb + hl of the row
            // (one coalesced 128-byte access per row), eight rows in flight
            const int hl = lane & 15, hw = lane >> 4;
            long long c0 = tim ? clock64() : 0;
            const double beta = sh.beta, inv = sh.inv;
            const double tdl = havep ? sh.tj * sh.d[hl] : 0.0;
            const int stp = havep ? tp : 0, sjj = form ? jj : 0;
            const bool incol = hl < bw;
            double acc = 0.0;
            const int64_t first = havep ? jp : j;
            const int64_t lo = r0 > first ? r0 : first;
            constexpr int RS = kTQ / 16;  // rows per CTA sweep
            for (int64_t wb = lo + 2 * warp; wb < r1; wb += 8 * RS) {  // warp-uniform
                double a[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int64_t i = wb + hw + k * RS;
                    a[k] = (i < r1 && incol) ? W[i * l + jb + hl] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int64_t i = wb + hw + k * RS;
                    const bool ok = i < r1;
                    double v = a[k];
                    const double ap = __shfl_sync(0xffffffffu, v, stp, 16);
                    if (havep) {
                        const double x = i == jp ? 1.0 : ap * inv;
                        if (hl == tp) v = i == jp ? beta : x;
                        else if (hl > tp) v -= tdl * x;
                        if (ok && incol && hl >= tp) W[i * l + jb + hl] = v;
                    }
                    const double y = __shfl_sync(0xffffffffu, v, sjj, 16);
                    if (form && ok) {
                        if (i == j) {
                            if (incol && hl >= jj) rowv[buf * QNB + hl] = v;
                        } else if (i > j && hl >= jj) {
                            acc = fma(y, v, acc);
                        }
                    }
                }
            }
            if (tim) { const long long c1 = clock64(); clk[0] += c1 - c0; c0 = c1; }
            if (!form) break;
            // CTA partial (the two half warps, then the warps in order)
            acc += __shfl_xor_sync(0xffffffffu, acc, 16);
            if (lane < QNB) sh.red[warp][lane] = acc;
            __syncthreads();
            if (tid < QNB) {
                double v = 0.0;
                for (int w = 0; w < kTQ / 32; ++w) v += sh.red[w][tid];
                part[(int64_t(buf) * G + b) * QNB + tid] = v;
            }
            grid.sync();
            {
                const volatile double* pp = part;
                if (warp < QNB) {
                    double v = 0.0;
                    for (int b0 = 0; b0 < G; b0 += 256) {
                        double x[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int bb = b0 + 32 * k + lane;
                            x[k] = bb < G ? pp[(int64_t(buf) * G + bb) * QNB + warp] : 0.0;
                        }
#pragma unroll
                        for (int k = 0; k < 8; ++k) v += x[k];
                    }
                    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if (lane == 0) sh.s[warp] = v;
                }
            }
            __syncthreads();
            if (warp == 0) {
                // Eigen makeHouseholderInPlace on (c0, tail); lane t holds column t's row value and sum
                const volatile double* rv = rowv + buf * QNB;
                const bool in_panel = lane >= jj && lane < bw;
                const double rvt = in_panel ? rv[lane] : 0.0;
                const double st = lane < QNB ? sh.s[lane] : 0.0;
                const double c0 = __shfl_sync(0xffffffffu, rvt, jj), tail = __shfl_sync(0xffffffffu, st, jj);
                double be, tj, in;
                if (tail <= DBL_MIN) {
                    tj = 0.0;
                    be = c0;
                    in = 0.0;
                } else {
                    be = sqrt(c0 * c0 + tail);
                    if (c0 >= 0.0) be = -be;
                    in = 1.0 / (c0 - be);
                    tj = (be - c0) / be;
                }
                if (lane < QNB) sh.d[lane] = (lane > jj && lane < bw) ? rvt + in * st : 0.0;
                if (lane == 0) {
                    sh.beta = be;
                    sh.tj = tj;
                    sh.inv = in;
                    sh.tau[jj] = tj;
                    if (b == 0) diag[j] = be;
                }
            }
            __syncthreads();
            if (tim) clk[1] += clock64() - c0;
        }
        __syncthreads();
        wy_stage(grid, sh, W, W, r0, r1, l, jb, bw, bw, jb + bw, l - jb - bw, true, wpart, wm, ldw,
                 Tall + int64_t(jb / QNB) * QNB * QNB, clk);
    }
    if (tim) {
        clk[5] = clk[2], clk[6] = clk[3], clk[7] = clk[4];  // factorisation's share of the block-reflector stages
    }
    // rank check on diag R (:40-44)
    if (b == 0 && tid == 0) {
        double maxd = 0.0;
        for (int j = 0; j < l; ++j) maxd = fmax(maxd, fabs(diag[j]));
        const double tol = double(r) * DBL_EPSILON * maxd;
        bool bad = maxd == 0.0;
        for (int j = 0; j < l; ++j) bad = bad || fabs(diag[j]) <= tol;
        if (bad) atomicCAS(err, 0, kErrOrthRank);
    }
    grid.sync();  // Tall written by CTA 0
    // Q = H_0 .. H_{l-1} Identity(r, l): block reflectors in reverse order
    for (int jb = ((l - 1) / QNB) * QNB; jb >= 0; jb -= QNB) {
        const int bw = l - jb < QNB ? l - jb : QNB;
        wy_stage(grid, sh, W, Qb, r0, r1, l, jb, bw, 0, jb, l - jb, false, wpart, wm, ldw,
                 Tall + int64_t(jb / QNB) * QNB * QNB, clk);
    }
}

}  // namespace

void orth_device(Ctx& c, double* W, int64_t r, int64_t l) {
    require(r >= l && l >= 1, "orth: input must be tall (rows >= cols >= 1)");
    require(l < (int64_t(1) << 24), "orth: cols must be < 2^24");
    Prof prof(c, "orth", 32.0 * r * l, 4.0 * double(r) * l * l);
    cudaStream_t s = c.stream;
    int per_sm = 0;
    FB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hqr, kTQ, 0));
    require(per_sm >= 1, "orth: kernel does not fit an SM");
    // at least 64 rows per CTA; one CTA per SM
    const int G = int(std::max<int64_t>(1, std::min<int64_t>(c.num_sms, (r + 63) / 64)));
    int64_t R = (r + G - 1) / G;
    int L = int(l), ldw = int(l) + QNB;
    const int npan = int((l + QNB - 1) / QNB);
    DBuf<double> Qb(size_t(r * l), s), part(size_t(2) * G * QNB, s), rowv(2 * QNB, s),
        wpart(size_t(G) * QNB * ldw, s), wm(size_t(QNB) * ldw, s), Tall(size_t(npan) * QNB * QNB, s),
        diag(size_t(l), s);
    double *Qp = Qb.get(), *pp = part.get(), *rp = rowv.get(), *wpp = wpart.get(), *wmp = wm.get(),
           *Tp = Tall.get(), *dp = diag.get();
    int* errp = err_flag(c);  // rank deficiency: deferred NumericalError (err_check)
    static const bool timing = std::getenv("FRPCA_ORTH_TIMING") != nullptr;
    DBuf<long long> clk(timing ? 8 : 0, s);
    if (timing) FB_CUDA(cudaMemsetAsync(clk.get(), 0, clk.bytes(), s));
    long long* clkp = clk.get();
    void* args[] = {&W, &Qp, &r, &L, &R, &pp, &rp, &wpp, &wmp, &ldw, &Tp, &dp, &errp, &clkp};
    FB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_hqr), dim3(G), dim3(kTQ), args, 0, s));
    count_launch();
    FB_CUDA(cudaMemcpyAsync(W, Qp, sizeof(double) * size_t(r * l), cudaMemcpyDeviceToDevice, s));
    if (timing) {
        FB_CUDA(cudaStreamSynchronize(s));
        long long h[8];
        FB_CUDA(cudaMemcpy(h, clk.get(), sizeof(h), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "orth %lld x %lld (CTA 0, cycles): column passes %lld, reduce+barrier %lld | block reflectors, "
                     "factorisation: partials %lld reduce+T %lld update %lld | forming Q: %lld %lld %lld\n",
                     (long long)r, (long long)l, h[0], h[1], h[5], h[6], h[7], h[2] - h[5], h[3] - h[6], h[4] - h[7]);
    }
}

}  // namespace fb
