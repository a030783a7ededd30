// K7: lu_basis (dense_kernels.hpp:50-116) on a tall row-major panel W (m x l).
//
// Same algorithm as the reference: blocked right-looking LU, nb = 32, first-max
// partial pivoting (largest |value|, ties to the smallest current position,
// :72-80), tol = l * eps * max|M| (:64-65, :81), TRSM for U12 (:98-100),
// trailing update (:101-104), P^T L assembly (:108-115).
//
// B200 design: ONE cooperative persistent kernel for the whole factorisation.
//  * Rows never move. Each thread owns a fixed set of rows for the whole run
//    and keeps their current positions (pos[]); a row interchange at step j
//    is resolved locally: the pivot row takes position j and the row that
//    held position j takes the pivot's old position, which travels with the
//    pivot candidate. No bookkeeping kernel, no race.
//  * The active 32-column panel lives in a column-major copy P (coalesced
//    thread-per-row access; L2-resident at the configs' heights).
//  * Column step = one grid barrier: every CTA reduces all per-CTA candidates
//    (deterministic: max |v|, ties to the lowest position), reads the pivot
//    row from P, updates its rows and publishes its best candidate for the
//    next column.
//  * After a panel, every CTA solves U12 = L11^{-1} A12 redundantly in shared
//    memory (U12 is never part of the output P^T L, so it is not stored), then
//    updates its own rows' trailing columns, stages the next panel into P and
//    publishes candidates for its first column.
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace fb {
namespace {

constexpr int NB = 32;

struct Cand {
    double v;
    int32_t pos, row;
};

__device__ __forceinline__ bool better(double v, int32_t p, double bv, int32_t bp) {
    return v > bv || (v == bv && p < bp);
}

__device__ __forceinline__ void cand_merge(Cand& c, const Cand& o) {
    if (better(o.v, o.pos, c.v, c.pos)) c = o;
}

// Warp-wide best candidate (cand_merge's total order), returned to every lane.
__device__ __forceinline__ Cand warp_best(Cand c) {
    for (int o = 16; o; o >>= 1) {
        Cand x;
        x.v = __shfl_xor_sync(0xffffffffu, c.v, o);
        x.pos = __shfl_xor_sync(0xffffffffu, c.pos, o);
        x.row = __shfl_xor_sync(0xffffffffu, c.row, o);
        cand_merge(c, x);
    }
    return c;
}

// block-wide reduction; the result is returned to every thread
template <int kT>
__device__ Cand block_best(Cand c, Cand* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    c = warp_best(c);
    if (lane == 0) sh[warp] = c;
    __syncthreads();
    Cand r = sh[0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w) cand_merge(r, sh[w]);
    __syncthreads();
    return r;
}

template <int kT, int NBK>
__global__ void __launch_bounds__(kT, 1)
k_lu(double* __restrict__ W, int64_t m, int l, const unsigned long long* __restrict__ dmax, double* __restrict__ P,
     int32_t* __restrict__ pos, Cand* __restrict__ cand, int* __restrict__ err, long long* __restrict__ clk) {
    const double tol = double(l) * DBL_EPSILON * __longlong_as_double((long long)*dmax);  // :64-65
    extern __shared__ double smem[];
    double* U12 = smem;                     // NBK x l (trailing part used)
    double* L11 = U12 + NBK * l;             // NBK x NBK
    double* u = L11 + NBK * (NBK + 1);        // NBK
    __shared__ Cand shc[kT / 32];
    __shared__ int32_t prow[NBK];
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = int64_t(blockIdx.x) * kT + threadIdx.x;
    const int64_t nthr = int64_t(gridDim.x) * kT;
    const int nblk = gridDim.x;

    // prologue: positions, panel 0, candidates of column 0
    {
        const int bw = min(NBK, l);
        Cand c{-1.0, INT32_MAX, -1};
        for (int64_t i = gtid; i < m; i += nthr) {
            pos[i] = int32_t(i);
            const double* wr = W + i * l;
            for (int t = 0; t < bw; ++t) P[int64_t(t) * m + i] = wr[t];
            cand_merge(c, Cand{fabs(wr[0]), int32_t(i), int32_t(i)});
        }
        c = block_best<kT>(c, shc);
        if (threadIdx.x == 0) cand[blockIdx.x] = c;
    }

    for (int jb = 0; jb < l; jb += NBK) {
        const int bw = min(NBK, l - jb);
        for (int jj = 0; jj < bw; ++jj) {
            const int j = jb + jj;
            const bool tim = clk && j == 100 && blockIdx.x == 0 && threadIdx.x == 0;
            if (tim) clk[0] = clock64();
            grid.sync();
            if (tim) clk[1] = clock64();
            // every CTA reduces the candidates identically
            Cand c{-1.0, INT32_MAX, -1};
            for (int k = threadIdx.x; k < nblk; k += kT) cand_merge(c, cand[k]);
            const Cand best = block_best<kT>(c, shc);
            if (tim) clk[2] = clock64();
            if (best.v <= tol || best.row < 0) {  // zero pivot (:81); NaN passes, as there
                if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(err, 0, kErrLuPivot);
                return;  // uniform across the grid
            }
            const int32_t pr = best.row, pb = best.pos;
            if (threadIdx.x < bw) u[threadIdx.x] = P[int64_t(threadIdx.x) * m + pr];
            if (threadIdx.x == 0) prow[jj] = pr;
            __syncthreads();
            if (tim) clk[3] = clock64();
            const double d = u[jj];
            Cand nc{-1.0, INT32_MAX, -1};
            for (int64_t i = gtid; i < m; i += nthr) {
                // all loads of the row first (position + remaining panel
                // entries are independent), so a row costs one round trip
                int32_t p = pos[i];
                double v[NBK];
#pragma unroll
                for (int t = 0; t < NBK; ++t)
                    if (t >= jj && t < bw) v[t] = P[int64_t(t) * m + i];
                if (i == pr) {
                    pos[i] = j;
                    continue;
                }
                if (p == j) {  // displaced by the interchange (:82-85)
                    p = pb;
                    pos[i] = p;
                }
                if (p > j) {
                    double mi = 0.0, nv = 0.0;
#pragma unroll
                    for (int t = 0; t < NBK; ++t)
                        if (t == jj) {
                            mi = v[t] / d;                             // :88
                            P[int64_t(t) * m + i] = mi;
                        }
#pragma unroll
                    for (int t = 0; t < NBK; ++t)                      // :89-92
                        if (t > jj && t < bw) {
                            v[t] = v[t] - mi * u[t];
                            P[int64_t(t) * m + i] = v[t];
                            if (t == jj + 1) nv = v[t];
                        }
                    if (jj + 1 < bw) cand_merge(nc, Cand{fabs(nv), p, int32_t(i)});
                }
            }
            if (tim) clk[4] = clock64();
            if (jj + 1 < bw) {
                nc = block_best<kT>(nc, shc);
                if (threadIdx.x == 0) cand[blockIdx.x] = nc;
            }
            if (tim) clk[5] = clock64();
        }
        const int c0 = jb + bw, tcols = l - c0;
        grid.sync();  // the last column's update of every pivot row is visible
        if (tcols > 0) {
            // L11 (unit lower) of the bw pivot rows and A12 = their trailing columns
            for (int e = threadIdx.x; e < bw * bw; e += kT) {
                const int t = e / bw, s = e % bw;
                L11[t * (NBK + 1) + s] = P[int64_t(s) * m + prow[t]];
            }
            for (int e = threadIdx.x; e < bw * tcols; e += kT) {
                const int t = e / tcols, cc = e % tcols;
                U12[t * tcols + cc] = W[int64_t(prow[t]) * l + c0 + cc];
            }
            __syncthreads();
            // U12 = L11^{-1} A12 (forward substitution, one column per thread)
            for (int cc = threadIdx.x; cc < tcols; cc += kT)
                for (int t = 1; t < bw; ++t) {
                    double acc = U12[t * tcols + cc];
                    for (int s = 0; s < t; ++s) acc -= L11[t * (NBK + 1) + s] * U12[s * tcols + cc];
                    U12[t * tcols + cc] = acc;
                }
            __syncthreads();
        }
        // own rows: write the finished panel back to W, trailing update
        // A22 -= L21 U12 (:101-104), stage the next panel, candidates.
        const int nbw = min(NBK, tcols);
        Cand nc{-1.0, INT32_MAX, -1};
        for (int64_t i = gtid; i < m; i += nthr) {
            const int32_t p = pos[i];
            if (p < jb) continue;  // pivot of an earlier panel: finished
            double* wr = W + i * l;
            double Lr[NBK];
#pragma unroll
            for (int t = 0; t < NBK; ++t) {
                if (t < bw) {
                    Lr[t] = P[int64_t(t) * m + i];
                    wr[jb + t] = Lr[t];
                }
            }
            // rows pivoted in this panel keep their P entries (other CTAs read
            // L11 from them) and their trailing columns (A12 of the TRSM)
            if (tcols > 0 && p >= c0) {
                // 8 trailing columns at a time: independent loads, then FMAs
                for (int cb = 0; cb < tcols; cb += 8) {
                    double a[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (cb + e < tcols) a[e] = wr[c0 + cb + e];
#pragma unroll
                    for (int t = 0; t < NBK; ++t)
                        if (t < bw) {
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                if (cb + e < tcols) a[e] -= Lr[t] * U12[t * tcols + cb + e];
                        }
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (cb + e < tcols) {
                            wr[c0 + cb + e] = a[e];
                            if (cb + e < nbw) P[int64_t(cb + e) * m + i] = a[e];
                        }
                }
                cand_merge(nc, Cand{fabs(wr[c0]), p, int32_t(i)});
            }
        }
        if (tcols > 0) {
            nc = block_best<kT>(nc, shc);
            if (threadIdx.x == 0) cand[blockIdx.x] = nc;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Shared-memory-resident variant (m <= ~119k at l = 200, e.g. C1's n x l
// panel): CTA b owns the contiguous rows [b R, (b+1) R) and keeps their 32
// panel columns in shared memory, so a column step touches no global memory
// but the candidates. Each CTA publishes its best candidate together with
// that row's remaining panel values, so after the grid barrier the pivot row
// is one load away. Trailing columns are solved/updated in chunks of UCH
// (last chunk first, so the chunk holding the next panel is done last and
// can overwrite the panel). Same arithmetic, in the same order, as k_lu.
constexpr int UCH = 64;

template <int kT, int NBK>
__global__ void __launch_bounds__(kT, 1)
k_lu_smem(double* __restrict__ W, int64_t m, int l, const unsigned long long* __restrict__ dmax, int R,
          int32_t* __restrict__ pos_g,
          Cand* __restrict__ cand, double* __restrict__ cvals, int* __restrict__ err, long long* __restrict__ clk,
          int novec) {
    const double tol = double(l) * DBL_EPSILON * __longlong_as_double((long long)*dmax);  // :64-65
    extern __shared__ double smem[];
    double* Ps = smem;                      // NBK x R (column t at Ps + t R)
    double* U12 = Ps + size_t(NBK) * R;      // NBK x UCH
    double* L11 = U12 + NBK * UCH;           // NBK x (NBK + 1)
    double* u = L11 + NBK * (NBK + 1);        // NBK
    int32_t* posS = reinterpret_cast<int32_t*>(u + NBK);  // R
    __shared__ Cand shc[kT / 32];
    __shared__ int32_t prow[NBK];
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x;
    const int64_t r0 = int64_t(blockIdx.x) * R;
    const int64_t rem = m - r0;
    const int nr = rem <= 0 ? 0 : (rem < R ? int(rem) : R);

    auto publish = [&](Cand c, int width) {  // after a block_best (Ps final)
        if (tid == 0) cand[blockIdx.x] = c;
        if (tid < width) cvals[size_t(blockIdx.x) * NBK + tid] = c.row >= 0 ? Ps[size_t(tid) * R + (c.row - r0)] : 0.0;
    };
    {
        const int bw = min(NBK, l);
        Cand c{-1.0, INT32_MAX, -1};
        for (int r = tid; r < nr; r += kT) {
            const int64_t i = r0 + r;
            posS[r] = int32_t(i);
            const double* wr = W + i * l;
            for (int t = 0; t < bw; ++t) Ps[size_t(t) * R + r] = wr[t];
            cand_merge(c, Cand{fabs(wr[0]), int32_t(i), int32_t(i)});
        }
        c = block_best<kT>(c, shc);
        publish(c, bw);
    }
    for (int jb = 0; jb < l; jb += NBK) {
        const int bw = min(NBK, l - jb);
        for (int jj = 0; jj < bw; ++jj) {
            const int j = jb + jj;
            const bool tim = clk && j == 100 && blockIdx.x == 0 && tid == 0;
            if (tim) clk[0] = clock64();
            grid.sync();
            if (tim) clk[1] = clock64();
            // every warp reduces all CTAs' candidates itself (a total order:
            // the same winner everywhere, no block barrier)
            // (all loads in flight before the merges: the merge order does not
            // matter, the order is total)
            Cand best{-1.0, INT32_MAX, -1};
            {
                constexpr int kPer = 8;
                const int lane = tid & 31, G = int(gridDim.x);
                Cand cs[kPer];
#pragma unroll
                for (int q = 0; q < kPer; ++q) {
                    const int k = lane + 32 * q;
                    cs[q] = k < G ? cand[k] : Cand{-1.0, INT32_MAX, -1};
                }
#pragma unroll
                for (int q = 0; q < kPer; ++q) cand_merge(best, cs[q]);
                for (int k = lane + 32 * kPer; k < G; k += 32) cand_merge(best, cand[k]);
            }
            best = warp_best(best);
            if (best.v <= tol || best.row < 0) {  // zero pivot (:81); NaN passes, as there
                if (blockIdx.x == 0 && tid == 0) atomicCAS(err, 0, kErrLuPivot);
                return;  // uniform across the grid
            }
            if (tim) clk[2] = clock64();
            const int32_t pr = best.row, pb = best.pos;
            if (tid < bw) u[tid] = cvals[size_t(pr / R) * NBK + tid];
            if (tid == 0) prow[jj] = pr;
            __syncthreads();
            if (tim) clk[3] = clock64();
            const double d = u[jj];
            Cand nc{-1.0, INT32_MAX, -1};
            for (int r = tid; r < nr; r += kT) {
                const int64_t i = r0 + r;
                int32_t p = posS[r];
                if (i == pr) {
                    posS[r] = j;
                    continue;
                }
                if (p == j) {  // displaced by the interchange (:82-85)
                    p = pb;
                    posS[r] = p;
                }
                if (p > j) {
                    double* pc = Ps + r;
                    const double mi = pc[size_t(jj) * R] / d;  // :88
                    pc[size_t(jj) * R] = mi;
                    double nv = 0.0;
                    if (jj + 1 < bw) {
                        nv = pc[size_t(jj + 1) * R] - mi * u[jj + 1];
                        pc[size_t(jj + 1) * R] = nv;
                    }
#pragma unroll 4
                    for (int t = jj + 2; t < bw; ++t)  // :89-92
                        pc[size_t(t) * R] = pc[size_t(t) * R] - mi * u[t];
                    if (jj + 1 < bw) cand_merge(nc, Cand{fabs(nv), p, int32_t(i)});
                }
            }
            if (tim) clk[4] = clock64();
            if (jj + 1 < bw) {
                nc = block_best<kT>(nc, shc);
                publish(nc, bw);
            }
            if (tim) clk[5] = clock64();
        }
        if (clk && blockIdx.x == 0 && tid == 0 && jb == 64) clk[6] = clock64();
        // finished panel of the own rows back to W (L of P^T L; L11 / A12 source);
        // a different thread <-> row map than the column steps: barrier first
        __syncthreads();
        for (int e = tid; e < nr * bw; e += kT) {
            const int r = e % nr, t = e / nr;
            if (posS[r] >= jb) W[(r0 + r) * l + jb + t] = Ps[size_t(t) * R + r];
        }
        const bool ptim = clk && blockIdx.x == 0 && tid == 0 && jb == 64;
        if (ptim) clk[8] = clock64();
        const int c0 = jb + bw, tcols = l - c0;
        grid.sync();
        if (ptim) clk[9] = clock64();
        if (tcols <= 0) break;
        for (int e = tid; e < bw * bw; e += kT) {
            const int t = e / bw, s2 = e % bw;
            L11[t * (NBK + 1) + s2] = W[int64_t(prow[t]) * l + jb + s2];
        }
        const int nbw = min(NBK, tcols);
        const int nch = (tcols + UCH - 1) / UCH;
        // nbw is a multiple of 8 whenever the vector path writes Ps (cc0 + cb < nbw)
        const bool vec = !novec && bw == NBK && (l % 2) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0 &&
                         (nbw % 8) == 0;
        Cand nc{-1.0, INT32_MAX, -1};
        for (int ch = nch - 1; ch >= 0; --ch) {
            const int cc0 = ch * UCH, cw = min(UCH, tcols - cc0);
            __syncthreads();  // L11 staged / previous chunk's U12 consumed
            for (int e = tid; e < bw * cw; e += kT) {
                const int t = e / cw, cc = e % cw;
                U12[t * UCH + cc] = W[int64_t(prow[t]) * l + c0 + cc0 + cc];
            }
            __syncthreads();
            if (ptim && ch < 2) clk[10 + 3 * ch] = clock64();
            for (int cc = tid; cc < cw; cc += kT)  // U12 = L11^{-1} A12, column by column
                for (int t = 1; t < bw; ++t) {
                    double acc = U12[t * UCH + cc];
                    for (int s2 = 0; s2 < t; ++s2) acc -= L11[t * (NBK + 1) + s2] * U12[s2 * UCH + cc];
                    U12[t * UCH + cc] = acc;
                }
            __syncthreads();
            if (ptim && ch < 2) clk[11 + 3 * ch] = clock64();
            for (int r = tid; r < nr; r += kT) {
                const int32_t p = posS[r];
                if (p < c0) continue;  // pivot of this or an earlier panel
                double* wr = W + (r0 + r) * l;
                double Lr[NBK];
#pragma unroll
                for (int t = 0; t < NBK; ++t)
                    if (t < bw) Lr[t] = Ps[size_t(t) * R + r];
                for (int cb = 0; cb < cw; cb += 8) {
                    if (vec && cb + 8 <= cw) {
                        // full panel, full 8-column block: no guards, W and
                        // U12 as double2 (same FMA order as below)
                        double2* w2 = reinterpret_cast<double2*>(wr + c0 + cc0 + cb);
                        double2 a2[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) a2[e] = w2[e];
#pragma unroll
                        for (int t = 0; t < NBK; ++t) {
                            const double2* u2 = reinterpret_cast<const double2*>(U12 + t * UCH + cb);
                            const double lt = -Lr[t];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const double2 uu = u2[e];
                                a2[e].x = fma(lt, uu.x, a2[e].x);
                                a2[e].y = fma(lt, uu.y, a2[e].y);
                            }
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) w2[e] = a2[e];
                        if (cc0 + cb < nbw)
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                Ps[size_t(cc0 + cb + 2 * e) * R + r] = a2[e].x;
                                Ps[size_t(cc0 + cb + 2 * e + 1) * R + r] = a2[e].y;
                            }
                        continue;
                    }
                    double a[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (cb + e < cw) a[e] = wr[c0 + cc0 + cb + e];
#pragma unroll
                    for (int t = 0; t < NBK; ++t)
                        if (t < bw) {
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                if (cb + e < cw) a[e] -= Lr[t] * U12[t * UCH + cb + e];
                        }
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (cb + e < cw) {
                            wr[c0 + cc0 + cb + e] = a[e];
                            if (cc0 + cb + e < nbw) Ps[size_t(cc0 + cb + e) * R + r] = a[e];
                        }
                }
                if (ch == 0) cand_merge(nc, Cand{fabs(Ps[r]), p, int32_t(r0 + r)});
            }
            if (ptim && ch < 2) clk[12 + 3 * ch] = clock64();
        }
        nc = block_best<kT>(nc, shc);
        publish(nc, nbw);
        if (clk && blockIdx.x == 0 && tid == 0 && jb == 64) clk[7] = clock64();
    }
    for (int r = tid; r < nr; r += kT) pos_g[r0 + r] = posS[r];
}

__global__ void k_assemble(double* __restrict__ W, int64_t m, int l, const int32_t* __restrict__ pos) {
    // (:108-115) X[r][j] = (j == pos) ? 1 : (j < pos ? W[r][j] : 0)
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * l;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / l;
        const int j = int(e - r * l);
        const int32_t p = pos[r];
        if (j == p) W[e] = 1.0;
        else if (j > p) W[e] = 0.0;
    }
}

}  // namespace

void lu_basis_device(Ctx& c, double* W, int64_t m, int64_t l) {
    require(m >= l && l >= 1, "lu_basis: input must be tall (rows >= cols >= 1)");
    require(m < (int64_t(1) << 31), "lu_basis: rows must be < 2^31");
    Prof prof(c, "lu_basis", 16.0 * m * l, double(m) * l * l - double(l) * l * l / 3.0);
    cudaStream_t s = c.stream;
    // tol = l eps max|M| (:64-65) is formed in the kernels from the device max
    DBuf<unsigned long long> dmax(1, s);
    maxabs_device_async(c, W, m * l, dmax.get());
    const unsigned long long* dmaxp = dmax.get();
    DBuf<int32_t> pos(size_t(m), s);
    int L = int(l);
    int32_t* posp = pos.get();
    int* errp = err_flag(c);  // zero pivot: deferred NumericalError (err_check)
    // shared-memory-resident panel when the rows fit one CTA per SM, 16
    // columns wide (rows up to ~214k: C1 and C4; C1 1.98 -> 1.94 ms at 16 vs
    // 32, C4 6.2 -> 3.4 ms against the global kernel); the width does not
    // change the arithmetic (see the global kernel below)
    constexpr int kTS = 512;
    const int R = int((m + c.num_sms - 1) / c.num_sms);
    auto smem_for = [&](int nb) {
        return sizeof(double) * (size_t(nb) * R + nb * UCH + nb * (nb + 1) + nb) + sizeof(int32_t) * R;
    };
    const char* esb = std::getenv("FRPCA_LU_SMEM_NB");
    const int snb = esb ? std::atoi(esb) : 16;
    const size_t smem_s = smem_for(snb);
    void* kfs = snb == 16 ? reinterpret_cast<void*>(k_lu_smem<kTS, 16>) : reinterpret_cast<void*>(k_lu_smem<kTS, 32>);
    const bool no_smem = std::getenv("FRPCA_LU_GLOBAL") != nullptr;  // tests compare both kernels
    if (!no_smem && (snb == 16 || snb == 32) && smem_s <= 220 * 1024) {
        FB_CUDA(cudaFuncSetAttribute(kfs, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_s)));
        int per_sm = 0;
        FB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfs, kTS, smem_s));
        if (per_sm >= 1) {
            const int grid = int((m + R - 1) / R);
            DBuf<Cand> cand(size_t(grid), s);
            DBuf<double> cvals(size_t(grid) * snb, s);
            Cand* candp = cand.get();
            double* cvp = cvals.get();
            const bool timing = std::getenv("FRPCA_LU_TIMING") != nullptr;
            DBuf<long long> clk(timing ? 24 : 0, s);
            if (timing) FB_CUDA(cudaMemsetAsync(clk.get(), 0, clk.bytes(), s));
            long long* clkp = clk.get();
            int novec = std::getenv("FRPCA_LU_NOVEC") != nullptr;
            void* args[] = {&W, &m, &L, const_cast<unsigned long long**>(&dmaxp), const_cast<int*>(&R), &posp, &candp,
                            &cvp, &errp,
                            &clkp, &novec};
            FB_CUDA(cudaLaunchCooperativeKernel(kfs, dim3(grid), dim3(kTS), args,
                                                smem_s, s));
            count_launch();
            if (timing) {
                FB_CUDA(cudaStreamSynchronize(s));
                long long h[24];
                FB_CUDA(cudaMemcpy(h, clk.get(), sizeof(h), cudaMemcpyDeviceToHost));
                std::fprintf(stderr, "lu_smem step 100 (cycles): sync %lld cand %lld u %lld rows %lld best %lld | panel end %lld\n",
                             h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4], h[7] - h[6]);
                std::fprintf(stderr, "  panel 64: writeback %lld gridsync %lld | chunk1 stage %lld trsm %lld update %lld |"
                             " chunk0 stage %lld trsm %lld update %lld | best %lld\n",
                             h[8] - h[6], h[9] - h[8], h[13] - h[9], h[14] - h[13], h[15] - h[14], h[10] - h[15],
                             h[11] - h[10], h[12] - h[11], h[7] - h[12]);
            }
            const int agrid = int(std::max<int64_t>(1, std::min<int64_t>(c.num_sms * 16, (m * l + 255) / 256)));
            k_assemble<<<agrid, 256, 0, s>>>(W, m, L, pos.get());
            FB_LAUNCH_CHECK();
            return;
        }
    }
    // Panel width of the global-panel kernel: the column-major panel copy P is
    // re-read and rewritten every column step; at 16 columns it is half the
    // traffic and stays L2-resident (C2 LU 9.1 -> 7.45 ms, C4 6.4 -> 6.2 ms). The width does not change the
    // arithmetic: every element receives the same FMAs in the same order
    // (in-panel rank-1 updates == TRSM + trailing update, both in pivot
    // order), checked bitwise against the shared-memory kernel (NB = 32).
    const char* enb = std::getenv("FRPCA_LU_NB");
    const int nbk = enb ? std::atoi(enb) : 16;
    require(nbk == 8 || nbk == 16 || nbk == 32, "FRPCA_LU_NB must be 8, 16 or 32");
    const size_t smem = sizeof(double) * (size_t(nbk) * size_t(l) + nbk * (nbk + 1) + nbk);
    static const int kT = [] {
        const char* e = std::getenv("FRPCA_LU_THREADS");
        return e && std::atoi(e) == 512 ? 512 : 256;
    }();
    void* kfn = nbk == 8 ? (kT == 256 ? reinterpret_cast<void*>(k_lu<256, 8>) : reinterpret_cast<void*>(k_lu<512, 8>))
              : nbk == 16 ? (kT == 256 ? reinterpret_cast<void*>(k_lu<256, 16>) : reinterpret_cast<void*>(k_lu<512, 16>))
                          : (kT == 256 ? reinterpret_cast<void*>(k_lu<256, 32>) : reinterpret_cast<void*>(k_lu<512, 32>));
    FB_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(std::max<size_t>(smem, 48 * 1024))));
    int per_sm = 0;
    FB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kT, smem));
    require(per_sm >= 1, "lu_basis: panel width too large for one CTA's shared memory");
    int grid = std::max(1, std::min<int>(per_sm * c.num_sms, int((m + kT - 1) / kT)));
    DBuf<Cand> cand(size_t(grid), s);
    DBuf<double> P(size_t(m) * nbk, s);
    double* Pp = P.get();
    Cand* candp = cand.get();
    static const bool timing = std::getenv("FRPCA_LU_TIMING") != nullptr;
    DBuf<long long> clk(timing ? 8 : 0, s);
    long long* clkp = clk.get();
    void* args[] = {&W, &m, &L, const_cast<unsigned long long**>(&dmaxp), &Pp, &posp, &candp, &errp, &clkp};
    FB_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kT), args, smem, s));
    count_launch();
    if (timing) {
        FB_CUDA(cudaStreamSynchronize(s));
        long long h[8];
        FB_CUDA(cudaMemcpy(h, clk.get(), sizeof(long long) * 6, cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "lu step 100 (cycles): sync %lld cand %lld u %lld rows %lld best %lld\n", h[1] - h[0],
                     h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4]);
    }
    const int agrid = int(std::max<int64_t>(1, std::min<int64_t>(c.num_sms * 16, (m * l + 255) / 256)));
    k_assemble<<<agrid, 256, 0, s>>>(W, m, L, pos.get());
    FB_LAUNCH_CHECK();
}

}  // namespace fb
