// K7: lu_basis (dense_kernels.hpp:50-116) on a tall row-major panel W (m x l).
//
// Same algorithm as the reference: blocked right-looking LU, nb = 32, first-max
// partial pivoting (largest |value|, ties to the smallest current position,
// :72-80), tol = l * eps * max|M| (:64-65, :81), TRSM for U12 (:98-100),
// trailing update (:101-104), P^T L assembly (:108-115).
//
// B200 layout: rows never move. A position array pos[] (and its inverse perm[])
// records the interchanges, so a "row swap" is two integer writes instead of
// two l*8-byte row copies. Each 32-column panel is factored out of a
// column-major copy P (coalesced thread-per-row access, L2-resident for the
// configs' panel heights); every column step is a tiny pivot kernel (argmax of
// the per-CTA candidates) plus one grid-wide update kernel that also emits the
// next column's candidates.
#include <cfloat>

#include "internal.cuh"

namespace fb {
namespace {

constexpr int NB = 32;
constexpr int kT = 256;

struct Cand {
    double v;
    int32_t pos, row;
};

__device__ __forceinline__ bool better(double v, int32_t p, double bv, int32_t bp) {
    return v > bv || (v == bv && p < bp);
}

// block-wide reduction of (v, pos, row); result valid in thread 0
__device__ Cand block_best(Cand c) {
    __shared__ Cand sh[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, c.v, o);
        const int32_t p = __shfl_xor_sync(0xffffffffu, c.pos, o);
        const int32_t r = __shfl_xor_sync(0xffffffffu, c.row, o);
        if (better(v, p, c.v, c.pos)) { c.v = v; c.pos = p; c.row = r; }
    }
    if (lane == 0) sh[warp] = c;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        c = lane < nw ? sh[lane] : Cand{-1.0, INT32_MAX, -1};
        for (int o = 16; o; o >>= 1) {
            const double v = __shfl_xor_sync(0xffffffffu, c.v, o);
            const int32_t p = __shfl_xor_sync(0xffffffffu, c.pos, o);
            const int32_t r = __shfl_xor_sync(0xffffffffu, c.row, o);
            if (better(v, p, c.v, c.pos)) { c.v = v; c.pos = p; c.row = r; }
        }
    }
    __syncthreads();
    return c;
}

__global__ void k_init(int32_t* pos, int32_t* perm, int64_t m) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x)
        pos[i] = perm[i] = int32_t(i);
}

// P (column-major m x bw) <- W[:, jb:jb+bw]; candidates for column jb.
__global__ void __launch_bounds__(kT)
k_panel_load(const double* __restrict__ W, int64_t m, int l, int jb, int bw, double* __restrict__ P,
             const int32_t* __restrict__ pos, Cand* __restrict__ cand) {
    const int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x;
    Cand c{-1.0, INT32_MAX, -1};
    if (i < m) {
        const double* wr = W + i * l + jb;
        for (int t = 0; t < bw; ++t) P[int64_t(t) * m + i] = wr[t];
        const int32_t p = pos[i];
        if (p >= jb) c = Cand{fabs(wr[0]), p, int32_t(i)};
    }
    c = block_best(c);
    if (threadIdx.x == 0) cand[blockIdx.x] = c;
}

__global__ void __launch_bounds__(kT)
k_panel_store(double* __restrict__ W, int64_t m, int l, int jb, int bw, const double* __restrict__ P) {
    const int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x;
    if (i >= m) return;
    double* wr = W + i * l + jb;
    for (int t = 0; t < bw; ++t) wr[t] = P[int64_t(t) * m + i];
}

// Reduce candidates -> pivot of step j; zero-pivot check (:81); interchange
// bookkeeping (:82-85) on pos/perm.
__global__ void __launch_bounds__(1024)
k_pivot(const Cand* __restrict__ cand, int ncand, int j, double tol, int32_t* __restrict__ pos,
        int32_t* __restrict__ perm, int32_t* __restrict__ pivrow, int* __restrict__ err) {
    Cand c{-1.0, INT32_MAX, -1};
    for (int k = threadIdx.x; k < ncand; k += blockDim.x) {
        const Cand o = cand[k];
        if (better(o.v, o.pos, c.v, c.pos)) c = o;
    }
    c = block_best(c);
    if (threadIdx.x == 0) {
        if (*err) return;
        if (!(c.v > tol) || c.row < 0) {  // best <= tol
            *err = 1;
            return;
        }
        const int32_t pr = c.row;
        const int32_t a = perm[j];
        const int32_t pb = pos[pr];
        perm[j] = pr;
        perm[pb] = a;
        pos[pr] = j;
        pos[a] = pb;
        pivrow[j] = pr;
    }
}

// Step j of the unblocked panel factorisation (:86-93) + candidates of j+1.
__global__ void __launch_bounds__(kT)
k_panel_update(double* __restrict__ P, int64_t m, int jb, int bw, int j,
               const int32_t* __restrict__ pos, const int32_t* __restrict__ pivrow,
               const int* __restrict__ err, Cand* __restrict__ cand) {
    if (*err) return;
    __shared__ double u[NB];
    const int cl = j - jb;
    const int32_t pr = pivrow[j];
    if (threadIdx.x < bw) u[threadIdx.x] = P[int64_t(threadIdx.x) * m + pr];
    __syncthreads();
    const double d = u[cl];
    const int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x;
    Cand c{-1.0, INT32_MAX, -1};
    if (i < m) {
        const int32_t p = pos[i];
        if (p > j) {
            const double mi = P[int64_t(cl) * m + i] / d;
            P[int64_t(cl) * m + i] = mi;
            for (int t = cl + 1; t < bw; ++t) {
                double* e = P + int64_t(t) * m + i;
                *e = *e - mi * u[t];
            }
            if (cl + 1 < bw) c = Cand{fabs(P[int64_t(cl + 1) * m + i]), p, int32_t(i)};
        }
    }
    if (cl + 1 < bw) {
        c = block_best(c);
        if (threadIdx.x == 0) cand[blockIdx.x] = c;
    }
}

// U12 = L11^{-1} A12 on the bw pivot rows (:98-100); one thread per column.
__global__ void k_trsm(double* __restrict__ W, int l, int jb, int bw, const int32_t* __restrict__ pivrow,
                       const int* __restrict__ err) {
    if (*err) return;
    __shared__ double L[NB][NB + 1];
    __shared__ int32_t rows[NB];
    if (threadIdx.x < bw) rows[threadIdx.x] = pivrow[jb + threadIdx.x];
    __syncthreads();
    for (int e = threadIdx.x; e < bw * bw; e += blockDim.x) {
        const int t = e / bw, s = e % bw;
        L[t][s] = W[int64_t(rows[t]) * l + jb + s];
    }
    __syncthreads();
    for (int c = jb + bw + blockIdx.x * blockDim.x + threadIdx.x; c < l; c += gridDim.x * blockDim.x) {
        double x[NB];
        for (int t = 0; t < bw; ++t) {
            double acc = W[int64_t(rows[t]) * l + c];
            for (int s = 0; s < t; ++s) acc -= L[t][s] * x[s];
            x[t] = acc;
            W[int64_t(rows[t]) * l + c] = acc;
        }
    }
}

// A22 -= L21 * U12 (:101-104) for non-pivot rows; candidates for column jb+bw.
// One warp per row; lanes over the trailing columns (coalesced row-major).
__global__ void __launch_bounds__(kT)
k_trailing(double* __restrict__ W, int64_t m, int l, int jb, int bw, const int32_t* __restrict__ pos,
           const int32_t* __restrict__ pivrow, const int* __restrict__ err, Cand* __restrict__ cand) {
    if (*err) return;
    extern __shared__ double U[];  // bw x tcols
    const int c0 = jb + bw, tcols = l - c0;
    for (int e = threadIdx.x; e < bw * tcols; e += blockDim.x) {
        const int t = e / tcols, cc = e % tcols;
        U[e] = W[int64_t(pivrow[jb + t]) * l + c0 + cc];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * kT + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * kT) >> 5;
    Cand best{-1.0, INT32_MAX, -1};
    for (int64_t i = warp; i < m; i += nwarps) {
        const int32_t p = pos[i];
        if (p < c0) continue;
        double* wr = W + i * l;
        const double lv = lane < bw ? wr[jb + lane] : 0.0;
        for (int cb = 0; cb < tcols; cb += 32) {
            const int cc = cb + lane;
            const bool on = cc < tcols;
            double acc = on ? wr[c0 + cc] : 0.0;
            for (int t = 0; t < bw; ++t) {
                const double lt = __shfl_sync(0xffffffffu, lv, t);
                if (on) acc -= lt * U[t * tcols + cc];
            }
            if (on) wr[c0 + cc] = acc;
            if (cc == 0) {
                const double v = fabs(acc);
                if (better(v, p, best.v, best.pos)) best = Cand{v, p, int32_t(i)};
            }
        }
    }
    best = block_best(best);
    if (threadIdx.x == 0) cand[blockIdx.x] = best;
}

// Output assembly (:108-115): X[r][j] = (j == pos) ? 1 : (j < pos ? W[r][j] : 0).
__global__ void k_assemble(double* __restrict__ W, int64_t m, int l, const int32_t* __restrict__ pos) {
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
    const double maxabs = maxabs_device(c, W, m * l);
    const double tol = double(l) * DBL_EPSILON * maxabs;
    DBuf<int32_t> pos(size_t(m), s), perm(size_t(m), s), pivrow(size_t(l), s);
    DBuf<int> err(1, s);
    FB_CUDA(cudaMemsetAsync(err.get(), 0, sizeof(int), s));
    const int nblk = int((m + kT - 1) / kT);
    const int tgrid = std::max(1, std::min(nblk, c.num_sms * 8));
    DBuf<Cand> cand(size_t(std::max(nblk, tgrid)), s);
    DBuf<double> P(size_t(m) * NB, s);
    k_init<<<std::min(nblk, c.num_sms * 16), kT, 0, s>>>(pos.get(), perm.get(), m);
    FB_LAUNCH_CHECK();
    const int L = int(l);
    for (int jb = 0; jb < L; jb += NB) {
        const int bw = std::min(NB, L - jb);
        // candidates for column jb come from the panel load (jb == 0) or the
        // previous trailing update
        int ncand = nblk;
        if (jb == 0) {
            k_panel_load<<<nblk, kT, 0, s>>>(W, m, L, jb, bw, P.get(), pos.get(), cand.get());
        } else {
            DBuf<Cand> dummy(size_t(nblk), s);
            k_panel_load<<<nblk, kT, 0, s>>>(W, m, L, jb, bw, P.get(), pos.get(), dummy.get());
            ncand = tgrid;
        }
        FB_LAUNCH_CHECK();
        for (int j = jb; j < jb + bw; ++j) {
            k_pivot<<<1, 1024, 0, s>>>(cand.get(), ncand, j, tol, pos.get(), perm.get(), pivrow.get(),
                                      err.get());
            FB_LAUNCH_CHECK();
            k_panel_update<<<nblk, kT, 0, s>>>(P.get(), m, jb, bw, j, pos.get(), pivrow.get(), err.get(),
                                              cand.get());
            FB_LAUNCH_CHECK();
            ncand = nblk;
        }
        k_panel_store<<<nblk, kT, 0, s>>>(W, m, L, jb, bw, P.get());
        FB_LAUNCH_CHECK();
        const int tcols = L - jb - bw;
        if (tcols > 0) {
            k_trsm<<<1, 256, 0, s>>>(W, L, jb, bw, pivrow.get(), err.get());
            FB_LAUNCH_CHECK();
            const size_t sm = sizeof(double) * size_t(bw) * tcols;
            if (sm > 48 * 1024)
                FB_CUDA(cudaFuncSetAttribute(k_trailing, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(sm)));
            k_trailing<<<tgrid, kT, sm, s>>>(W, m, L, jb, bw, pos.get(), pivrow.get(), err.get(),
                                            cand.get());
            FB_LAUNCH_CHECK();
        }
    }
    int h_err = 0;
    FB_CUDA(cudaMemcpyAsync(&h_err, err.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaStreamSynchronize(s));
    if (h_err) throw NumericalError("lu_basis: zero pivot, input is rank-deficient");
    const int agrid = int(std::max<int64_t>(1, std::min<int64_t>(c.num_sms * 16, (m * l + 255) / 256)));
    k_assemble<<<agrid, 256, 0, s>>>(W, m, L, pos.get());
    FB_LAUNCH_CHECK();
}

}  // namespace fb
