// Validation metrics on the device (validation.hpp:125-282):
// low_rank_error (spectral: matrix-free power iteration on R^T R with
// R = A - U diag(S) V^T, through the K1/K2 SpMM kernels; Frobenius: dense
// residual below the entry limit, cross-term identity above it),
// pc_correlation and projector_distance. Same start vectors (the Omega stream
// with the reference's seeds), stopping rule and messages as the reference;
// every reduction is in a fixed order (deterministic).
#include <cfloat>
#include <cmath>

#include "driver.cuh"

namespace fb {
namespace {

constexpr int kVT = 256;
constexpr int kVBlocks = 296;  // 2 per SM

__device__ __forceinline__ double block_reduce(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
    return s;  // valid on thread 0
}

// part[blk][i] = sum over the block's rows of A[r, i] * B[r, i] (column-major,
// ld = rows); B == nullptr: A[r, i] * x[r] with x = xv
__global__ void __launch_bounds__(kVT)
k_coldot_part(const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ xv,
              int64_t rows, int k, double* __restrict__ part) {
    __shared__ double red[kVT / 32];
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = int64_t(blockIdx.x) * per, r1 = min(rows, r0 + per);
    for (int i = 0; i < k; ++i) {
        const double* a = A + int64_t(i) * rows;
        const double* b = B ? B + int64_t(i) * rows : xv;
        double s = 0.0;
        for (int64_t r = r0 + threadIdx.x; r < r1; r += kVT) s = fma(a[r], b[r], s);
        s = block_reduce(s, red);
        if (threadIdx.x == 0) part[int64_t(blockIdx.x) * k + i] = s;
    }
}

__global__ void k_part_sum(const double* __restrict__ part, int nblk, int k, const double* __restrict__ scale,
                           double* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < nblk; ++b) s += part[int64_t(b) * k + i];
        out[i] = scale ? scale[i] * s : s;
    }
}

// y[r] += sgn * sum_i M[r, i] t[i]  (M column-major rows x k)
__global__ void k_gemv_acc(const double* __restrict__ M, int64_t rows, int k, const double* __restrict__ t,
                           double sgn, double* __restrict__ y) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < k; ++i) s = fma(M[r + int64_t(i) * rows], t[i], s);
        y[r] = fma(sgn, s, y[r]);
    }
}

// X[:, i] -= mean[i] (column-major rows x k)
__global__ void k_center(double* __restrict__ X, int64_t rows, int k, const double* __restrict__ mean) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < rows * k; e += int64_t(gridDim.x) * blockDim.x)
        X[e] -= mean[e / rows];
}

__global__ void k_vdiv(const double* __restrict__ u, int64_t n, double d, double* __restrict__ v) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        v[i] = u[i] / d;
}

// dense residual R (column-major m x n) = A - U diag(S) V^T
__global__ void k_lowrank_dense(const double* __restrict__ U, const double* __restrict__ S,
                                const double* __restrict__ V, int64_t m, int64_t n, int k, double* __restrict__ R) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * n; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e % m, c = e / m;
        double s = 0.0;
        for (int i = 0; i < k; ++i) s += U[r + int64_t(i) * m] * S[i] * V[c + int64_t(i) * n];
        R[e] -= s;
    }
}

// (A's ids may carry the A*X launch encodings: decoded through rank_ids)
__global__ void k_scatter_dense(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                const double* __restrict__ val, int64_t m, const int32_t* __restrict__ rank_ids,
                                double* __restrict__ R) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            const int32_t e = col[p];
            const int32_t cc = (e & kColHot) ? rank_ids[e & kRankMask] : (e & kColMask);
            R[i + int64_t(cc) * m] = val[p];
        }
}

int vgrid(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>(4096, (n + 255) / 256))); }

// per-column dot products (or M^T x), fixed order: out (device, k)
void coldots(Ctx& c, const double* A, const double* B, const double* x, int64_t rows, int k, double* out,
             const double* scale = nullptr) {
    DBuf<double> part(size_t(kVBlocks) * k, c.stream);
    k_coldot_part<<<kVBlocks, kVT, 0, c.stream>>>(A, B, x, rows, k, part.get());
    FB_LAUNCH_CHECK();
    k_part_sum<<<1, 256, 0, c.stream>>>(part.get(), kVBlocks, k, scale, out);
    FB_LAUNCH_CHECK();
}

double dot_host(Ctx& c, const double* a, const double* b, int64_t n) {
    DBuf<double> d(1, c.stream);
    coldots(c, a, nullptr, b, n, 1, d.get());
    double h = 0.0;
    FB_CUDA(cudaMemcpyAsync(&h, d.get(), sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    FB_CUDA(cudaStreamSynchronize(c.stream));
    return h;
}

// operator_two_norm (validation.hpp:145-165) on device vectors
template <class Ap, class ApT>
double two_norm(Ctx& c, int64_t ncols, int64_t nrows, uint64_t seed, Ap apply, ApT apply_t) {
    DBuf<double> v(size_t(ncols), c.stream), w(size_t(std::max<int64_t>(nrows, 1)), c.stream),
        u(size_t(ncols), c.stream);
    gaussian_stream_device(c, seed, ncols, v.get());
    const double nv = std::sqrt(dot_host(c, v.get(), v.get(), ncols));
    k_vdiv<<<vgrid(ncols), 256, 0, c.stream>>>(v.get(), ncols, nv, v.get());
    FB_LAUNCH_CHECK();
    double lambda_prev = 0.0;
    for (int it = 0; it < 2000; ++it) {
        apply(v.get(), w.get());
        apply_t(w.get(), u.get());
        const double lambda = dot_host(c, v.get(), u.get(), ncols);
        const double nu = std::sqrt(dot_host(c, u.get(), u.get(), ncols));
        if (nu == 0.0) return 0.0;
        k_vdiv<<<vgrid(ncols), 256, 0, c.stream>>>(u.get(), ncols, nu, v.get());
        FB_LAUNCH_CHECK();
        if (it > 0 && std::fabs(lambda - lambda_prev) <= 1e-12 * std::fabs(lambda)) {
            lambda_prev = lambda;
            break;
        }
        lambda_prev = lambda;
    }
    return std::sqrt(std::max(lambda_prev, 0.0));
}

// column-major (rows x k) -> row-major copy
void to_rowmajor(Ctx& c, const double* cm, int64_t rows, int64_t k, double* rm) {
    transpose_device(c, cm, k, rows, rm);
}

}  // namespace

double low_rank_error_device(Ctx& c, DMat& M, int64_t k, const double* U, const double* S, const double* V,
                             int norm, uint64_t entry_limit) {
    require(c.world == 1, "low_rank_error: single GPU only");
    const int64_t m = M.A.rows, n = M.A.cols;
    cudaStream_t s = c.stream;
    if (norm == FRPCA_NORM_SPECTRAL) {
        DBuf<double> t(size_t(std::max<int64_t>(k, 1)), s);
        auto apply = [&](const double* x, double* y) {  // y = A x - U (S .* (V^T x))
            spmm_pass(c, M, false, x, 1, y);
            if (k) {
                coldots(c, V, nullptr, x, n, int(k), t.get(), S);
                k_gemv_acc<<<vgrid(m), 256, 0, s>>>(U, m, int(k), t.get(), -1.0, y);
                FB_LAUNCH_CHECK();
            }
        };
        auto apply_t = [&](const double* y, double* x) {  // x = A^T y - V (S .* (U^T y))
            spmm_pass(c, M, true, y, 1, x);
            if (k) {
                coldots(c, U, nullptr, y, m, int(k), t.get(), S);
                k_gemv_acc<<<vgrid(n), 256, 0, s>>>(V, n, int(k), t.get(), -1.0, x);
                FB_LAUNCH_CHECK();
            }
        };
        return two_norm(c, n, m, 0x9e3779b9u, apply, apply_t);
    }
    const uint64_t entries = uint64_t(m) * uint64_t(n);
    if (entries <= entry_limit) {
        DBuf<double> R(size_t(std::max<uint64_t>(entries, 1)), s);
        FB_CUDA(cudaMemsetAsync(R.get(), 0, R.bytes(), s));
        if (m) {
            k_scatter_dense<<<vgrid(m), 256, 0, s>>>(M.A.rowptr.get(), M.A.col.get(), M.A.val.get(), m,
                                                     M.A.rank_ids.get(), R.get());
            FB_LAUNCH_CHECK();
        }
        if (k && entries) {
            k_lowrank_dense<<<vgrid(int64_t(entries)), 256, 0, s>>>(U, S, V, m, n, int(k), R.get());
            FB_LAUNCH_CHECK();
        }
        return std::sqrt(dot_host(c, R.get(), R.get(), int64_t(entries)));
    }
    // |A - M|^2 = |A|^2 - 2 <A, M> + |M|^2 (validation.hpp:189-202)
    const double a2 = dot_host(c, M.A.val.get(), M.A.val.get(), M.A.nnz);
    if (k == 0) return std::sqrt(std::max(a2, 0.0));
    DBuf<double> Vr(size_t(n * k), s), Wr(size_t(m * k), s), Wc(size_t(m * k), s), Ur(size_t(m * k), s),
        d(size_t(k), s), gu(size_t(k * k), s), gv(size_t(k * k), s);
    to_rowmajor(c, V, n, k, Vr.get());
    spmm_pass(c, M, false, Vr.get(), k, Wr.get());          // W = A V, m x k
    transpose_device(c, Wr.get(), m, k, Wc.get());          // column-major
    coldots(c, U, Wc.get(), nullptr, m, int(k), d.get(), S);  // S_i U_i . W_i
    to_rowmajor(c, U, m, k, Ur.get());
    gram_device(c, Ur.get(), m, k, gu.get());
    gram_device(c, Vr.get(), n, k, gv.get());
    std::vector<double> hd(static_cast<size_t>(k)), hgu(static_cast<size_t>(k * k)), hgv(static_cast<size_t>(k * k)),
        hS(static_cast<size_t>(k));
    FB_CUDA(cudaMemcpyAsync(hd.data(), d.get(), sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaMemcpyAsync(hgu.data(), gu.get(), sizeof(double) * k * k, cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaMemcpyAsync(hgv.data(), gv.get(), sizeof(double) * k * k, cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaMemcpyAsync(hS.data(), S, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaStreamSynchronize(s));
    double cross = 0.0, m2 = 0.0;
    for (int64_t i = 0; i < k; ++i) cross += hd[size_t(i)];
    for (int64_t i = 0; i < k; ++i)
        for (int64_t j = 0; j < k; ++j)
            m2 += hS[size_t(i)] * hS[size_t(j)] * hgu[size_t(i + j * k)] * hgv[size_t(i + j * k)];
    return std::sqrt(std::max(a2 - 2.0 * cross + m2, 0.0));
}

void pc_correlation_device(Ctx& c, int64_t m, int64_t k, const double* Ut, const double* Ur, double* corr_host) {
    require(m >= 2, "pc_correlation: need at least two samples");
    if (k == 0) return;
    cudaStream_t s = c.stream;
    DBuf<double> ones(size_t(m), s), sx(size_t(k), s), sy(size_t(k), s), Xc(size_t(m * k), s), Yc(size_t(m * k), s),
        xy(size_t(k), s), xx(size_t(k), s), yy(size_t(k), s);
    std::vector<double> h1(static_cast<size_t>(m), 1.0);
    FB_CUDA(cudaMemcpyAsync(ones.get(), h1.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s));
    coldots(c, Ut, nullptr, ones.get(), m, int(k), sx.get());
    coldots(c, Ur, nullptr, ones.get(), m, int(k), sy.get());
    std::vector<double> mx(static_cast<size_t>(k)), my(static_cast<size_t>(k));
    FB_CUDA(cudaMemcpyAsync(mx.data(), sx.get(), sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaMemcpyAsync(my.data(), sy.get(), sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaStreamSynchronize(s));
    // centred copies (validation.hpp:237-238)
    for (int64_t i = 0; i < k; ++i) {
        mx[size_t(i)] /= double(m);
        my[size_t(i)] /= double(m);
    }
    FB_CUDA(cudaMemcpyAsync(sx.get(), mx.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s));
    FB_CUDA(cudaMemcpyAsync(sy.get(), my.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s));
    FB_CUDA(cudaMemcpyAsync(Xc.get(), Ut, sizeof(double) * m * k, cudaMemcpyDeviceToDevice, s));
    FB_CUDA(cudaMemcpyAsync(Yc.get(), Ur, sizeof(double) * m * k, cudaMemcpyDeviceToDevice, s));
    k_center<<<vgrid(m * k), 256, 0, s>>>(Xc.get(), m, int(k), sx.get());
    FB_LAUNCH_CHECK();
    k_center<<<vgrid(m * k), 256, 0, s>>>(Yc.get(), m, int(k), sy.get());
    FB_LAUNCH_CHECK();
    coldots(c, Xc.get(), Yc.get(), nullptr, m, int(k), xy.get());
    coldots(c, Xc.get(), Xc.get(), nullptr, m, int(k), xx.get());
    coldots(c, Yc.get(), Yc.get(), nullptr, m, int(k), yy.get());
    std::vector<double> hxy(static_cast<size_t>(k)), hxx(static_cast<size_t>(k)), hyy(static_cast<size_t>(k));
    FB_CUDA(cudaMemcpyAsync(hxy.data(), xy.get(), sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaMemcpyAsync(hxx.data(), xx.get(), sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaMemcpyAsync(hyy.data(), yy.get(), sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaStreamSynchronize(s));
    for (int64_t j = 0; j < k; ++j) {
        const double denom = std::sqrt(hxx[size_t(j)]) * std::sqrt(hyy[size_t(j)]);
        if (denom == 0.0) throw InvalidArgument("pc_correlation: zero-variance column " + std::to_string(j));
        corr_host[j] = std::fabs(hxy[size_t(j)] / denom);
    }
}

double projector_distance_device(Ctx& c, int64_t m, int64_t k1, const double* Q1, int64_t k2, const double* Q2) {
    cudaStream_t s = c.stream;
    auto check = [&](const double* Q, int64_t k, const char* which) {
        if (k == 0) return;
        DBuf<double> Qr(size_t(m * k), s), G(size_t(k * k), s);
        to_rowmajor(c, Q, m, k, Qr.get());
        gram_device(c, Qr.get(), m, k, G.get());
        std::vector<double> h(static_cast<size_t>(k * k));
        FB_CUDA(cudaMemcpyAsync(h.data(), G.get(), sizeof(double) * k * k, cudaMemcpyDeviceToHost, s));
        FB_CUDA(cudaStreamSynchronize(s));
        double mx = 0.0;
        for (int64_t i = 0; i < k; ++i)
            for (int64_t j = 0; j < k; ++j) mx = std::max(mx, std::fabs(h[size_t(i + j * k)] - (i == j ? 1.0 : 0.0)));
        if (mx > 1e-8)
            throw InvalidArgument(std::string("projector_distance: ") + which + " is not orthonormal within 1e-8");
    };
    check(Q1, k1, "first basis");
    check(Q2, k2, "second basis");
    DBuf<double> t1(size_t(std::max<int64_t>(k1, 1)), s), t2(size_t(std::max<int64_t>(k2, 1)), s);
    auto apply = [&](const double* x, double* y) {  // y = Q1 Q1^T x - Q2 Q2^T x
        FB_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * m, s));
        if (k1) {
            coldots(c, Q1, nullptr, x, m, int(k1), t1.get());
            k_gemv_acc<<<vgrid(m), 256, 0, s>>>(Q1, m, int(k1), t1.get(), 1.0, y);
            FB_LAUNCH_CHECK();
        }
        if (k2) {
            coldots(c, Q2, nullptr, x, m, int(k2), t2.get());
            k_gemv_acc<<<vgrid(m), 256, 0, s>>>(Q2, m, int(k2), t2.get(), -1.0, y);
            FB_LAUNCH_CHECK();
        }
    };
    return two_norm(c, m, m, 0x51f15eedu, apply, apply);
}

}  // namespace fb
