// Device drivers of the two fast algorithms: frpca (Alg. 5, randsvd.hpp:224-276)
// and frpcat (Alg. 6, randsvd.hpp:278-328), plus eig_svd (dense_kernels.hpp:
// 145-174) as the device pipeline Gram -> syevd -> rank check -> rescale.
//
// All intermediate panels stay in HBM, row-major r x l. The host sees only the
// final U/S/V (column-major, like SvdResult) and the scalars needed for the
// reference's error checks (the l eigenvalues for the rank test).
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstring>

#include "driver.cuh"

namespace fb {
namespace {

// RunStats stage times (randsvd.hpp:42-53) from events on the run's stream,
// so the stages need no host synchronisation between them.
struct StageTimer {
    cudaStream_t s;
    cudaEvent_t ev[4] = {};
    explicit StageTimer(cudaStream_t st) : s(st) {
        for (auto& e : ev) FB_CUDA(cudaEventCreate(&e));
    }
    ~StageTimer() {
        for (auto e : ev) cudaEventDestroy(e);
    }
    void mark(int i) { FB_CUDA(cudaEventRecord(ev[i], s)); }
    double seconds(int i) const {  // stage i: between marks i and i + 1 (stream complete)
        float ms = 0.f;
        FB_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
        return 1e-3 * double(ms);
    }
};

// M (row-major l x ncols): column t takes eigenvector src(t) of V (column-major
// l x l), src(t) = rev ? s + k - 1 - t : t, scaled by 1/S[src] when `scale`
// (V * diag(1/S), dense_kernels.hpp:172; reversal ind = s+k-1..s,
// randsvd.hpp:265-267 / :317-319).
__global__ void k_factor(const double* __restrict__ V, const double* __restrict__ D, int l, int s,
                         int k, int ncols, int rev, int scale, double* __restrict__ M) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < l * ncols; e += gridDim.x * blockDim.x) {
        const int kk = e / ncols, t = e % ncols;
        const int src = rev ? (s + k - 1 - t) : t;
        double v = V[kk + int64_t(src) * l];
        if (scale) {
            const double inv = 1.0 / sqrt(D[src]);
            v = v * inv;
        }
        M[e] = v;
    }
}

// rank check of eig_svd (dense_kernels.hpp:163-167) on the device: the same
// comparison as the reference (a NaN spectrum passes it, as there)
__global__ void k_rank_check(const double* __restrict__ D, int n, int* __restrict__ flag) {
    const double lambda_max = D[n - 1];
    if (lambda_max <= 0.0 || D[0] <= double(n) * DBL_EPSILON * lambda_max) atomicCAS(flag, 0, kErrEigRank);
}

__global__ void k_sing_out(const double* __restrict__ D, int s, int k, int rev, double* __restrict__ S) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < k; t += gridDim.x * blockDim.x)
        S[t] = sqrt(D[rev ? (s + k - 1 - t) : t]);
}

}  // namespace

void EigWork::run(Ctx& c, const double* W, int64_t r, int64_t n, bool row_sharded, double* keep_gram) {
    B.alloc(size_t(n * n), c.stream);
    D.alloc(size_t(n), c.stream);
    gram_device(c, W, r, n, B.get());
    if (row_sharded) allreduce_sum(c, B.get(), n * n);  // Gram partials of the rank's rows
    if (keep_gram)
        FB_CUDA(cudaMemcpyAsync(keep_gram, B.get(), sizeof(double) * size_t(n * n), cudaMemcpyDeviceToDevice,
                                c.stream));
    syevd_device(c, B.get(), n, D.get(), row_sharded);
    // rank check (dense_kernels.hpp:163-167), reported by err_check
    k_rank_check<<<1, 1, 0, c.stream>>>(D.get(), int(n), err_flag(c));
    FB_LAUNCH_CHECK();
    l = n;
}

void EigWork::factor(Ctx& c, int s, int k, int ncols, bool rev, bool scale, double* M) {
    const int total = int(l) * ncols;
    k_factor<<<std::max(1, std::min(1024, (total + 255) / 256)), 256, 0, c.stream>>>(
        B.get(), D.get(), int(l), s, k, ncols, rev ? 1 : 0, scale ? 1 : 0, M);
    FB_LAUNCH_CHECK();
}

void EigWork::singular_values(Ctx& c, int s, int k, bool rev, double* S) {
    k_sing_out<<<1, 256, 0, c.stream>>>(D.get(), s, k, rev ? 1 : 0, S);
    FB_LAUNCH_CHECK();
}

// eig_svd(W).U: Uout (row-major r x n) = W * V diag(1/S), for a W that is
// replicated on every rank (the power iteration's Z / Y after their allreduce).
//
// Refinement of the rescale factor. In exact arithmetic M0 = V diag(1/S)
// satisfies M0^T B M0 = I (B = W^T W), i.e. Q = W M0 is orthonormal. A
// tridiagonal eigensolver resolves B's eigenpairs to eps*lambda_max
// (absolute), so for a graded power-iteration panel (lambda_max/lambda_min up
// to ~1e12 after two applications of A^T A) Q loses orthonormality by
// 1e-8..1e-4 and the error leaks into the leading k directions: 3e-9 on sigma
// where the oracle (Jacobi, relative accuracy, like the reference's Eigen
// solver on a graded matrix) is at 2e-14 from the long-double arbiter
// (tools/fuzz_parity.py, tools/probe/eig_loop_orth.py). The defect E =
// M0^T B M0 - I is an l x l quantity: it is measured from the Gram matrix
// already at hand and removed with the symmetric (Loewdin) correction
// T = I - E/2 + 3/8 E^2 = (I + E)^(-1/2) + O(E^3), folded into the factor
// before the one tall product: Q = W (M0 T). T is the orthonormaliser closest
// to the identity, so the basis keeps the eigenvector rotation of the
// reference's result. Four l x l x l products (~64 MFLOP at l = 200, tens of
// microseconds); no extra pass over W. FRPCA_EIG_REFINE=0 disables (A/B).
namespace {
constexpr int MT = 16;
// C (row-major l x l) = A * Bm with element strides (row, col) per operand,
// k summed in index order. mode 0: the product; 1: product - I; 2:
// I - X/2 + 3/8 product (X row-major, the matrix being squared).
__global__ void k_mm_ll(const double* __restrict__ A, int ar, int ac, const double* __restrict__ Bm, int br,
                        int bc, double* __restrict__ C, int l, int mode, const double* __restrict__ X) {
    __shared__ double sa[MT][MT + 1], sb[MT][MT + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int i = blockIdx.y * MT + ty, j = blockIdx.x * MT + tx;
    double acc = 0.0;
    for (int k0 = 0; k0 < l; k0 += MT) {
        const int ka = k0 + tx, kb = k0 + ty;
        sa[ty][tx] = (i < l && ka < l) ? A[int64_t(i) * ar + int64_t(ka) * ac] : 0.0;
        sb[ty][tx] = (kb < l && j < l) ? Bm[int64_t(kb) * br + int64_t(j) * bc] : 0.0;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MT; ++k) acc = fma(sa[ty][k], sb[k][tx], acc);
        __syncthreads();
    }
    if (i < l && j < l) {
        const double eye = (i == j) ? 1.0 : 0.0;
        double out = acc;
        if (mode == 1) out = acc - eye;
        else if (mode == 2) out = eye - 0.5 * X[int64_t(i) * l + j] + 0.375 * acc;
        C[int64_t(i) * l + j] = out;
    }
}
void mm_ll(Ctx& c, const double* A, int ar, int ac, const double* Bm, int br, int bc, double* C, int l, int mode,
           const double* X = nullptr) {
    const dim3 grid((l + MT - 1) / MT, (l + MT - 1) / MT), block(MT, MT);
    k_mm_ll<<<grid, block, 0, c.stream>>>(A, ar, ac, Bm, br, bc, C, l, mode, X);
    FB_LAUNCH_CHECK();
}
}  // namespace

void eig_svd_U(Ctx& c, const double* W, int64_t r, int64_t n, double* Uout) {
    const char* env = std::getenv("FRPCA_EIG_REFINE");
    const bool refine = !(env && *env == '0');
    EigWork e;
    DBuf<double> G;
    if (refine) G.alloc(size_t(n * n), c.stream);
    e.run(c, W, r, n, /*row_sharded=*/false, refine ? G.get() : nullptr);
    DBuf<double> M(size_t(n * n), c.stream);
    e.factor(c, 0, int(n), int(n), false, true, M.get());   // M0 = V diag(1/S), row-major
    if (!refine) {
        gemm_device(c, W, r, n, M.get(), n, Uout, n, false);
        return;
    }
    const int l = int(n);
    DBuf<double> P(size_t(n * n), c.stream), E(size_t(n * n), c.stream);
    {
    Prof prof(c, "eig_refine", 8.0 * 9 * n * n, 8.0 * n * n * n);
    mm_ll(c, G.get(), 1, l, M.get(), l, 1, P.get(), l, 0);             // P = B M0 (B column-major, symmetric)
    mm_ll(c, M.get(), 1, l, P.get(), l, 1, E.get(), l, 1);             // E = M0^T P - I
    mm_ll(c, E.get(), l, 1, E.get(), l, 1, P.get(), l, 2, E.get());    // T = I - E/2 + 3/8 E E   (into P)
    mm_ll(c, M.get(), l, 1, P.get(), l, 1, G.get(), l, 0);             // M = M0 T               (into G)
    }
    gemm_device(c, W, r, n, G.get(), n, Uout, n, false);
}

// Omega of the sketch (randsvd.hpp:65-76): `count` doubles in stream order
// (the column-major fill of gaussian_matrix), either the injected matrix or
// the seeded stream, into device memory.
void sketch_stream(Ctx& c, const RunArgs& a, int64_t rows, int64_t cols, double* dst) {
    const int64_t count = rows * cols;
    if (a.omega) {
        require(a.omega_rows == rows && a.omega_cols == cols, "injected sketch has the wrong shape");
        FB_CUDA(cudaMemcpyAsync(dst, a.omega, sizeof(double) * count,
                                a.device_io ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                c.stream));
        return;
    }
    const uint64_t seed = mix_seed(a.cfg.seed, 0xA11CEull);
    if (a.cfg.flags & FRPCA_FLAG_HOST_OMEGA) {
        Prof prof(c, "omega_host", 8.0 * count, 0.0);
        std::vector<double> h(static_cast<size_t>(count));
        gaussian_stream_host(seed, count, h.data());
        FB_CUDA(cudaMemcpyAsync(dst, h.data(), sizeof(double) * count, cudaMemcpyHostToDevice, c.stream));
        FB_CUDA(cudaStreamSynchronize(c.stream));
    } else {
        gaussian_stream_device(c, seed, count, dst);
    }
}

// Rows [r0, r1) of the sketch Omega (rows x cols, column-major stream order)
// into dst ((r1 - r0) x cols, column-major): a rank's slice of the sketch of a
// sharded run. Only the slice is written (the device generator emits just
// the slice's stream positions).
static void sketch_rows(Ctx& c, const RunArgs& a, int64_t rows, int64_t cols, int64_t r0, int64_t r1,
                        double* dst) {
    const int64_t nr = r1 - r0;
    if (nr == rows) return sketch_stream(c, a, rows, cols, dst);
    if (a.omega) {
        require(a.omega_rows == rows && a.omega_cols == cols, "injected sketch has the wrong shape");
        FB_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * nr, a.omega + r0, sizeof(double) * rows, sizeof(double) * nr,
                                  size_t(cols), a.device_io ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                  c.stream));
        return;
    }
    const uint64_t seed = mix_seed(a.cfg.seed, 0xA11CEull);
    if (a.cfg.flags & FRPCA_FLAG_HOST_OMEGA) {
        std::vector<double> h(static_cast<size_t>(rows * cols));
        gaussian_stream_host(seed, rows * cols, h.data());
        FB_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * nr, h.data() + r0, sizeof(double) * rows, sizeof(double) * nr,
                                  size_t(cols), cudaMemcpyHostToDevice, c.stream));
        FB_CUDA(cudaStreamSynchronize(c.stream));
        return;
    }
    // the stream up to the slice's last element
    gaussian_stream_window(c, seed, (cols - 1) * rows + r1, rows, r0, r1, dst);
}

// Columns [c0, c1) of Omega (rows x cols, column-major): one contiguous run
// of the stream, [c0 rows, c1 rows), generated only up to its end.
static void sketch_cols(Ctx& c, const RunArgs& a, int64_t rows, int64_t cols, int64_t c0, int64_t c1, double* dst) {
    if (c0 == 0 && c1 == cols) return sketch_stream(c, a, rows, cols, dst);
    const int64_t b0 = c0 * rows, b1 = c1 * rows;
    if (a.omega) {
        require(a.omega_rows == rows && a.omega_cols == cols, "injected sketch has the wrong shape");
        FB_CUDA(cudaMemcpyAsync(dst, a.omega + b0, sizeof(double) * (b1 - b0),
                                a.device_io ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
        return;
    }
    const uint64_t seed = mix_seed(a.cfg.seed, 0xA11CEull);
    if (a.cfg.flags & FRPCA_FLAG_HOST_OMEGA) {
        std::vector<double> h(static_cast<size_t>(b1));
        gaussian_stream_host(seed, b1, h.data());
        FB_CUDA(cudaMemcpyAsync(dst, h.data() + b0, sizeof(double) * (b1 - b0), cudaMemcpyHostToDevice, c.stream));
        FB_CUDA(cudaStreamSynchronize(c.stream));
        return;
    }
    gaussian_stream_window(c, seed, b1, b1, b0, b1, dst);
}

// Omega (rows x cols, column-major stream order) into dst: the pre-generated
// stream when frpca_run_csr overlapped it with the upload, else generated now.
static void sketch_into(Ctx& c, const RunArgs& a, int64_t rows, int64_t cols, DBuf<double>& dst) {
    const size_t count = size_t(rows) * size_t(cols);
    if (a.pre && !a.pre_rowmajor && a.pre->get() && a.pre->n >= count && !a.omega) {
        cudaStream_t ps = a.pre->s;
        std::swap(dst, *a.pre);  // both buffers stay allocated (workspace slots)
        dst.s = c.stream;
        a.pre->s = ps;
        return;
    }
    if (dst.n < count) dst.alloc(count, c.stream);
    sketch_stream(c, a, rows, cols, dst.get());
}

// Rows [r0, r1) of Omega (rows x cols, column-major stream order) as the
// row-major (r1 - r0) x cols panel the products gather from: generated
// straight into that layout (rng.cu k_place_rm), or the pre-generated one of
// frpca_run_csr; an injected or host-generated sketch is transposed.
static void sketch_rowmajor(Ctx& c, const RunArgs& a, int64_t rows, int64_t cols, int64_t r0, int64_t r1,
                            DBuf<double>& dst) {
    const int64_t nr = r1 - r0;
    const size_t count = size_t(nr) * size_t(cols);
    if (a.pre && a.pre_rowmajor && a.pre->get() && a.pre->n >= count && !a.omega && nr == rows) {
        cudaStream_t ps = a.pre->s;
        std::swap(dst, *a.pre);  // both buffers stay allocated (workspace slots)
        dst.s = c.stream;
        a.pre->s = ps;
        return;
    }
    if (dst.n < count) dst.alloc(count, c.stream);
    if (a.omega || (a.cfg.flags & FRPCA_FLAG_HOST_OMEGA)) {
        DBuf<double> t(count, c.stream);
        sketch_rows(c, a, rows, cols, r0, r1, t.get());   // nr x cols column-major
        transpose_device(c, t.get(), cols, nr, dst.get());
        return;
    }
    const uint64_t seed = mix_seed(a.cfg.seed, 0xA11CEull);
    gaussian_stream_window(c, seed, (cols - 1) * rows + r1, rows, r0, r1, dst.get(), /*rowmajor=*/true);
}

static void check_common(const frpca_config& cfg) {  // randsvd.hpp:78-81
    require(cfg.k >= 1, "config: rank k must be >= 1");
    require(cfg.oversample >= 0, "config: oversampling must be >= 0");
}

static void copy_out(Ctx& c, const RunArgs& a, double* dst_user, const double* src_dev, int64_t count) {
    if (!dst_user || count == 0) return;
    FB_CUDA(cudaMemcpyAsync(dst_user, src_dev, sizeof(double) * count,
                            a.device_io ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c.stream));
}

// column-major rows x k (ld = rows) -> the caller's matrix with leading dimension ld
static void copy_out_ld(Ctx& c, const RunArgs& a, double* dst_user, int64_t ld, const double* src_dev, int64_t rows,
                        int64_t k, cudaStream_t s) {
    if (!dst_user || rows == 0 || k == 0) return;
    const cudaMemcpyKind kind = a.device_io ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (ld == 0 || ld == rows) {
        FB_CUDA(cudaMemcpyAsync(dst_user, src_dev, sizeof(double) * rows * k, kind, s));
        return;
    }
    FB_CUDA(cudaMemcpy2DAsync(dst_user, sizeof(double) * ld, src_dev, sizeof(double) * rows, sizeof(double) * rows,
                              size_t(k), kind, s));
}

// Q (row-major r x l) -> column-major output basis (RunStats::basis).
static void basis_out(Ctx& c, const RunArgs& a, const double* Q, int64_t r, int64_t l) {
    if (!a.basis) return;
    DBuf<double> t(size_t(r * l), c.stream);
    transpose_device(c, Q, r, l, t.get());
    copy_out(c, a, a.basis, t.get(), r * l);
}


// The two output products (U = W_u MU, V = W_v MV, column-major, ld = rows)
// and S. With host outputs, the device->host copies overlap the GEMMs: the
// smaller product and S are computed first and copied on the copy stream
// while the larger one runs in row chunks, each chunk copied as soon as it is
// done. Chunks keep >= 4096 rows, so every entry comes from the same kernel
// and K order as the unchunked product.
struct OutProduct {
    const double* W;  // rows x l, row-major
    int64_t rows;
    const double* M;  // l x k
    double* dev;      // rows x k, column-major
    double* user;     // U or V of the call (may be null)
    int64_t ld;       // leading dimension of `user` (0: rows)
};

static void output_products(Ctx& c, const RunArgs& a, int64_t l, int64_t k, OutProduct u, OutProduct v,
                            EigWork& e, int s, double* So) {
    cudaStream_t S = c.stream;
    const bool overlap = !a.device_io && (u.user || v.user || a.S);
    if (!overlap) {
        gemm_device(c, u.W, u.rows, l, u.M, k, u.dev, std::max<int64_t>(u.rows, 1), true);
        gemm_device(c, v.W, v.rows, l, v.M, k, v.dev, std::max<int64_t>(v.rows, 1), true);
        e.singular_values(c, s, int(k), true, So);
        copy_out_ld(c, a, u.user, u.ld, u.dev, u.rows, k, S);
        copy_out_ld(c, a, v.user, v.ld, v.dev, v.rows, k, S);
        copy_out(c, a, a.S, So, k);
        return;
    }
    if (!c.copy) FB_CUDA(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
    OutProduct& big = u.rows >= v.rows ? u : v;
    OutProduct& sml = u.rows >= v.rows ? v : u;
    std::vector<cudaEvent_t> evs;
    auto fence = [&](cudaStream_t from, cudaStream_t to) {
        cudaEvent_t ev;
        FB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        evs.push_back(ev);
        FB_CUDA(cudaEventRecord(ev, from));
        FB_CUDA(cudaStreamWaitEvent(to, ev, 0));
    };
    gemm_device(c, sml.W, sml.rows, l, sml.M, k, sml.dev, std::max<int64_t>(sml.rows, 1), true);
    e.singular_values(c, s, int(k), true, So);
    fence(S, c.copy);
    copy_out_ld(c, a, sml.user, sml.ld, sml.dev, sml.rows, k, c.copy);
    if (a.S && k) FB_CUDA(cudaMemcpyAsync(a.S, So, sizeof(double) * k, cudaMemcpyDeviceToHost, c.copy));
    const int64_t R = big.rows;
    static const int64_t maxch = [] {
        const char* e = std::getenv("FRPCA_OUT_CHUNKS");
        return e ? std::max(1, std::atoi(e)) : 8;
    }();
    const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(maxch, R / 4096));
    for (int64_t q = 0; q < nch; ++q) {
        const int64_t r0 = R * q / nch, r1 = R * (q + 1) / nch;
        if (r1 == r0) continue;
        gemm_device(c, big.W + r0 * l, r1 - r0, l, big.M, k, big.dev + r0, R, true);
        if (!big.user || !k) continue;
        fence(S, c.copy);
        const int64_t ldu = big.ld ? big.ld : R;
        FB_CUDA(cudaMemcpy2DAsync(big.user + r0, sizeof(double) * ldu, big.dev + r0, sizeof(double) * R,
                                  sizeof(double) * (r1 - r0), size_t(k), cudaMemcpyDeviceToHost, c.copy));
    }
    {
        Prof pw(c, "out_d2h_tail", 0.0, 0.0);  // the copies still running after the last GEMM
        fence(c.copy, S);  // the run's final synchronisation covers the copies
    }
    FB_CUDA(cudaStreamSynchronize(S));
    for (auto ev : evs) cudaEventDestroy(ev);
}

// ---------------------------------------------------------------------------
// frpcat (Alg. 6), randsvd.hpp:278-328. Row-sharded: this rank holds rows
// [offset, offset + m_loc) of A; A^T partials and Gram partials are summed
// across ranks.
void run_frpcat(Ctx& c, DMat& M, const RunArgs& a, frpca_stats* st) {
    const frpca_config& cfg = a.cfg;
    check_common(cfg);
    require(M.grows >= M.gcols, "frpcat: requires rows >= cols (use frpca otherwise)");
    require(cfg.passes >= 2, "frpcat: pass count q must be >= 2");
    const int64_t l = cfg.k + cfg.oversample;
    require(l <= M.gcols, "frpcat: k + oversample must be <= cols");
    require(!M.col_shard, "frpcat: needs a row-sharded matrix");
    const int64_t q = cfg.passes, loops = (q - 1) / 2;
    const int64_t m = M.A.rows, n = M.A.cols, k = cfg.k, s = cfg.oversample;
    const uint64_t passes0 = M.passes.load();
    cudaStream_t S = c.stream;

    DBuf<double>& bufM = c.slot(0, size_t(std::max<int64_t>(m, 1) * l));
    DBuf<double>& Q = c.slot(1, size_t(n * l));
    DBuf<double>& Z = c.slot(2, size_t(n * l));

    StageTimer T(S);
    T.mark(0);
    if (q % 2 == 0) {
        // Omega (l x grows, column-major) == Omega^T row-major: this rank's rows
        // are the stream slice [offset*l, (offset+m)*l).
        if (M.offset == 0 && m == M.grows) sketch_into(c, a, l, M.grows, bufM);
        else sketch_cols(c, a, l, M.grows, M.offset, M.offset + m, bufM.get());
        spmm_pass_reduced(c, M, /*transpose=*/true, bufM.get(), l, Z.get());  // (Omega A)^T, n x l, summed
        if (q == 2) {
            eig_svd_U(c, Z.get(), n, l, Q.get());
        } else {
            lu_basis_device(c, Z.get(), n, l);
            std::swap(Q, Z);
        }
    } else {
        sketch_rowmajor(c, a, n, l, 0, n, Q);             // Q = Omega, row-major n x l
    }
    T.mark(1);

    for (int64_t i = 1; i <= loops; ++i) {
        spmm_pass(c, M, false, Q.get(), l, bufM.get());   // A Q, m x l
        spmm_pass_reduced(c, M, true, bufM.get(), l, Z.get());  // A^T (A Q), n x l, summed over ranks
        if (i == loops) {
            eig_svd_U(c, Z.get(), n, l, Q.get());
        } else {
            lu_basis_device(c, Z.get(), n, l);
            std::swap(Q, Z);
        }
    }
    T.mark(2);

    spmm_pass(c, M, false, Q.get(), l, bufM.get());       // W = A Q, m x l
    EigWork e;
    e.run(c, bufM.get(), m, l, /*row_sharded=*/true);     // this rank's rows of W
    DBuf<double> MU(size_t(l * k), S), MV(size_t(l * k), S);
    e.factor(c, int(s), int(k), int(k), true, true, MU.get());
    e.factor(c, int(s), int(k), int(k), true, false, MV.get());
    DBuf<double>& Uo = c.slot(4, size_t(std::max<int64_t>(m, 1) * k));
    DBuf<double>& Vo = c.slot(5, size_t(n * k));
    DBuf<double> So(size_t(k), S);
    output_products(c, a, l, k, {bufM.get(), m, MU.get(), Uo.get(), a.U, a.u_ld},
                    {Q.get(), n, MV.get(), Vo.get(), a.V, a.v_ld}, e, int(s), So.get());
    basis_out(c, a, Q.get(), n, l);
    T.mark(3);
    FB_CUDA(cudaStreamSynchronize(S));
    if (st) {
        st->sketch_seconds = T.seconds(0);
        st->power_seconds = T.seconds(1);
        st->finalize_seconds = T.seconds(2);
        st->passes_over_matrix = M.passes.load() - passes0;
    }
}

// ---------------------------------------------------------------------------
// frpca (Alg. 5), randsvd.hpp:224-276. Column-sharded: this rank holds
// columns [offset, offset + n_loc) of A; the m x l products A*X are summed
// across ranks and the final Gram of A^T Q (n-sharded rows) too.
void run_frpca(Ctx& c, DMat& M, const RunArgs& a, frpca_stats* st) {
    const frpca_config& cfg = a.cfg;
    check_common(cfg);
    require(M.grows <= M.gcols, "frpca: requires rows <= cols (use frpcat otherwise)");
    require(cfg.passes >= 2, "frpca: pass count q must be >= 2");
    const int64_t l = cfg.k + cfg.oversample;
    require(l <= M.grows, "frpca: k + oversample must be <= rows");
    require(M.col_shard || c.world == 1, "frpca: needs a column-sharded matrix");
    const int64_t q = cfg.passes, loops = (q - 1) / 2;
    const int64_t m = M.A.rows, n = M.A.cols, k = cfg.k, s = cfg.oversample;
    const uint64_t passes0 = M.passes.load();
    cudaStream_t S = c.stream;

    DBuf<double>& Q = c.slot(0, size_t(m * l));
    DBuf<double>& Y = c.slot(1, size_t(m * l));
    DBuf<double>& bufN = c.slot(2, size_t(std::max<int64_t>(n, 1) * l));

    StageTimer T(S);
    T.mark(0);
    if (q % 2 == 0) {
        // Omega: gcols x l column-major; this rank needs rows [offset, offset+n),
        // row-major
        sketch_rowmajor(c, a, M.gcols, l, M.offset, M.offset + n, bufN);
        spmm_pass_reduced(c, M, false, bufN.get(), l, Y.get());  // A Omega, m x l, summed over ranks
        if (q > 2) {
            lu_basis_device(c, Y.get(), m, l);
            std::swap(Q, Y);
        } else {
            eig_svd_U(c, Y.get(), m, l, Q.get());
        }
    } else {
        sketch_rowmajor(c, a, m, l, 0, m, Q);              // Q = Omega, row-major m x l
    }
    T.mark(1);

    for (int64_t i = 1; i <= loops; ++i) {
        spmm_pass(c, M, true, Q.get(), l, bufN.get());    // A^T Q, n x l
        spmm_pass_reduced(c, M, false, bufN.get(), l, Y.get());  // A (A^T Q), m x l, summed over ranks
        if (i == loops) {
            eig_svd_U(c, Y.get(), m, l, Q.get());
        } else {
            lu_basis_device(c, Y.get(), m, l);
            std::swap(Q, Y);
        }
    }
    T.mark(2);

    spmm_pass(c, M, true, Q.get(), l, bufN.get());        // W = A^T Q, n x l
    EigWork e;
    e.run(c, bufN.get(), n, l, /*row_sharded=*/true);     // this rank's columns of A = rows of W
    DBuf<double> MU(size_t(l * k), S), MV(size_t(l * k), S);
    e.factor(c, int(s), int(k), int(k), true, false, MU.get());   // U = Q * V(:, ind)
    e.factor(c, int(s), int(k), int(k), true, true, MV.get());    // V = f.U(:, ind)
    DBuf<double>& Uo = c.slot(4, size_t(m * k));
    DBuf<double>& Vo = c.slot(5, size_t(std::max<int64_t>(n, 1) * k));
    DBuf<double> So(size_t(k), S);
    output_products(c, a, l, k, {Q.get(), m, MU.get(), Uo.get(), a.U, a.u_ld},
                    {bufN.get(), n, MV.get(), Vo.get(), a.V, a.v_ld}, e, int(s), So.get());
    basis_out(c, a, Q.get(), m, l);
    T.mark(3);
    FB_CUDA(cudaStreamSynchronize(S));
    if (st) {
        st->sketch_seconds = T.seconds(0);
        st->power_seconds = T.seconds(1);
        st->finalize_seconds = T.seconds(2);
        st->passes_over_matrix = M.passes.load() - passes0;
    }
}

// ---------------------------------------------------------------------------
// Baselines: basic_rpca, randsvd.hpp:95-134 (sketch on the
// right) and basic_rpcat, :136-175 (sketch on the left). Q is re-orthonormalised
// by Householder QR after every product; the small SVD of B = Q^T A (resp.
// (A Q)^T) is eig_svd of its transpose reversed (economic_svd_short_fat,
// dense_kernels.hpp:179-190), i.e. the same finalisation as frpca (resp.
// frpcat). 2p + 2 passes. Single GPU.
void run_basic(Ctx& c, DMat& M, const RunArgs& a, frpca_stats* st, bool left) {
    const frpca_config& cfg = a.cfg;
    const char* nm = left ? "basic_rpcat" : "basic_rpca";
    check_common(cfg);
    require(cfg.power >= 0, left ? "basic_rpcat: power p must be >= 0" : "basic_rpca: power p must be >= 0");
    const int64_t l = cfg.k + cfg.oversample;
    require(l <= std::min(M.grows, M.gcols), left ? "basic_rpcat: k + oversample must be <= min(rows, cols)"
                                                  : "basic_rpca: k + oversample must be <= min(rows, cols)");
    require(c.world == 1, "basic_rpca / basic_rpcat: single GPU only");
    (void)nm;
    const int64_t m = M.A.rows, n = M.A.cols, k = cfg.k, s = cfg.oversample, p = cfg.power;
    const uint64_t passes0 = M.passes.load();
    cudaStream_t S = c.stream;
    DBuf<double>& bufM = c.slot(0, size_t(std::max<int64_t>(m, 1) * l));
    DBuf<double>& bufN = c.slot(1, size_t(std::max<int64_t>(n, 1) * l));

    StageTimer T(S);
    T.mark(0);
    if (!left) {
        // Omega n x l column-major -> row-major; Q = orth(A Omega), m x l
        DBuf<double>& om = c.slot(3, 0);
        sketch_into(c, a, n, l, om);
        transpose_device(c, om.get(), l, n, bufN.get());
        spmm_pass(c, M, false, bufN.get(), l, bufM.get());
        orth_device(c, bufM.get(), m, l);
    } else {
        // Omega l x m column-major == Omega^T row-major m x l; Q = orth(A^T Omega^T), n x l
        sketch_into(c, a, l, m, bufM);
        spmm_pass(c, M, true, bufM.get(), l, bufN.get());
        orth_device(c, bufN.get(), n, l);
    }
    T.mark(1);

    for (int64_t i = 0; i < p; ++i) {
        if (!left) {
            spmm_pass(c, M, true, bufM.get(), l, bufN.get());   // G = orth(A^T Q)
            orth_device(c, bufN.get(), n, l);
            spmm_pass(c, M, false, bufN.get(), l, bufM.get());  // Q = orth(A G)
            orth_device(c, bufM.get(), m, l);
        } else {
            spmm_pass(c, M, false, bufN.get(), l, bufM.get());  // G = orth(A Q)
            orth_device(c, bufM.get(), m, l);
            spmm_pass(c, M, true, bufM.get(), l, bufN.get());   // Q = orth(A^T G)
            orth_device(c, bufN.get(), n, l);
        }
    }
    T.mark(2);

    DBuf<double>& Uo = c.slot(4, size_t(std::max<int64_t>(m, 1) * k));
    DBuf<double>& Vo = c.slot(5, size_t(std::max<int64_t>(n, 1) * k));
    DBuf<double> So(size_t(k), S);
    DBuf<double> MU(size_t(l * k), S), MV(size_t(l * k), S);
    EigWork e;
    if (!left) {
        DBuf<double>& W = c.slot(2, size_t(std::max<int64_t>(n, 1) * l));
        spmm_pass(c, M, true, bufM.get(), l, W.get());          // W = A^T Q, n x l
        e.run(c, W.get(), n, l, false);
        e.factor(c, int(s), int(k), int(k), true, false, MU.get());  // U = Q V(:, ind)
        e.factor(c, int(s), int(k), int(k), true, true, MV.get());   // V = W V(:, ind) / S
        gemm_device(c, bufM.get(), m, l, MU.get(), k, Uo.get(), std::max<int64_t>(m, 1), true);
        gemm_device(c, W.get(), n, l, MV.get(), k, Vo.get(), std::max<int64_t>(n, 1), true);
        basis_out(c, a, bufM.get(), m, l);
    } else {
        DBuf<double>& W = c.slot(2, size_t(std::max<int64_t>(m, 1) * l));
        spmm_pass(c, M, false, bufN.get(), l, W.get());         // W = A Q, m x l
        e.run(c, W.get(), m, l, false);
        e.factor(c, int(s), int(k), int(k), true, true, MU.get());   // U = W V(:, ind) / S
        e.factor(c, int(s), int(k), int(k), true, false, MV.get());  // V = Q V(:, ind)
        gemm_device(c, W.get(), m, l, MU.get(), k, Uo.get(), std::max<int64_t>(m, 1), true);
        gemm_device(c, bufN.get(), n, l, MV.get(), k, Vo.get(), std::max<int64_t>(n, 1), true);
        basis_out(c, a, bufN.get(), n, l);
    }
    e.singular_values(c, int(s), int(k), true, So.get());
    copy_out(c, a, a.U, Uo.get(), m * k);
    copy_out(c, a, a.V, Vo.get(), n * k);
    copy_out(c, a, a.S, So.get(), k);
    T.mark(3);
    FB_CUDA(cudaStreamSynchronize(S));
    if (st) {
        st->sketch_seconds = T.seconds(0);
        st->power_seconds = T.seconds(1);
        st->finalize_seconds = T.seconds(2);
        st->passes_over_matrix = M.passes.load() - passes0;
    }
}

// spmm_pass followed by the sum of Y over the ranks, overlapped chunk by chunk
// (the exchange steps of randsvd.hpp:255-258 / :307-310 when sharded)
void spmm_pass_reduced(Ctx& c, DMat& M, bool transpose, const double* X, int64_t ncols, double* Y) {
    if (transpose) spmm_t_device_reduced(c, M.At, X, ncols, Y, "spmm_AtY");
    else spmm_device_reduced(c, M.A, X, ncols, Y, "spmm_AX");
    M.passes.fetch_add(1, std::memory_order_relaxed);  // recordPass, sparse_matrix.hpp:119-122
}

void spmm_pass(Ctx& c, DMat& M, bool transpose, const double* X, int64_t ncols, double* Y) {
    if (transpose) spmm_t_device(c, M.At, X, ncols, Y, "spmm_AtY");
    else spmm_device(c, M.A, X, ncols, ncols, Y, ncols, "spmm_AX");
    M.passes.fetch_add(1, std::memory_order_relaxed);  // recordPass, sparse_matrix.hpp:119-122
}

uint64_t mix_seed(uint64_t seed, uint64_t tag) {  // types.hpp:52-57
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// Deferred errors (Ctx::dflag): first failure code of the running call.
int* err_flag(Ctx& c) {
    if (!c.dflag.get()) {
        c.dflag.alloc(1, c.stream);
        FB_CUDA(cudaMemsetAsync(c.dflag.get(), 0, sizeof(int), c.stream));
    }
    return c.dflag.get();
}

void err_reset(Ctx& c) { FB_CUDA(cudaMemsetAsync(err_flag(c), 0, sizeof(int), c.stream)); }

void err_check(Ctx& c) {
    int h = 0;
    FB_CUDA(cudaMemcpyAsync(&h, err_flag(c), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    FB_CUDA(cudaStreamSynchronize(c.stream));
    if (h == 0) return;
    FB_CUDA(cudaMemsetAsync(c.dflag.get(), 0, sizeof(int), c.stream));
    if (h == kErrLuPivot) throw NumericalError("lu_basis: zero pivot, input is rank-deficient");  // :81
    if (h == kErrEigRank) throw NumericalError("eig_svd: input does not have full numerical column rank");
    if (h == kErrEigFail) throw NumericalError("eig_svd: eigendecomposition failed to converge");  // :160-161
    if (h == kErrOrthRank) throw NumericalError("orth: numerically rank-deficient input");  // :43-44
    if (h == kErrEigNoConv) {
        const char* mode = std::getenv("FRPCA_EIG");
        if (mode && std::strcmp(mode, "strict") == 0)
            throw CudaError("syev_small: did not converge (FRPCA_EIG=strict)");
        throw RetryCall(kErrEigNoConv);
    }
    if (h == kErrOmegaShort) throw RetryCall(kErrOmegaShort);
    throw CudaError("unknown deferred error code " + std::to_string(h));
}

void run_algorithm(Ctx& c, DMat& M, const RunArgs& a, frpca_stats* st, int algo) {
    const uint64_t passes0 = M.passes.load();
    RunArgs cur = a;
    with_checks(c, [&] {
        M.passes.store(passes0);  // a re-run counts its passes once
        const RunArgs now = cur;
        cur.pre = nullptr;        // the pre-generated Omega is consumed by the first attempt only
        if (algo == FRPCA_ALGO_FRPCA) run_frpca(c, M, now, st);
        else if (algo == FRPCA_ALGO_FRPCAT) run_frpcat(c, M, now, st);
        else run_basic(c, M, now, st, algo == FRPCA_ALGO_BASIC_RPCAT);
    });
}

}  // namespace fb
