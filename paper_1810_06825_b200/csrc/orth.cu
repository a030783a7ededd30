// orth (dense_kernels.hpp:30-48): orthonormal basis of range(M) for tall M by
// Householder QR, with the reference's rank check (|diag R| <= m eps max|diag R|
// is an error). Used by the baseline algorithms basic_rpca / basic_rpcat
// (SURVEY §8 row f4), off the fast path: cuSOLVER geqrf + orgqr on the
// column-major copy of the row-major panel (the same Householder convention as
// Eigen::HouseholderQR: beta = -sign(alpha) ||x||).
#include <cfloat>
#include <cmath>

#include "internal.cuh"

namespace fb {

void orth_device(Ctx& c, double* W, int64_t r, int64_t l) {
    require(r >= l && l >= 1, "orth: input must be tall (rows >= cols >= 1)");
    require(r < (int64_t(1) << 31), "orth: rows must be < 2^31");
    Prof prof(c, "orth", 32.0 * r * l, 4.0 * double(r) * l * l);
    cudaStream_t s = c.stream;
    const int m = int(r), n = int(l);
    DBuf<double> A(size_t(r * l), s), tau(size_t(l), s);
    DBuf<int> info(1, s);
    transpose_device(c, W, r, l, A.get());  // row-major r x l -> column-major r x l
    int lw1 = 0, lw2 = 0;
    if (cusolverDnDgeqrf_bufferSize(c.solver, m, n, A.get(), m, &lw1) != CUSOLVER_STATUS_SUCCESS ||
        cusolverDnDorgqr_bufferSize(c.solver, m, n, n, A.get(), m, tau.get(), &lw2) != CUSOLVER_STATUS_SUCCESS)
        throw CudaError("orth: cuSOLVER buffer size query failed");
    const int lwork = std::max(std::max(lw1, lw2), 1);
    DBuf<double> work(size_t(lwork), s);
    if (cusolverDnDgeqrf(c.solver, m, n, A.get(), m, tau.get(), work.get(), lwork, info.get()) !=
        CUSOLVER_STATUS_SUCCESS)
        throw CudaError("orth: cusolverDnDgeqrf failed");
    // rank check on the diagonal of R (:40-44)
    std::vector<double> d(static_cast<size_t>(l));
    FB_CUDA(cudaMemcpy2DAsync(d.data(), sizeof(double), A.get(), sizeof(double) * (size_t(r) + 1), sizeof(double),
                              size_t(l), cudaMemcpyDeviceToHost, s));
    FB_CUDA(cudaStreamSynchronize(s));
    double maxd = 0.0;
    for (double x : d) maxd = std::max(maxd, std::fabs(x));
    const double tol = double(r) * DBL_EPSILON * maxd;
    bool bad = maxd == 0.0;
    for (double x : d) bad = bad || std::fabs(x) <= tol;
    if (bad) throw NumericalError("orth: numerically rank-deficient input");
    if (cusolverDnDorgqr(c.solver, m, n, n, A.get(), m, tau.get(), work.get(), lwork, info.get()) !=
        CUSOLVER_STATUS_SUCCESS)
        throw CudaError("orth: cusolverDnDorgqr failed");
    transpose_device(c, A.get(), l, r, W);  // column-major r x l -> row-major
}

}  // namespace fb
