// K5: the l x l symmetric eigenproblem of eig_svd (dense_kernels.hpp:159-161,
// Eigen SelfAdjointEigenSolver): the library's own l <= 232 solver in syev.cu,
// cuSOLVER syevd above that size or when the small solver reports failure.
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace fb {

bool syev_small(Ctx& c, double* B, int64_t n, double* d_D);

void syevd_device(Ctx& c, double* B, int64_t n, double* d_D, bool final_step) {
    Prof prof(c, "syevd", 8.0 * n * n * 2, 4.0 / 3.0 * n * n * n);
    // The small solver (syev.cu) by default: faster than syevd at l = 200
    // (DESIGN.md §4); its non-convergence is reported by err_check, which makes
    // the caller re-run the call with cuSOLVER (or fail, FRPCA_EIG=strict).
    // FRPCA_EIG=cusolver forces syevd; FRPCA_EIG_LOOP / FRPCA_EIG_FINAL
    // (cusolver | small) choose per role: the power iteration's eig_svd or the
    // final one (A/B of accuracy against the arbiter).
    const char* mode = std::getenv(final_step ? "FRPCA_EIG_FINAL" : "FRPCA_EIG_LOOP");
    if (!mode || !*mode) mode = std::getenv("FRPCA_EIG");
    if (!(mode && std::strcmp(mode, "cusolver") == 0)) {
        if (syev_small(c, B, n, d_D)) return;
    }
    int lwork = 0;
    if (cusolverDnDsyevd_bufferSize(c.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                    int(n), B, int(n), d_D, &lwork) != CUSOLVER_STATUS_SUCCESS)
        throw CudaError("cusolverDnDsyevd_bufferSize failed");
    DBuf<double> work(size_t(std::max(lwork, 1)), c.stream);
    DBuf<int> info(1, c.stream);
    if (cusolverDnDsyevd(c.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, int(n), B,
                         int(n), d_D, work.get(), lwork, info.get()) != CUSOLVER_STATUS_SUCCESS)
        throw CudaError("cusolverDnDsyevd failed");
    int h_info = 0;
    FB_CUDA(cudaMemcpyAsync(&h_info, info.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    FB_CUDA(cudaStreamSynchronize(c.stream));
    if (h_info != 0) throw NumericalError("eig_svd: eigendecomposition failed to converge");
}

}  // namespace fb
