// K5: the l x l symmetric eigenproblem of eig_svd (dense_kernels.hpp:159-161,
// Eigen SelfAdjointEigenSolver). The north_star allows cuSOLVER here: it is
// O(l^3) on a 200 x 200 matrix, off the bandwidth-critical path.
#include "internal.cuh"

namespace fb {

void syevd_device(Ctx& c, double* B, int64_t n, double* d_D, std::vector<double>& h_D) {
    Prof prof(c, "syevd", 8.0 * n * n * 2, 4.0 / 3.0 * n * n * n);
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
    h_D.resize(size_t(n));
    FB_CUDA(cudaMemcpyAsync(&h_info, info.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    FB_CUDA(cudaMemcpyAsync(h_D.data(), d_D, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
    FB_CUDA(cudaStreamSynchronize(c.stream));
    if (h_info != 0) throw NumericalError("eig_svd: eigendecomposition failed to converge");
}

}  // namespace fb
