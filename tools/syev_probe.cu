// Probe: cuSOLVER symmetric eigensolvers on an l x l Gram matrix (l = 200):
// Dsyevd vs XsyevBatched (batch 1) vs Xsyevd; time (events, after warm-up)
// and residual max|B V - V D| / ||B||.
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>

#define CK(x) do { auto _e = (x); if ((int)_e) { printf("fail %s line %d: %d\n", #x, __LINE__, (int)_e); exit(1); } } while (0)

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 200;
    std::mt19937_64 g(1);
    std::normal_distribution<double> N(0, 1);
    const int r = 4 * n;
    std::vector<double> W(size_t(r) * n), B(size_t(n) * n, 0.0);
    for (auto& x : W) x = N(g);
    for (int j = 0; j < n; ++j) for (int i = 0; i < r; ++i) W[size_t(j) * r + i] *= std::pow(0.93, j);
    for (int a = 0; a < n; ++a) for (int b = 0; b < n; ++b) { double s = 0; for (int i = 0; i < r; ++i) s += W[size_t(a) * r + i] * W[size_t(b) * r + i]; B[size_t(a) * n + b] = s; }
    cusolverDnHandle_t h; CK(cusolverDnCreate(&h));
    cudaStream_t st; cudaStreamCreate(&st); CK(cusolverDnSetStream(h, st));
    cusolverDnParams_t prm; CK(cusolverDnCreateParams(&prm));
    double *dB, *dA, *dD; int* info;
    cudaMalloc(&dB, sizeof(double) * n * n); cudaMalloc(&dA, sizeof(double) * n * n); cudaMalloc(&dD, sizeof(double) * n); cudaMalloc(&info, sizeof(int));
    cudaMemcpy(dB, B.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto resid = [&](const char* name, float ms) {
        std::vector<double> V(size_t(n) * n), D(n);
        cudaMemcpy(V.data(), dA, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
        cudaMemcpy(D.data(), dD, sizeof(double) * n, cudaMemcpyDeviceToHost);
        double mx = 0, nb = 0;
        for (auto x : B) nb = std::max(nb, std::fabs(x));
        for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) { double s = 0; for (int k = 0; k < n; ++k) s += B[size_t(k) * n + i] * V[size_t(j) * n + k]; mx = std::max(mx, std::fabs(s - D[j] * V[size_t(j) * n + i])); }
        printf("%-16s n=%d %.3f ms  resid %.2e  dmin %.3e dmax %.3e\n", name, n, ms, mx / nb, D[0], D[n - 1]);
    };
    // Dsyevd
    int lw = 0; CK(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dD, &lw));
    double* wk; cudaMalloc(&wk, sizeof(double) * lw);
    for (int it = 0; it < 4; ++it) {
        cudaMemcpyAsync(dA, dB, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st);
        cudaEventRecord(e0, st);
        CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dD, wk, lw, info));
        cudaEventRecord(e1, st); cudaStreamSynchronize(st);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (it == 3) resid("Dsyevd", ms);
    }
    // XsyevBatched
    size_t wd = 0, wh = 0;
    CK(cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dD, CUDA_R_64F, &wd, &wh, 1));
    void* bd; cudaMalloc(&bd, wd + 8); std::vector<char> bh(wh + 8);
    for (int it = 0; it < 4; ++it) {
        cudaMemcpyAsync(dA, dB, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st);
        cudaEventRecord(e0, st);
        CK(cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dD, CUDA_R_64F, bd, wd, bh.data(), wh, info, 1));
        cudaEventRecord(e1, st); cudaStreamSynchronize(st);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (it == 3) resid("XsyevBatched", ms);
    }
    // Xsyevd
    CK(cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dD, CUDA_R_64F, &wd, &wh));
    void* bd2; cudaMalloc(&bd2, wd + 8); std::vector<char> bh2(wh + 8);
    for (int it = 0; it < 4; ++it) {
        cudaMemcpyAsync(dA, dB, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st);
        cudaEventRecord(e0, st);
        CK(cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dD, CUDA_R_64F, bd2, wd, bh2.data(), wh, info));
        cudaEventRecord(e1, st); cudaStreamSynchronize(st);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (it == 3) resid("Xsyevd", ms);
    }
    return 0;
}
