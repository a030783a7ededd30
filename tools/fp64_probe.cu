// Measures the fp64 ceilings that bound the dense stages on this B200:
// DFMA (SIMT fp64 pipe), DMMA.8x8x4 (fp64 tensor pipe), cusolver syevd / syevj
// on the l x l eigenproblem. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   tools/fp64_probe.cu -lcusolver -lcublas -o tools/_build/fp64_probe
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cstdio>
#include <vector>
#include <random>

__global__ void dfma_loop(double* out, int iters) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 1.0000001, c = 1e-9;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
    double d[8][2];
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 20000;
    for (int blocksPerSm : {4, 8}) {
        const int grid = sms * blocksPerSm, threads = 256;
        dfma_loop<<<grid, threads>>>(out, 100);
        cudaEventRecord(a);
        dfma_loop<<<grid, threads>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * 8 * iters * double(grid) * threads;
        printf("DFMA  blocks/SM=%d: %.2f TFLOP/s\n", blocksPerSm, fl / (ms * 1e-3) / 1e12);
        dmma_loop<<<grid, threads>>>(out, 100);
        cudaEventRecord(a);
        dmma_loop<<<grid, threads>>>(out, iters / 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        fl = 2.0 * 256 * 8 * (iters / 4) * double(grid) * (threads / 32);
        printf("DMMA  blocks/SM=%d: %.2f TFLOP/s\n", blocksPerSm, fl / (ms * 1e-3) / 1e12);
    }
    // l x l symmetric eigensolvers
    cusolverDnHandle_t h; cusolverDnCreate(&h);
    for (int n : {40, 150, 200}) {
        std::vector<double> B(size_t(n) * n);
        std::mt19937_64 g(1); std::normal_distribution<double> nd;
        std::vector<double> W(size_t(n) * 3 * n);
        for (auto& x : W) x = nd(g);
        for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < 3 * n; ++k) s += W[i + k * size_t(n)] * W[j + k * size_t(n)]; B[i + j * size_t(n)] = s; }
        double *dB, *dA, *dW, *work; int* info;
        cudaMalloc(&dB, 8 * n * n); cudaMalloc(&dA, 8 * n * n); cudaMalloc(&dW, 8 * n); cudaMalloc(&info, 4);
        cudaMemcpy(dB, B.data(), 8 * n * n, cudaMemcpyHostToDevice);
        int lw; cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw);
        cudaMalloc(&work, 8 * size_t(lw));
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemcpy(dA, dB, 8 * n * n, cudaMemcpyDeviceToDevice);
            cudaEventRecord(a);
            cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lw, info);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("syevd n=%d: %.3f ms\n", n, ms);
        }
        syevjInfo_t params; cusolverDnCreateSyevjInfo(&params);
        cusolverDnXsyevjSetTolerance(params, 1e-15);
        int lwj; cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lwj, params);
        double* workj; cudaMalloc(&workj, 8 * size_t(lwj));
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemcpy(dA, dB, 8 * n * n, cudaMemcpyDeviceToDevice);
            cudaEventRecord(a);
            cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, workj, lwj, info, params);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("syevj n=%d: %.3f ms\n", n, ms);
        }
    }
    return 0;
}
