// L2 read bandwidth on this B200 (diagnostic, for the SpMM roofline):
//  (1) streaming reads of an L2-resident buffer (double2 per lane),
//  (2) warp gathers of random 1600-byte rows from an L2-resident table (the
//      SpMM access: one 200-double row per nonzero).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
__global__ void k_stream(const double2* __restrict__ x, size_t n2, int reps, double* out) {
    double acc = 0.0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x) {
            const double2 v = __ldg(x + i);
            acc += v.x + v.y;
        }
    if (acc == 1.2345) out[0] = acc;
}
__global__ void k_gather(const double* __restrict__ tab, const int* __restrict__ ids, int nids, int ld, double* out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    double2 acc[4] = {};
    for (int i = warp * 4; i < nids; i += nw * 4) {
        double2 v[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double* row = tab + size_t(ids[i + u]) * ld + lane * 2;
#pragma unroll
            for (int c = 0; c < 4; ++c) v[u][c] = (lane * 2 + c * 64 < ld) ? __ldg(reinterpret_cast<const double2*>(row + c * 64)) : double2{0, 0};
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < 4; ++c) { acc[c].x += v[u][c].x; acc[c].y += v[u][c].y; }
    }
    double s = 0;
    for (int c = 0; c < 4; ++c) s += acc[c].x + acc[c].y;
    if (s == 1.2345) out[0] = s;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (size_t mb : {32, 64, 96}) {
        const size_t n2 = mb * (1 << 20) / 16;
        double2* x;
        cudaMalloc(&x, n2 * 16);
        cudaMemset(x, 0, n2 * 16);
        const int reps = 20;
        k_stream<<<sms * 8, 256>>>(x, n2, 2, out);
        cudaEventRecord(a);
        k_stream<<<sms * 8, 256>>>(x, n2, reps, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("stream %zu MB: %.1f GB/s\n", mb, double(n2) * 16 * reps / (ms * 1e-3) / 1e9);
        cudaFree(x);
    }
    for (size_t mb : {32, 64, 96, 160}) {
        const int ld = 200;
        const size_t rows = mb * (1 << 20) / (8 * ld);
        double* tab;
        cudaMalloc(&tab, rows * ld * 8);
        cudaMemset(tab, 0, rows * ld * 8);
        const int nids = 8 << 20;
        std::vector<int> h(nids);
        std::mt19937 g(1);
        for (auto& v : h) v = int(g() % rows);
        int* ids;
        cudaMalloc(&ids, nids * 4);
        cudaMemcpy(ids, h.data(), nids * 4, cudaMemcpyHostToDevice);
        k_gather<<<sms * 4, 256>>>(tab, ids, nids, ld, out);
        cudaEventRecord(a);
        k_gather<<<sms * 4, 256>>>(tab, ids, nids, ld, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("gather 1600-B rows from %zu MB: %.1f GB/s (%s)\n", mb, double(nids) * ld * 8 / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
        cudaFree(tab);
        cudaFree(ids);
    }
}
