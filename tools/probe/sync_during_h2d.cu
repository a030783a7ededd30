// Latency of a tiny kernel + stream synchronisation on one stream while a
// large pinned host->device copy runs on another (diagnostic for the
// pipelined upload's host read-backs). Variants: plain kernel; kernel that
// writes a word into mapped pinned host memory; cudaMemcpyAsync D2H of 8 bytes.
#include <cstdio>
#include <chrono>
#include <vector>
#include <algorithm>
__global__ void k_tiny(int* d) { if (threadIdx.x == 0) d[0] += 1; }
__global__ void k_put(const int* d, volatile int* h) { if (threadIdx.x == 0) h[0] = d[0]; }
int main() {
    const size_t big = size_t(3200) << 20;
    char *hbig, *dbig; cudaHostAlloc(&hbig, big, 0); cudaMalloc(&dbig, big);
    int* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
    int* hm; cudaHostAlloc(&hm, 64, cudaHostAllocMapped); int* dm; cudaHostGetDevicePointer((void**)&dm, hm, 0);
    int hv = 0;
    cudaStream_t sa, sb; cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
    for (int variant = 0; variant < 3; ++variant) {
      for (int rep = 0; rep < 3; ++rep) {
        std::vector<double> lat;
        cudaDeviceSynchronize();
        // 8 chunks like the upload
        for (int c = 0; c < 8; ++c) cudaMemcpyAsync(dbig + c * (big / 8), hbig + c * (big / 8), big / 8, cudaMemcpyHostToDevice, sa);
        cudaEvent_t done; cudaEventCreate(&done); cudaEventRecord(done, sa);
        while (cudaEventQuery(done) == cudaErrorNotReady) {
            auto t0 = std::chrono::steady_clock::now();
            k_tiny<<<1, 32, 0, sb>>>(d);
            if (variant == 1) k_put<<<1, 32, 0, sb>>>(d, dm);
            if (variant == 2) cudaMemcpyAsync(&hv, d, 4, cudaMemcpyDeviceToHost, sb);
            cudaStreamSynchronize(sb);
            lat.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        }
        std::sort(lat.begin(), lat.end());
        printf("variant %d rep %d: n=%zu median %.3f ms p99 %.3f max %.3f\n", variant, rep, lat.size(),
               lat[lat.size() / 2], lat[size_t(lat.size() * 0.99)], lat.back());
        cudaEventDestroy(done);
      }
    }
    return 0;
}
