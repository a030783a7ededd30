// Probe: cost of one grid-wide barrier on B200 (148 CTAs x 256 threads):
// cooperative_groups grid.sync() vs a hand-rolled generation barrier, each
// with and without a per-step "every CTA reads all CTAs' candidates" round trip.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void my_barrier(unsigned* count, volatile unsigned* gen, unsigned nblk, unsigned& g) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned my = g + 1;
        __threadfence();
        if (atomicAdd(count, 1u) == nblk - 1) {
            *count = 0;
            __threadfence();
            atomicExch((unsigned*)gen, my);
        } else {
            while (*gen < my) { }
        }
        __threadfence();
    }
    __syncthreads();
    ++g;
}

__global__ void k_cg(int iters, double* cand, int read) {
    cg::grid_group grid = cg::this_grid();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) cand[blockIdx.x] = i + acc;
        grid.sync();
        if (read && threadIdx.x < gridDim.x) acc += ((volatile double*)cand)[threadIdx.x];
    }
    if (acc == -1) cand[0] = acc;
}

__global__ void k_my(int iters, double* cand, int read, unsigned* count, unsigned* gen) {
    unsigned g = 0;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) cand[blockIdx.x] = i + acc;
        my_barrier(count, gen, gridDim.x, g);
        if (read && threadIdx.x < gridDim.x) acc += ((volatile double*)cand)[threadIdx.x];
    }
    if (acc == -1) cand[0] = acc;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* cand; unsigned *count, *gen;
    cudaMalloc(&cand, 8 * 4096); cudaMalloc(&count, 4); cudaMalloc(&gen, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 2000;
    for (int read = 0; read < 2; ++read) {
        for (int kind = 0; kind < 2; ++kind) {
            cudaMemset(count, 0, 4); cudaMemset(gen, 0, 4);
            void* args_cg[] = {(void*)&iters, &cand, &read};
            void* args_my[] = {(void*)&iters, &cand, &read, &count, &gen};
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(count, 0, 4); cudaMemset(gen, 0, 4);
                cudaEventRecord(a);
                if (kind == 0) cudaLaunchCooperativeKernel((void*)k_cg, sms, 256, args_cg, 0, 0);
                else cudaLaunchCooperativeKernel((void*)k_my, sms, 256, args_my, 0, 0);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep == 1) printf("%s read=%d: %.3f us per step\n", kind ? "custom" : "cg", read, 1000.0 * ms / iters);
            }
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
