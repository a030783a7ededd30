// Checks fb's warp_best against a sequential cand_merge (diagnostic).
#include <cstdio>
#include <cstdint>
#include <climits>
#include <cstdlib>
struct Cand { double v; int32_t pos, row; };
__device__ __forceinline__ bool better(double v, int32_t p, double bv, int32_t bp) { return v > bv || (v == bv && p < bp); }
__device__ __forceinline__ void cand_merge(Cand& c, const Cand& o) { if (better(o.v, o.pos, c.v, c.pos)) c = o; }
__device__ __forceinline__ Cand warp_best(const Cand& c) {
    const unsigned long long key = c.v >= 0.0 ? (unsigned long long)__double_as_longlong(c.v) + 1ull : 0ull;
    unsigned long long kmax = key;
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmax = x > kmax ? x : kmax;
    }
    const int pmin = __reduce_min_sync(0xffffffffu, key == kmax ? int(c.pos) : INT32_MAX);
    const unsigned who = __ballot_sync(0xffffffffu, key == kmax && c.pos == pmin);
    const int src = __ffs(int(who)) - 1;
    Cand r;
    r.v = __shfl_sync(0xffffffffu, c.v, src);
    r.pos = pmin;
    r.row = __shfl_sync(0xffffffffu, c.row, src);
    return r;
}
template <int kT>
__device__ Cand block_best(Cand c, Cand* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    c = warp_best(c);
    if (lane == 0) sh[warp] = c;
    __syncthreads();
    const Cand r = warp_best(lane < int(blockDim.x >> 5) ? sh[lane] : Cand{-1.0, INT32_MAX, -1});
    __syncthreads();
    return r;
}
__global__ void kb(const Cand* in, Cand* out, Cand* ref) {
    __shared__ Cand sh[16];
    const int b = blockIdx.x;
    Cand c = in[b * 512 + threadIdx.x];
    Cand r = block_best<512>(c, sh);
    if (r.v != out[0].v && false) out[0] = r;
    // every thread must hold the same result
    Cand s{-1.0, INT32_MAX, -1};
    for (int i = 0; i < 512; ++i) cand_merge(s, in[b * 512 + i]);
    if (r.v != s.v || r.pos != s.pos || r.row != s.row) { out[b] = r; ref[b] = s; }
}
__global__ void k(const Cand* in, Cand* out, Cand* ref, int n) {
    const int w = blockIdx.x, lane = threadIdx.x;
    Cand c = in[w * 32 + lane];
    Cand r = warp_best(c);
    if (lane == 0) out[w] = r;
    if (lane == 0) { Cand s{-1.0, INT32_MAX, -1}; for (int i = 0; i < 32; ++i) cand_merge(s, in[w * 32 + i]); ref[w] = s; }
}
int main() {
    const int W = 4096;
    Cand* h = (Cand*)malloc(sizeof(Cand) * W * 32);
    srand(1);
    for (int i = 0; i < W * 32; ++i) {
        int kind = rand() % 4;
        h[i].v = kind == 0 ? -1.0 : (kind == 1 ? (rand() % 4) * 0.5 : rand() / double(RAND_MAX));
        h[i].pos = kind == 0 ? INT32_MAX : rand() % 1000;
        h[i].row = i;
    }
    Cand *d, *o, *r;
    cudaMalloc(&d, sizeof(Cand) * W * 32); cudaMalloc(&o, sizeof(Cand) * W); cudaMalloc(&r, sizeof(Cand) * W);
    cudaMemcpy(d, h, sizeof(Cand) * W * 32, cudaMemcpyHostToDevice);
    k<<<W, 32>>>(d, o, r, W);
    Cand* ho = (Cand*)malloc(sizeof(Cand) * W); Cand* hr = (Cand*)malloc(sizeof(Cand) * W);
    cudaMemcpy(ho, o, sizeof(Cand) * W, cudaMemcpyDeviceToHost); cudaMemcpy(hr, r, sizeof(Cand) * W, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int w = 0; w < W; ++w)
        if (ho[w].v != hr[w].v || ho[w].pos != hr[w].pos || ho[w].row != hr[w].row) {
            if (bad < 5) printf("warp %d: got (%g,%d,%d) want (%g,%d,%d)\n", w, ho[w].v, ho[w].pos, ho[w].row, hr[w].v, hr[w].pos, hr[w].row);
            ++bad;
        }
    printf("mismatches %d of %d (%s)\n", bad, W, cudaGetErrorString(cudaGetLastError()));
    // block-level: W*32/512 blocks of 512
    const int B = W * 32 / 512;
    cudaMemset(o, 0, sizeof(Cand) * W); cudaMemset(r, 0, sizeof(Cand) * W);
    kb<<<B, 512>>>(d, o, r);
    cudaMemcpy(ho, o, sizeof(Cand) * W, cudaMemcpyDeviceToHost); cudaMemcpy(hr, r, sizeof(Cand) * W, cudaMemcpyDeviceToHost);
    bad = 0;
    for (int b = 0; b < B; ++b) if (ho[b].pos != 0 || hr[b].pos != 0) { if (bad < 5) printf("block %d: got (%g,%d,%d) want (%g,%d,%d)\n", b, ho[b].v, ho[b].pos, ho[b].row, hr[b].v, hr[b].pos, hr[b].row); ++bad; }
    printf("block mismatches %d of %d (%s)\n", bad, B, cudaGetErrorString(cudaDeviceSynchronize()));
}
