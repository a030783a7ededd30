// K9: the sketch Omega on the device, bit-compatible with the reference's
// gaussian_matrix (dense_kernels.hpp:19-28): std::mt19937_64(seed) feeding
// libstdc++'s std::normal_distribution<double> (Marsaglia polar method,
// random.tcc: each attempt draws two generate_canonical<double> uniforms from
// one 64-bit output each, rejects r2 > 1 or r2 == 0, and an accepted pair
// yields y*mult then the cached x*mult), in stream (column-major fill) order.
//
// Parallelisation: the raw 64-bit stream is cut into K segments of J words
// (J = 156 * 2^e: even, so every segment starts on an attempt boundary, and a
// whole number of 156-word generation steps). Segment k's engine state
// T^(kJ) s0 is reached by MT19937-64 jump-ahead (Horner over the jump
// polynomials of rng_poly.cpp, 32 coefficients per step using the 32 shifted
// windows of the base sequence). Each segment then (1) counts its accepted
// pairs, an exclusive scan gives every segment its output offset, and (2)
// regenerates the segment and writes its normals. The arithmetic of every
// accepted pair is the host's, operation for operation, in IEEE round-to-
// nearest without contraction; only log() may differ from glibc's in the last
// ulp, which changes no accept/reject decision (that uses r2 alone).
#include <cub/cub.cuh>

#include <cmath>
#include <map>
#include <mutex>

#include "internal.cuh"

namespace fb {

int mt64_jump_polys(int log2_steps, int n, std::vector<uint32_t>& out, int& groups);
void mt64_seed_state(uint64_t seed, uint64_t* state312);

namespace {

constexpr int NN = 312;
constexpr int MM = 156;
constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MA = 0xB5026F5AA96619E9ULL;
constexpr int kMaxJumps = 16;

__device__ __forceinline__ uint64_t mt_next(uint64_t a, uint64_t b, uint64_t c) {
    const uint64_t y = (a & UM) | (b & LM);
    return c ^ (y >> 1) ^ ((y & 1ull) ? MA : 0ull);
}

__device__ __forceinline__ uint64_t temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

// generate_canonical<double, 53>(mt19937_64): one draw, (double)w / 2^64,
// clamped below 1 (random.tcc generate_canonical).
__device__ __forceinline__ double canonical(uint64_t w) {
    double u = __dmul_rn(__ull2double_rn(w), 0x1.0p-64);
    if (u >= 1.0) u = 0x1.fffffffffffffp-1;
    return u;
}

__device__ __forceinline__ int wrap(int i) { return i >= NN ? i - NN : i; }

// Segment start states: state_k = T^(k J) s0, applying the jump for every set
// bit a of k with polynomial x^(J 2^a) mod P.
__global__ void __launch_bounds__(320)
k_jump(const uint64_t* __restrict__ s0, const uint32_t* __restrict__ polys, int groups,
       uint64_t* __restrict__ states) {
    __shared__ uint64_t base[NN + 32];
    __shared__ uint64_t R[NN];
    const int tid = threadIdx.x;
    const unsigned k = blockIdx.x;
    if (tid < NN) base[tid] = s0[tid];
    __syncthreads();
    for (int a = 0; a < kMaxJumps; ++a) {
        if (!((k >> a) & 1u)) continue;
        // the 31 words after the base window give the shifted windows T^b base
        if (tid < 32) base[NN + tid] = mt_next(base[tid], base[tid + 1], base[tid + MM]);
        if (tid < NN) R[tid] = 0;
        int h = 0;
        __syncthreads();
        const uint32_t* co = polys + size_t(a) * groups;
        for (int g = groups - 1; g >= 0; --g) {
            // r <- T^32 r
            uint64_t nw = 0;
            if (tid < 32) {
                const int i0 = wrap(h + tid);
                nw = mt_next(R[i0], R[wrap(i0 + 1)], R[wrap(i0 + MM)]);
            }
            __syncthreads();
            if (tid < 32) R[wrap(h + tid)] = nw;
            h = wrap(h + 32);
            __syncthreads();
            // r <- r + sum_b c_(32g+b) T^b base
            uint32_t c = co[g];
            if (tid < NN && c) {
                uint64_t x = 0;
                while (c) {
                    const int b = __ffs(c) - 1;
                    x ^= base[tid + b];
                    c &= c - 1;
                }
                R[wrap(h + tid)] ^= x;
            }
            __syncthreads();
        }
        uint64_t v = 0;
        if (tid < NN) v = R[wrap(h + tid)];
        __syncthreads();
        if (tid < NN) base[tid] = v;
        __syncthreads();
    }
    if (tid < NN) states[size_t(k) * NN + tid] = base[tid];
}

// MODE 0: count accepted pairs per segment. MODE 1: write the normals.
template <int MODE>
__global__ void __launch_bounds__(160)
k_polar(const uint64_t* __restrict__ states, int64_t steps, const int64_t* __restrict__ pair_off,
        int64_t* __restrict__ counts, double* __restrict__ out, int64_t count) {
    __shared__ uint64_t X[NN];
    __shared__ uint64_t O[MM];
    __shared__ int wsum[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t k = blockIdx.x;
    int64_t base_pair = 0;
    if (MODE == 1) {
        base_pair = pair_off[k];
        if (2 * base_pair >= count) return;
    }
    for (int i = tid; i < NN; i += blockDim.x) X[i] = states[k * NN + i];
    __syncthreads();
    int h = 0;
    int64_t acc = 0;
    for (int64_t st = 0; st < steps; ++st) {
        uint64_t nw = 0;
        if (tid < MM) {
            const int i0 = wrap(h + tid);
            nw = mt_next(X[i0], X[wrap(i0 + 1)], X[wrap(i0 + MM)]);
        }
        __syncthreads();
        if (tid < MM) {
            X[wrap(h + tid)] = nw;
            O[tid] = temper(nw);
        }
        h = wrap(h + MM);
        __syncthreads();
        bool ok = false;
        double x = 0, y = 0, r2 = 0;
        if (tid < MM / 2) {
            x = __dsub_rn(__dmul_rn(2.0, canonical(O[2 * tid])), 1.0);
            y = __dsub_rn(__dmul_rn(2.0, canonical(O[2 * tid + 1])), 1.0);
            r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
            ok = !(r2 > 1.0 || r2 == 0.0);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0 && warp < 3) wsum[warp] = __popc(bal);
        __syncthreads();
        const int tot = wsum[0] + wsum[1] + wsum[2];
        if (MODE == 1 && ok) {
            int pre = __popc(bal & ((1u << lane) - 1u));
            for (int w = 0; w < warp; ++w) pre += wsum[w];
            const int64_t idx = 2 * (base_pair + acc + pre);
            // mult = sqrt(-2 log(r2) / r2); returns y*mult, then the saved x*mult;
            // each passes through `ret * stddev + mean` with (1, 0).
            const double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
            if (idx < count) out[idx] = __dadd_rn(__dmul_rn(__dmul_rn(y, mult), 1.0), 0.0);
            if (idx + 1 < count) out[idx + 1] = __dadd_rn(__dmul_rn(__dmul_rn(x, mult), 1.0), 0.0);
        }
        acc += tot;
        if (MODE == 1 && 2 * (base_pair + acc) >= count) break;
        __syncthreads();
    }
    if (MODE == 0 && tid == 0) counts[k] = acc;
}

struct PolyCache {
    std::mutex mu;
    std::map<std::pair<int, int>, uint32_t*> dev;  // (device, log2 steps) -> polys
    int groups = 0;
};
PolyCache& cache() {
    static PolyCache c;
    return c;
}

const uint32_t* device_polys(Ctx& c, int log2S, int& groups) {
    PolyCache& pc = cache();
    std::lock_guard<std::mutex> lk(pc.mu);
    auto key = std::make_pair(c.device, log2S);
    auto it = pc.dev.find(key);
    if (it != pc.dev.end()) {
        groups = pc.groups;
        return it->second;
    }
    std::vector<uint32_t> h;
    mt64_jump_polys(log2S, kMaxJumps, h, groups);
    pc.groups = groups;
    uint32_t* d = nullptr;
    FB_CUDA(cudaMalloc(&d, h.size() * sizeof(uint32_t)));
    FB_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    pc.dev[key] = d;
    return d;
}

}  // namespace

void gaussian_stream_device(Ctx& c, uint64_t seed, int64_t count, double* out) {
    if (count <= 0) return;
    Prof prof(c, "omega_device", 8.0 * count, 0.0);
    cudaStream_t s = c.stream;
    // pairs needed with margin: accepted pairs ~ Bin(P, pi/4), need 2*acc >= count
    const double half = 0.5 * double(count);
    int64_t P = int64_t(half / (M_PI / 4.0) + 8.0 * std::sqrt(half / (M_PI / 4.0)) + 64.0);
    // segments of J = 156 * 2^e words (~2k segments at most per 2^e step)
    int log2S = 6;
    while (log2S < 14 && (2 * P) / (int64_t(MM) << log2S) > 2048) ++log2S;
    const int64_t J = int64_t(MM) << log2S;
    int groups = 0;
    const uint32_t* polys = device_polys(c, log2S, groups);
    uint64_t s0[NN];
    mt64_seed_state(seed, s0);
    DBuf<uint64_t> d_s0(NN, s);
    FB_CUDA(cudaMemcpyAsync(d_s0.get(), s0, sizeof(s0), cudaMemcpyHostToDevice, s));
    for (int attempt = 0; attempt < 4; ++attempt) {
        const int64_t K = (2 * P + J - 1) / J;
        require(K < (int64_t(1) << kMaxJumps), "gaussian_matrix: stream too long for the jump table");
        DBuf<uint64_t> states(size_t(K) * NN, s);
        DBuf<int64_t> counts(size_t(K) + 1, s), offs(size_t(K) + 1, s);
        k_jump<<<unsigned(K), 320, 0, s>>>(d_s0.get(), polys, groups, states.get());
        FB_LAUNCH_CHECK();
        FB_CUDA(cudaMemsetAsync(counts.get(), 0, counts.bytes(), s));
        k_polar<0><<<unsigned(K), 160, 0, s>>>(states.get(), J / MM, nullptr, counts.get(), nullptr, count);
        FB_LAUNCH_CHECK();
        size_t tb = 0;
        FB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts.get(), offs.get(), K + 1, s));
        DBuf<unsigned char> tmp(tb, s);
        FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, counts.get(), offs.get(), K + 1, s));
        int64_t total = 0;
        FB_CUDA(cudaMemcpyAsync(&total, offs.get() + K, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        FB_CUDA(cudaStreamSynchronize(s));
        if (2 * total >= count) {
            k_polar<1><<<unsigned(K), 160, 0, s>>>(states.get(), J / MM, offs.get(), nullptr, out, count);
            FB_LAUNCH_CHECK();
            return;
        }
        P = P + P / 8 + 1024;
    }
    throw CudaError("gaussian_matrix: device stream generation did not converge");
}

}  // namespace fb
