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
// nearest without contraction, and log(r2) is glibc's log restated operation
// for operation (glibc_log.cuh: the FMA build the host's ifunc selects), so
// every normal is bitwise equal to libstdc++'s.
#include <cub/cub.cuh>

#include <cmath>
#include <map>
#include <mutex>

#include "glibc_log.cuh"
#include <cstdlib>

#include "internal.cuh"

namespace fb {

int mt64_jump_polys(int log2_steps, int levels, std::vector<uint32_t>& out, int& groups);
void mt64_seed_state(uint64_t seed, uint64_t* state312);

namespace {

constexpr int NN = 312;
constexpr int MM = 156;
constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MA = 0xB5026F5AA96619E9ULL;
constexpr int kJumpLevels = 4;  // 16-ary jump tree: up to 16^4 segments

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

// Segment start states by a 16-ary tree: level a computes, for every
// k = q 16^a + r in [16^a, 16^(a+1)) (q = 1..15, r < 16^a),
// state_k = T^(J q 16^a) state_r with the jump polynomial x^(J q 16^a) mod P
// (one jump per segment in total, ceil(log16 K) dependent levels). Horner over the 19937
// coefficients, 64 per step: r <- T^64 r + sum_b c_(64g+b) T^b base.
// The window T^b base is the base sequence shifted by b, so one shared table
// serves every thread: N[v][j] = XOR of ext[j + i] over the set bits i of the
// nibble v, and the 64-coefficient sum for thread j is
//   XOR_q N[nibble_q(c)][j + 4q], q = 0..15  (16 conflict-free shared loads).
// The window r is ping-ponged, so a step is one barrier.
constexpr int JW = 64;             // coefficients per Horner step
constexpr int NTAB = NN + JW;      // table row length (j + 4q + 3 < NN + 63)
constexpr size_t kNibBytes = sizeof(uint64_t) * 16 * NTAB;

// (ext is dead once the nibble table is built and holds the first window:
// 56 KB per CTA, four CTAs per SM)
__global__ void __launch_bounds__(320, 4)
k_jump_level(uint64_t* __restrict__ states, const uint32_t* __restrict__ polys, int groups, int64_t first,
             int64_t k0, int64_t k1) {
    __shared__ uint64_t ext[NN + JW];
    extern __shared__ uint64_t nib_dyn[];  // [16][NTAB]
    uint64_t (*nib)[NTAB] = reinterpret_cast<uint64_t (*)[NTAB]>(nib_dyn);
    __shared__ uint64_t R1[NN];
    __shared__ uint32_t co[640];
    const int tid = threadIdx.x;
    const int64_t k = k0 + blockIdx.x;
    if (k >= k1) return;
    const uint64_t* src = states + size_t(k % first) * NN;
    const uint32_t* poly = polys + size_t(k / first - 1) * groups;
    if (tid < NN) ext[tid] = src[tid];
    for (int g = tid; g < groups; g += blockDim.x) co[g] = poly[g];
    __syncthreads();
    if (tid < JW) ext[NN + tid] = mt_next(ext[tid], ext[tid + 1], ext[tid + MM]);
    __syncthreads();
    for (int e = tid; e < 16 * NTAB; e += blockDim.x) {
        const int v = e / NTAB, j = e % NTAB;
        uint64_t x = 0;
        #pragma unroll
        for (int i = 0; i < 4; ++i)
            if (((v >> i) & 1) && j + i < NN + JW) x ^= ext[j + i];
        nib[v][j] = x;
    }
    __syncthreads();
    if (tid < NN) ext[tid] = 0;  // window 0
    __syncthreads();
    int cur = 0;
    const int ng = (groups + 1) / 2;  // 64-bit coefficient groups
    for (int g = ng - 1; g >= 0; --g) {
        const uint32_t lo = co[2 * g], hi = (2 * g + 1 < groups) ? co[2 * g + 1] : 0u;
        if (tid < NN) {
            uint64_t x = 0;
            #pragma unroll
            for (int q = 0; q < 8; ++q) x ^= nib[(lo >> (4 * q)) & 15u][tid + 4 * q];
            #pragma unroll
            for (int q = 0; q < 8; ++q) x ^= nib[(hi >> (4 * q)) & 15u][tid + 32 + 4 * q];
            const uint64_t* r = cur ? R1 : ext;
            uint64_t v;
            if (tid < NN - JW) {
                v = r[tid + JW];
            } else {
                const int t = tid - (NN - JW);
                v = mt_next(r[t], r[t + 1], r[t + MM]);
            }
            (cur ? ext : R1)[tid] = v ^ x;
        }
        cur ^= 1;
        __syncthreads();
    }
    if (tid < NN) states[size_t(k) * NN + tid] = (cur ? R1 : ext)[tid];
}

// Raw stream of a segment: 156 new words per step, one barrier per step. The
// words live in a ring of 4 x 156: step s reads its window at ring offset
// (s mod 4) 156 ([b, b + 312)) and writes the new words at [b + 312, b + 468)
// (mod 624), so no window copy; the tempered outputs go straight to global
// memory (coalesced). 160 threads: the last 4 only keep the barrier count.
constexpr int GT = 160;
constexpr int kGenPerSm = 6;  // segments per SM the host plans for (5 warps each)
__global__ void __launch_bounds__(GT)
k_gen(const uint64_t* __restrict__ states, int64_t seg0, int64_t steps, uint64_t* __restrict__ raw) {
    constexpr int RING = 4 * MM;
    __shared__ uint64_t X[RING];
    const int tid = threadIdx.x;
    const int64_t seg = seg0 + blockIdx.x;
    for (int i = tid; i < NN; i += GT) X[i] = states[seg * NN + i];
    __syncthreads();
    uint64_t* dst = raw + int64_t(blockIdx.x) * steps * MM + tid;
    int b = 0;
    for (int64_t st = 0; st < steps; ++st) {
        if (tid < MM) {
            const int i0 = b + tid;
            const int i1 = i0 + 1 < RING ? i0 + 1 : i0 + 1 - RING;
            const int i2 = i0 + MM < RING ? i0 + MM : i0 + MM - RING;
            const int io = i0 + 2 * MM < RING ? i0 + 2 * MM : i0 + 2 * MM - RING;
            const uint64_t nw = mt_next(X[i0], X[i1], X[i2]);
            X[io] = nw;
            dst[st * MM] = temper(nw);
        }
        b = b + MM < RING ? b + MM : 0;
        __syncthreads();
    }
}

// polar attempt on raw words (w0, w1): x = 2u1 - 1, y = 2u2 - 1, r2 = x^2 + y^2
__device__ __forceinline__ bool attempt(uint64_t w0, uint64_t w1, double& x, double& y, double& r2) {
    x = __dsub_rn(__dmul_rn(2.0, canonical(w0)), 1.0);
    y = __dsub_rn(__dmul_rn(2.0, canonical(w1)), 1.0);
    r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    return !(r2 > 1.0 || r2 == 0.0);
}

constexpr int PT = 256;      // threads per chunk CTA
constexpr int PPT = 4;       // attempts per thread
constexpr int CHUNK = PT * PPT;

// accepted attempts per chunk of CHUNK consecutive attempts
__global__ void __launch_bounds__(PT)
k_count(const uint64_t* __restrict__ raw, int64_t npairs, int64_t* __restrict__ cnt) {
    __shared__ int red[PT / 32];
    // chunk b = attempts [b CHUNK, (b + 1) CHUNK), lane-interleaved (coalesced)
    const int64_t p0 = int64_t(blockIdx.x) * CHUNK + threadIdx.x;
    int c = 0;
    #pragma unroll
    for (int e = 0; e < PPT; ++e) {
        const int64_t q = p0 + int64_t(e) * PT;
        if (q < npairs) {
            const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(raw + 2 * q);
            double x, y, r2;
            c += attempt(w.x, w.y, x, y, r2) ? 1 : 0;
        }
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < PT / 32; ++w) t += red[w];
        cnt[blockIdx.x] = t;
    }
}

// A window of the stream: positions p < count with (p mod P) in [w0, w1) go
// to out[(p / P) (w1 - w0) + (p mod P - w0)] -- a rank's rows of a
// column-major sketch (P = rows), or a contiguous slice (P = count).
struct Window {
    int64_t P, w0, w1;
    bool ident;  // the whole stream, out[p]
};

__device__ __forceinline__ void emit_win(double* __restrict__ out, int64_t p, double v, int64_t count,
                                         const Window& w) {
    if (p >= count) return;
    const int64_t q = p / w.P, r = p - q * w.P;
    if (r < w.w0 || r >= w.w1) return;
    out[q * (w.w1 - w.w0) + (r - w.w0)] = v;
}

// normals of the accepted attempts, written at their stream positions
__global__ void __launch_bounds__(PT, 5)
k_emit(const uint64_t* __restrict__ raw, int64_t npairs, const int64_t* __restrict__ off,
       double* __restrict__ out, int64_t count, Window win) {
    // round e of the chunk = attempts b CHUNK + e PT + [0, PT) (coalesced
    // loads); the stream position of an accepted attempt = accepted attempts
    // of the earlier rounds + of the lower lanes of its round: one block scan
    // of the per-round flags packed in 16-bit fields
    using Scan = cub::BlockScan<unsigned long long, PT>;
    __shared__ typename Scan::TempStorage tmp;
    const int64_t base = off[blockIdx.x];
    if (2 * base >= count) return;
    const int64_t p0 = int64_t(blockIdx.x) * CHUNK + threadIdx.x;
    double xs[PPT], ys[PPT], rs[PPT];
    bool ok[PPT];
    unsigned long long flags = 0;
    #pragma unroll
    for (int e = 0; e < PPT; ++e) {
        const int64_t q = p0 + int64_t(e) * PT;
        ok[e] = false;
        if (q < npairs) {
            const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(raw + 2 * q);
            ok[e] = attempt(w.x, w.y, xs[e], ys[e], rs[e]);
        }
        flags |= (ok[e] ? 1ull : 0ull) << (16 * e);
    }
    unsigned long long pre = 0, tot = 0;
    Scan(tmp).ExclusiveSum(flags, pre, tot);
    const bool vec = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    int64_t rb = base;
    #pragma unroll
    for (int e = 0; e < PPT; ++e) {
        if (ok[e]) {
            const int64_t idx = 2 * (rb + int64_t((pre >> (16 * e)) & 0xffffull));
            // mult = sqrt(-2 log(r2) / r2); y*mult first, then the saved
            // x*mult; each passes through `ret * stddev + mean` with (1, 0)
            // (random.tcc).
            const double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, glibc_log::log_polar(rs[e])), rs[e]));
            const double a = __dadd_rn(__dmul_rn(__dmul_rn(ys[e], mult), 1.0), 0.0);
            const double b = __dadd_rn(__dmul_rn(__dmul_rn(xs[e], mult), 1.0), 0.0);
            if (!win.ident) {
                emit_win(out, idx, a, count, win);
                emit_win(out, idx + 1, b, count, win);
            } else if (vec && idx + 1 < count) {
                __stcs(reinterpret_cast<double2*>(out + idx), make_double2(a, b));
            } else {
                if (idx < count) out[idx] = a;
                if (idx + 1 < count) out[idx + 1] = b;
            }
        }
        rb += int64_t((tot >> (16 * e)) & 0xffffull);
    }
}

// single-batch Omega: the shortfall check of the host loop, on the device
__global__ void k_check_short(const int64_t* __restrict__ pairs, int64_t count, int* __restrict__ flag) {
    if (2 * pairs[0] < count) atomicCAS(flag, 0, kErrOmegaShort);
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
    mt64_jump_polys(log2S, kJumpLevels, h, groups);
    pc.groups = groups;
    uint32_t* d = nullptr;
    FB_CUDA(cudaMalloc(&d, h.size() * sizeof(uint32_t)));
    FB_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    pc.dev[key] = d;
    return d;
}

// start states of segments [k0, k1) (those below k0 already computed), level
// by level of the 16-ary tree
void jump_states(Ctx& c, uint64_t* states, const uint32_t* polys, int groups, int64_t k0, int64_t k1) {
    for (int a = 0; a < kJumpLevels; ++a) {
        const int64_t first = int64_t(1) << (4 * a);
        const int64_t lo = std::max(k0, first), hi = std::min(k1, 16 * first);
        if (lo >= hi) continue;
        k_jump_level<<<unsigned(hi - lo), 320, kNibBytes, c.stream>>>(states, polys + size_t(a) * 15 * groups,
                                                                      groups, first, lo, hi);
        FB_LAUNCH_CHECK();
    }
}

}  // namespace

void gaussian_stream_device(Ctx& c, uint64_t seed, int64_t count, double* out) {
    gaussian_stream_window(c, seed, count, count, 0, count, out);
}

void gaussian_stream_window(Ctx& c, uint64_t seed, int64_t count, int64_t period, int64_t w0, int64_t w1,
                            double* out) {
    if (count <= 0) return;
    const Window win{period, w0, w1, period >= count && w0 == 0 && w1 >= count};
    Prof prof(c, "omega_total", 8.0 * double(count) * double(w1 - w0) / double(period), 0.0);
    cudaStream_t s = c.stream;
    // attempts needed with margin: accepted ~ Bin(P, pi/4), need 2*acc >= count
    const double half = 0.5 * double(count);
    const int64_t P = int64_t(half / (M_PI / 4.0) + 8.0 * std::sqrt(half / (M_PI / 4.0)) + 64.0);
    // segments of J = 156 * 2^e words: the fewest that still fill the
    // generator (one CTA per segment, kGenPerSm per SM), capped so
    // that a batch of <= 2^30 raw words holds >= that many segments
    const int64_t fill = int64_t(c.num_sms) * kGenPerSm;
    int log2S = 6;
    while (log2S < 12 && (2 * P + (int64_t(MM) << log2S) - 1) / (int64_t(MM) << log2S) > fill) ++log2S;
    if (const char* e = std::getenv("FRPCA_OMEGA_LOG2S"))  // segment length override (A/B, tests)
        if (*e) log2S = std::max(6, std::min(14, std::atoi(e)));
    const int64_t steps = int64_t(1) << log2S, J = int64_t(MM) << log2S;
    int groups = 0;
    const uint32_t* polys = nullptr;
    {
        Prof pp(c, "omega_polys", 0.0, 0.0);
        polys = device_polys(c, log2S, groups);
    }
    smem_optin(k_jump_level, size_t(kNibBytes));
    uint64_t s0[NN];
    mt64_seed_state(seed, s0);
    int64_t K = (2 * P + J - 1) / J;
    // room for 2K + 1 segments so that the rare shortfall extends in place
    const int64_t Kmax = 2 * K + 1;
    require(Kmax <= (int64_t(1) << (4 * kJumpLevels)), "gaussian_matrix: stream too long for the jump table");
    DBuf<uint64_t> states(size_t(Kmax) * NN, s);
    {
        Prof pj(c, "omega_jump", 0.0, 0.0);
        FB_CUDA(cudaMemcpyAsync(states.get(), s0, sizeof(s0), cudaMemcpyHostToDevice, s));
        jump_states(c, states.get(), polys, groups, 1, K);
    }
    // batches of segments: raw words -> per-chunk counts -> scan -> normals
    const int64_t seg_per_batch = std::max<int64_t>(1, (int64_t(1) << 30) / J);
    DBuf<uint64_t>& raw = c.omega_raw;  // kept on the context (see DESIGN: pool remaps)
    {
        Prof pa(c, "omega_alloc", 0.0, 0.0);
        const size_t need = size_t(std::min(K, seg_per_batch) * J);
        if (raw.n < need) raw.alloc(need, s);
    }
    int64_t pairs_done = 0;  // accepted attempts emitted so far
    // one batch covers the stream (every BASELINE config): no host round trip,
    // the shortfall test is deferred (err_check re-runs the call with
    // omega_sync); otherwise the batches are checked on the host
    const bool defer = c.checked && !c.omega_sync && K <= seg_per_batch;
    for (int64_t seg0 = 0; 2 * pairs_done < count; seg0 += seg_per_batch) {
        if (seg0 >= K) {
            // shortfall (probability ~ 1e-15): extend the jump table to Kmax
            require(seg0 < Kmax, "gaussian_matrix: device stream generation did not converge");
            jump_states(c, states.get(), polys, groups, K, Kmax);
            K = Kmax;
        }
        const int64_t nseg = std::min(seg_per_batch, K - seg0);
        const int64_t npairs = nseg * J / 2;
        const int64_t nchunks = (npairs + CHUNK - 1) / CHUNK;
        {
            Prof pg(c, "omega_gen", 8.0 * nseg * J, 0.0);
            k_gen<<<unsigned(nseg), GT, 0, s>>>(states.get(), seg0, steps, raw.get());
            FB_LAUNCH_CHECK();
        }
        DBuf<int64_t> cnt(size_t(nchunks) + 1, s), off(size_t(nchunks) + 1, s);
        {
            Prof pc(c, "omega_count", 8.0 * nseg * J, 0.0);
            FB_CUDA(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));
            k_count<<<unsigned(nchunks), PT, 0, s>>>(raw.get(), npairs, cnt.get());
            FB_LAUNCH_CHECK();
            size_t tb = 0;
            FB_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, tb, cnt.get(), off.get(), cub::Sum(),
                                                   pairs_done, nchunks + 1, s));
            DBuf<unsigned char> tmp(tb, s);
            FB_CUDA(cub::DeviceScan::ExclusiveScan(tmp.get(), tb, cnt.get(), off.get(), cub::Sum(),
                                                   pairs_done, nchunks + 1, s));
        }
        {
            Prof pe(c, "omega_emit", 8.0 * nseg * J + 8.0 * count, 0.0);
            k_emit<<<unsigned(nchunks), PT, 0, s>>>(raw.get(), npairs, off.get(), out, count, win);
            FB_LAUNCH_CHECK();
        }
        if (defer) {
            // FRPCA_TEST_OMEGA_SHORT: tests force the shortfall -> re-run path
            const bool force = std::getenv("FRPCA_TEST_OMEGA_SHORT") != nullptr;
            k_check_short<<<1, 1, 0, s>>>(off.get() + nchunks, force ? INT64_MAX : count, err_flag(c));
            FB_LAUNCH_CHECK();
            break;
        }
        FB_CUDA(cudaMemcpyAsync(&pairs_done, off.get() + nchunks, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        FB_CUDA(cudaStreamSynchronize(s));
    }
}

}  // namespace fb
