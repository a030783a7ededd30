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

// polar attempt on raw words (w0, w1): x = 2u1 - 1, y = 2u2 - 1, r2 = x^2 + y^2
__device__ __forceinline__ bool attempt(uint64_t w0, uint64_t w1, double& x, double& y, double& r2) {
    x = __dsub_rn(__dmul_rn(2.0, canonical(w0)), 1.0);
    y = __dsub_rn(__dmul_rn(2.0, canonical(w1)), 1.0);
    r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    return !(r2 > 1.0 || r2 == 0.0);
}

// the two normals of an accepted attempt: mult = sqrt(-2 log(r2) / r2);
// y*mult first, then the saved x*mult, each through `ret * stddev + mean`
// with (1, 0) (random.tcc)
__device__ __forceinline__ void polar_pair(double x, double y, double r2, double& a, double& b) {
    const double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, glibc_log::log_polar(r2)), r2));
    a = __dadd_rn(__dmul_rn(__dmul_rn(y, mult), 1.0), 0.0);
    b = __dadd_rn(__dmul_rn(__dmul_rn(x, mult), 1.0), 0.0);
}

// Phase 1, one CTA per segment (seg0 + blockIdx.x): the raw stream, 156 new
// words per step from a ring of 4 x 156 words (step s reads [b, b + 312) and
// writes [b + 312, b + 468) mod 624, b = 156 (s mod 4)), in rounds of four
// steps. After a round the ring holds its 624 words, word w at (312 + w) mod
// 624: 312 polar attempts (threads t < 156 take attempts t and t + 156),
// whose normals go, in stream order, to the segment's staging slots
// stage[seg J + i]; cnt[seg] = normals of the segment. Nothing but the
// normals reaches global memory (no raw-word buffer).
constexpr int GT = 160;
constexpr int kGenPerSm = 9;  // segments per SM the host plans for (5 warps each; 9 fit by registers)
__global__ void __launch_bounds__(GT)
k_gen_polar(const uint64_t* __restrict__ states, int64_t seg0, int64_t steps, int64_t J,
            double* __restrict__ stage, int64_t* __restrict__ cnt) {
    constexpr int RING = 4 * MM;
    using Scan = cub::BlockScan<unsigned, GT>;
    __shared__ uint64_t X[RING];
    __shared__ typename Scan::TempStorage tmp;
    const int tid = threadIdx.x;
    const int64_t seg = seg0 + blockIdx.x;
    for (int i = tid; i < NN; i += GT) X[i] = states[seg * NN + i];
    double* out = stage + int64_t(blockIdx.x) * J;  // the batch's staging starts at segment seg0
    int64_t pairs = 0;  // accepted attempts so far (block-uniform)
    for (int64_t r = 0; r < steps; r += 4) {
        __syncthreads();  // (the previous round's ring reads are done)
#pragma unroll
        for (int st = 0; st < 4; ++st) {
            if (tid < MM) {
                const int i0 = st * MM + tid;
                const int i1 = i0 + 1 < RING ? i0 + 1 : i0 + 1 - RING;
                const int i2 = i0 + MM < RING ? i0 + MM : i0 + MM - RING;
                const int io = i0 + 2 * MM < RING ? i0 + 2 * MM : i0 + 2 * MM - RING;
                X[io] = mt_next(X[i0], X[i1], X[i2]);
            }
            __syncthreads();
        }
        bool ok0 = false, ok1 = false;
        double x0 = 0, y0 = 0, r0 = 0, x1 = 0, y1 = 0, r1 = 0;
        if (tid < MM) {
            // attempt t: words 2t, 2t + 1 at ring 312 + 2t (+1); attempt t + 156:
            // words 312 + 2t (+1) at ring 2t (+1)
            ok0 = attempt(temper(X[2 * MM + 2 * tid]), temper(X[2 * MM + 2 * tid + 1]), x0, y0, r0);
            ok1 = attempt(temper(X[2 * tid]), temper(X[2 * tid + 1]), x1, y1, r1);
        }
        unsigned pre = 0, tot = 0;
        Scan(tmp).ExclusiveSum((ok0 ? 1u : 0u) | ((ok1 ? 1u : 0u) << 16), pre, tot);
        const int64_t first = int64_t(tot & 0xffffu);
        if (ok0) {
            double a, b;
            polar_pair(x0, y0, r0, a, b);
            const int64_t o = 2 * (pairs + int64_t(pre & 0xffffu));
            out[o] = a;
            out[o + 1] = b;
        }
        if (ok1) {
            double a, b;
            polar_pair(x1, y1, r1, a, b);
            const int64_t o = 2 * (pairs + first + int64_t(pre >> 16));
            out[o] = a;
            out[o + 1] = b;
        }
        pairs += first + int64_t(tot >> 16);
    }
    if (tid == 0) cnt[seg] = 2 * pairs;
}

// A window of the stream: positions p < count with (p mod P) in [w0, w1).
// Column-major: out[(p / P) (w1 - w0) + (p mod P - w0)] (a rank's rows of a
// column-major sketch; P = count: a contiguous slice). Row-major (k_place_rm):
// out[(p mod P - w0) ncols + p / P], the transposed layout the products read.
struct Window {
    int64_t P, w0, w1;
    bool ident;  // the whole stream, out[p]
};

// Phase 2, column-major window: segment s0 + blockIdx.x's normals to their
// stream positions (positions in [plo, phi) only)
__global__ void __launch_bounds__(256)
k_place(const double* __restrict__ stage, int64_t J, const int64_t* __restrict__ off,
        const int64_t* __restrict__ cnt, int64_t s0, int64_t count, Window w, double* __restrict__ out) {
    const int64_t seg = s0 + blockIdx.x;
    const int64_t base = off[seg], n = cnt[seg];
    const double* src = stage + int64_t(blockIdx.x) * J;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t p = base + i;
        if (p >= count) break;
        const double v = __ldcs(src + i);
        if (w.ident) {
            __stcs(out + p, v);
            continue;
        }
        const int64_t q = p / w.P, r = p - q * w.P;
        if (r >= w.w0 && r < w.w1) __stcs(out + q * (w.w1 - w.w0) + (r - w.w0), v);
    }
}

// Segment lookup of the row-major placement: seg_at[b] = the segment holding
// stream position b * kBucket (segments hold thousands of normals, so a
// position's segment is seg_at[p / kBucket] or one of the next few).
constexpr int64_t kBucket = 1024;
__global__ void k_seg_buckets(const int64_t* __restrict__ off, int64_t s0, int64_t s1, int64_t nbuck,
                              int32_t* __restrict__ seg_at) {
    for (int64_t k = s0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < s1; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b0 = (off[k] + kBucket - 1) / kBucket;
        const int64_t b1 = min(nbuck, (off[k + 1] + kBucket - 1) / kBucket);
        for (int64_t b = b0; b < b1; ++b) seg_at[b] = int32_t(k);
    }
}

__device__ __forceinline__ int64_t seg_of(const int64_t* __restrict__ off, const int32_t* __restrict__ seg_at,
                                          int64_t nseg, int64_t p) {
    int64_t k = seg_at[p / kBucket];
    while (k + 1 < nseg && off[k + 1] <= p) ++k;
    return k;
}

// Phase 2, row-major window: a 128-row x 32-column tile of the output per
// CTA. Column q's rows r0..r0+127 are the stream run q P + r: read from the
// staging (one or two segments) into shared memory, 16 independent loads in
// flight per thread, then written as 256-byte row segments. Positions
// outside [plo, phi) are left to another batch.
constexpr int kTR = 128, kTC = 32;
__global__ void __launch_bounds__(256)
k_place_rm(const double* __restrict__ stage, int64_t J, const int64_t* __restrict__ off,
           const int32_t* __restrict__ seg_at, int64_t s0, int64_t s1, int64_t count, int64_t P, int64_t w0,
           int64_t w1, int64_t ncols, int64_t ncb_launch, double* __restrict__ out) {
    __shared__ double tile[kTC][kTR + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // column blocks vary fastest across CTAs, so the CTAs in flight complete
    // whole output rows (full lines merge in L2 before they reach DRAM)
    // this batch's stream positions: segments [s0, s1); its columns start at
    // block plo / P / kTC, and ncb_launch column blocks cover any batch
    const int64_t plo = off[s0], phi = min(off[s1], count);
    const int64_t ncb = (ncols + kTC - 1) / kTC;
    const int64_t cb = (plo / P) / kTC + int64_t(blockIdx.x % ncb_launch);
    if (cb >= ncb) return;
    const int64_t r0 = w0 + int64_t(blockIdx.x / ncb_launch) * kTR, q0 = cb * kTC;
    const int64_t qlast = min(q0 + kTC, ncols) - 1;
    if (q0 * P + r0 >= phi || qlast * P + min(r0 + kTR, w1) - 1 < plo) return;  // tile outside the batch
    double v[kTC / 8][kTR / 32];
#pragma unroll
    for (int j = 0; j < kTC / 8; ++j) {
        const int64_t q = q0 + warp + 8 * j;
#pragma unroll
        for (int h = 0; h < kTR / 32; ++h) {
            const int rr = lane + 32 * h;
            const int64_t p = q * P + r0 + rr;
            v[j][h] = 0.0;
            if (q < ncols && r0 + rr < w1 && p >= plo && p < phi) {
                const int64_t k = seg_of(off, seg_at, s1, p);
                v[j][h] = __ldcs(stage + (k - s0) * J + (p - off[k]));
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kTC / 8; ++j)
#pragma unroll
        for (int h = 0; h < kTR / 32; ++h) tile[warp + 8 * j][lane + 32 * h] = v[j][h];
    __syncthreads();
    const int64_t q = q0 + lane;
    for (int rr = warp; rr < kTR; rr += 8) {
        const int64_t r = r0 + rr;
        if (r >= w1 || q >= ncols) continue;
        const int64_t p = q * P + r;
        if (p < plo || p >= phi) continue;
        __stcs(out + (r - w0) * ncols + q, tile[lane][rr]);
    }
}

// single-batch Omega: the shortfall check of the host loop, on the device
__global__ void k_check_short(const int64_t* __restrict__ total, int64_t count, int* __restrict__ flag) {
    if (total[0] < count) atomicCAS(flag, 0, kErrOmegaShort);
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
    gaussian_stream_window(c, seed, count, count, 0, count, out, false);
}

void gaussian_stream_window(Ctx& c, uint64_t seed, int64_t count, int64_t period, int64_t w0, int64_t w1,
                            double* out, bool rowmajor) {
    if (count <= 0) return;
    const Window win{period, w0, w1, period >= count && w0 == 0 && w1 >= count};
    const int64_t ncols = (count + period - 1) / period;  // columns of the (row-major) window
    Prof prof(c, "omega_total", 8.0 * double(count) * double(w1 - w0) / double(period), 0.0);
    cudaStream_t s = c.stream;
    // attempts needed with margin: accepted ~ Bin(P, pi/4), need 2*acc >= count
    const double half = 0.5 * double(count);
    const int64_t P = int64_t(half / (M_PI / 4.0) + 8.0 * std::sqrt(half / (M_PI / 4.0)) + 64.0);
    // segments of J = 156 * 2^e words: the fewest that still fill the
    // generator (one CTA per segment, kGenPerSm per SM), at most 2^12 steps
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
    // one batch of K segments covers the stream (shortfall probability
    // ~1e-15): the deferred check re-runs the call with omega_sync, whose
    // host check regenerates with the 2K + 1 segments of the jump table
    int64_t K = (2 * P + J - 1) / J;
    const int64_t Kmax = 2 * K + 1;
    require(Kmax <= (int64_t(1) << (4 * kJumpLevels)), "gaussian_matrix: stream too long for the jump table");
    const bool defer = c.checked && !c.omega_sync;
    DBuf<uint64_t> states(size_t(defer ? K : Kmax) * NN, s);
    {
        Prof pj(c, "omega_jump", 0.0, 0.0);
        FB_CUDA(cudaMemcpyAsync(states.get(), s0, sizeof(s0), cudaMemcpyHostToDevice, s));
        jump_states(c, states.get(), polys, groups, 1, K);
    }
    // Staging: J normals per segment at most, kept on the context (Ctx::
    // omega_stage: re-taking a 41 GB block per call stalls on pool re-maps)
    // and grown only while 24 GB of device memory stay free; beyond that the
    // segments go in batches. One batch is faster for the row-major placement
    // (the CTAs in flight complete whole output rows; a batch covers only
    // some columns): C4 16.7 ms vs 24.4 ms in 5 batches.
    DBuf<double>& stage = c.omega_stage;
    {
        const size_t need = sizeof(double) * size_t(K) * size_t(J);
        if (stage.bytes() < need) {
            size_t fr = 0, tot = 0;
            FB_CUDA(cudaMemGetInfo(&fr, &tot));
            const size_t head = size_t(24) << 30, have = stage.bytes();
            const size_t room = fr + have > head ? fr + have - head : 0;
            const size_t want = std::min(need, std::max(room, size_t(2) << 30));
            if (want > have) {
                stage.release();
                stage.alloc(std::max<size_t>(J, want / sizeof(double)), s);
            }
        }
    }
    const int64_t spb = std::max<int64_t>(1, int64_t(stage.n / size_t(J)));
    const int64_t nbuck = (count + kBucket - 1) / kBucket;
    for (int attempt_no = 0;; ++attempt_no) {
        DBuf<int64_t> cnt(size_t(K) + 1, s), off(size_t(K) + 1, s);
        FB_CUDA(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));
        DBuf<int32_t> seg_at;
        if (rowmajor) {
            seg_at.alloc(size_t(nbuck), s);
            FB_CUDA(cudaMemsetAsync(seg_at.get(), 0, seg_at.bytes(), s));  // (a deferred shortfall leaves a tail)
        }
        size_t tb = 0;
        FB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), off.get(), K + 1, s));
        DBuf<unsigned char> tmp(tb, s);
        for (int64_t s0 = 0; s0 < K; s0 += spb) {
            const int64_t s1 = std::min(K, s0 + spb);
            {
                Prof pg(c, "omega_gen", 8.0 * double(count) * double(s1 - s0) / double(K), 0.0);
                k_gen_polar<<<unsigned(s1 - s0), GT, 0, s>>>(states.get(), s0, steps, J, stage.get(), cnt.get());
                FB_LAUNCH_CHECK();
                // offsets of segments [0, s1] (cnt past s1 is still 0)
                FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt.get(), off.get(), s1 + 1, s));
            }
            Prof pe(c, "omega_place", 16.0 * double(count) * double(w1 - w0) / double(period) * double(s1 - s0) / double(K),
                    0.0);
            if (rowmajor) {
                k_seg_buckets<<<unsigned((s1 - s0 + 255) / 256), 256, 0, s>>>(off.get(), s0, s1, nbuck, seg_at.get());
                FB_LAUNCH_CHECK();
                // a batch holds at most (s1 - s0) J normals: the column blocks it can touch
                const int64_t ncb = (ncols + kTC - 1) / kTC;
                const int64_t ncb_launch = K <= spb ? ncb : std::min(ncb, ((s1 - s0) * J / period + 1) / kTC + 2);
                const int64_t ntiles = (w1 - w0 + kTR - 1) / kTR * ncb_launch;
                require(ntiles < (int64_t(1) << 31), "gaussian_matrix: window too large");
                k_place_rm<<<unsigned(ntiles), 256, 0, s>>>(stage.get(), J, off.get(), seg_at.get(), s0, s1, count,
                                                            period, w0, w1, ncols, ncb_launch, out);
            } else {
                k_place<<<unsigned(s1 - s0), 256, 0, s>>>(stage.get(), J, off.get(), cnt.get(), s0, count, win, out);
            }
            FB_LAUNCH_CHECK();
        }
        // FRPCA_TEST_OMEGA_SHORT: tests force the shortfall -> re-run path
        const bool force = std::getenv("FRPCA_TEST_OMEGA_SHORT") != nullptr;
        if (defer) {
            k_check_short<<<1, 1, 0, s>>>(off.get() + K, force ? INT64_MAX : count, err_flag(c));
            FB_LAUNCH_CHECK();
            break;
        }
        const int64_t total = read_i64(c, off.get() + K);
        if (total >= count && !(force && attempt_no == 0)) break;
        // shortfall: the whole stream again over the longer jump table
        require(K < Kmax, "gaussian_matrix: device stream generation did not converge");
        jump_states(c, states.get(), polys, groups, K, Kmax);
        K = Kmax;
    }
}

}  // namespace fb
