// Seeded synthetic CSR generators for BASELINE.json's configs C0-C4
// (SURVEY §8d). The paper's datasets (MovieLens / AMiner / SNAP) are not in
// this environment; these generators reproduce the shapes, nnz and the value /
// degree / popularity laws BASELINE.json names, deterministically for a seed,
// and are shared by the oracle checks and the GPU runs (same CSR bytes).
// Host-only input preparation (not part of the measured hot path).
//
// Conventions (documented in DESIGN.md):
//  * every row draws DISTINCT column ids (duplicates are redrawn), then sorts;
//  * degree laws: scale first, then clip: d = clip(round(s*z), lo, hi), the
//    scale s solved so that E[d] * rows = target nnz;
//  * column popularity: rank ~ Zipf(a) on [1, cols], column = perm[rank-1] for a
//    seeded permutation of the columns;
//  * per-row RNG streams (xoshiro256** seeded by SplitMix64(seed, row)), so the
//    generation is parallel and independent of the thread count.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

namespace {

inline uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

struct Rng {  // xoshiro256**
    uint64_t s[4];
    Rng(uint64_t seed, uint64_t stream) {
        uint64_t x = seed ^ (0xD1B54A32D192ED03ULL * (stream + 1));
        for (auto& w : s) w = splitmix(x);
    }
    static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    inline uint64_t next() {
        const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
        return r;
    }
    inline double uniform() { return double(next() >> 11) * 0x1.0p-53; }        // [0, 1)
    inline double uniform_open() { return (double(next() >> 11) + 0.5) * 0x1.0p-53; }  // (0, 1)
    inline double normal() {  // Box-Muller
        const double u1 = uniform_open(), u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
};

// Rejection-inversion sampling of Zipf(a) on [1, N] (Hoermann & Derflinger 1996).
struct Zipf {
    double a, hx1, hn, s;
    int64_t N;
    static double helper1(double x) { return std::abs(x) > 1e-8 ? std::log1p(x) / x : 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x)); }
    static double helper2(double x) { return std::abs(x) > 1e-8 ? std::expm1(x) / x : 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x)); }
    double H(double x) const { const double lx = std::log(x); return helper2((1.0 - a) * lx) * lx; }
    double h(double x) const { return std::exp(-a * std::log(x)); }
    double Hinv(double x) const {
        double t = x * (1.0 - a);
        if (t < -1.0) t = -1.0;
        return std::exp(helper1(t) * x);
    }
    Zipf(double a_, int64_t N_) : a(a_), N(N_) {
        hx1 = H(1.5) - 1.0;
        hn = H(double(N) + 0.5);
        s = 2.0 - Hinv(H(2.5) - h(2.0));
    }
    int64_t operator()(Rng& r) const {
        for (;;) {
            const double u = hn + r.uniform() * (hx1 - hn);
            const double x = Hinv(u);
            int64_t k = int64_t(x + 0.5);
            if (k < 1) k = 1; else if (k > N) k = N;
            if (double(k) - x <= s || u >= H(double(k) + 0.5) - h(double(k))) return k;
        }
    }
};

int64_t poisson(Rng& r, double lam) {
    if (lam < 30.0) {  // multiplication method
        const double L = std::exp(-lam);
        int64_t k = 0;
        double p = r.uniform();
        while (p > L) { ++k; p *= r.uniform(); }
        return k;
    }
    // PTRS transformed rejection (Hoermann 1993)
    const double slam = std::sqrt(lam), loglam = std::log(lam);
    const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
    const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2.0);
    for (;;) {
        const double U = r.uniform() - 0.5, V = r.uniform();
        const double us = 0.5 - std::abs(U);
        const int64_t k = int64_t(std::floor((2.0 * a / us + b) * U + lam + 0.43));
        if (us >= 0.07 && V <= vr) return k;
        if (k < 0 || (us < 0.013 && V > us)) continue;
        if (std::log(V) + std::log(invalpha) - std::log(a / (us * us) + b) <=
            -lam + double(k) * loglam - std::lgamma(double(k) + 1.0))
            return k;
    }
}

template <class F>
void parallel_blocks(int64_t n, int threads, int64_t block, F&& f) {
    std::atomic<int64_t> next{0};
    const int t = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int w = 0; w < t; ++w)
        pool.emplace_back([&] {
            for (int64_t b = next.fetch_add(block); b < n; b = next.fetch_add(block))
                f(b, std::min(n, b + block));
        });
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// row_law: 0 Bernoulli(p) per entry (uniform columns), 1 Zipf(row_a) scaled+clipped,
//          2 Poisson(row_lambda)
// col_law: 0 uniform (implied by row_law 0), 1 Zipf(col_a) over a seeded permutation
// val_law: 0 U(0,1), 1 lognormal(0,1), 2 Poisson(1)+1, 3 1.0 or (10%) U(1,5), 4 N(0,1)
typedef struct {
    int64_t rows, cols;
    int32_t row_law, col_law, val_law, pad;
    double row_p, row_a, row_lo, row_hi, row_scale, row_lambda, col_a;
    uint64_t seed;
} synth_spec;

// Expected degree E[clip(round(s*z), lo, hi)] for z ~ Zipf(a) on [1, inf).
double synth_expected_degree(double a, double s, double lo, double hi) {
    // truncate the Zipf sum once s*z > hi (mass of the tail goes to hi)
    double zeta = 0.0;
    const int64_t K = 50000000;
    std::vector<double> unused;
    double acc = 0.0, mass = 0.0;
    int64_t k = 1;
    for (; k <= K; ++k) {
        const double pk = std::pow(double(k), -a);
        zeta += pk;
        double d = std::round(s * double(k));
        if (d >= hi) break;
        if (d < lo) d = lo;
        acc += pk * d;
        mass += pk;
    }
    // zeta(a) by the partial sum + Euler-Maclaurin tail
    double z = 0.0;
    const int64_t M = 100000;
    for (int64_t j = 1; j <= M; ++j) z += std::pow(double(j), -a);
    z += std::pow(double(M), 1.0 - a) / (a - 1.0) - 0.5 * std::pow(double(M), -a);
    (void)zeta;
    return (acc + (z - mass) * hi) / z;
}

// Solve s with E[degree] * rows = target (bisection).
double synth_solve_scale(double a, double lo, double hi, double mean_target) {
    double l = 1e-3, h = hi;
    for (int it = 0; it < 80; ++it) {
        const double mid = 0.5 * (l + h);
        if (synth_expected_degree(a, mid, lo, hi) < mean_target) l = mid; else h = mid;
    }
    return 0.5 * (l + h);
}

static int64_t row_degree(const synth_spec& sp, int64_t i, Rng& r) {
    switch (sp.row_law) {
        case 0: {  // count of Bernoulli(p) successes: replay the skip process
            int64_t c = 0;
            const double lq = std::log1p(-sp.row_p);
            int64_t j = -1;
            for (;;) {
                j += 1 + int64_t(std::floor(std::log(r.uniform_open()) / lq));
                if (j >= sp.cols) break;
                ++c;
            }
            return c;
        }
        case 1: {
            static thread_local Zipf* zr = nullptr;
            static thread_local double za = 0;
            if (!zr || za != sp.row_a) { delete zr; zr = new Zipf(sp.row_a, int64_t(1) << 40); za = sp.row_a; }
            const double z = double((*zr)(r));
            double d = std::round(sp.row_scale * z);
            d = std::min(std::max(d, sp.row_lo), sp.row_hi);
            return std::min<int64_t>(int64_t(d), sp.cols);
        }
        default: {
            const int64_t d = poisson(r, sp.row_lambda);
            return std::min<int64_t>(std::max<int64_t>(d, 0), sp.cols);
        }
    }
    (void)i;
}

int synth_degrees(const synth_spec* sp, int threads, int64_t* row_ptr) {
    row_ptr[0] = 0;
    parallel_blocks(sp->rows, threads, 16384, [&](int64_t b, int64_t e) {
        for (int64_t i = b; i < e; ++i) {
            Rng r(sp->seed, uint64_t(2 * i));
            row_ptr[i + 1] = row_degree(*sp, i, r);
        }
    });
    for (int64_t i = 0; i < sp->rows; ++i) row_ptr[i + 1] += row_ptr[i];
    return 0;
}

static double draw_value(int law, Rng& r) {
    switch (law) {
        case 0: return r.uniform_open();
        case 1: return std::exp(r.normal());
        case 2: return double(poisson(r, 1.0) + 1);
        case 3: return r.uniform() < 0.1 ? 1.0 + 4.0 * r.uniform_open() : 1.0;
        default: {
            double v;
            do { v = r.normal(); } while (v == 0.0);
            return v;
        }
    }
}

int synth_fill(const synth_spec* sp, int threads, const int64_t* row_ptr, int64_t* col_idx,
               double* values) {
    std::vector<int32_t> perm;
    if (sp->col_law == 1) {
        perm.resize(size_t(sp->cols));
        std::iota(perm.begin(), perm.end(), 0);
        Rng pr(sp->seed ^ 0x5eed5eedULL, ~0ull);
        for (int64_t j = sp->cols - 1; j > 0; --j) {
            const int64_t k = int64_t(pr.next() % uint64_t(j + 1));
            std::swap(perm[size_t(j)], perm[size_t(k)]);
        }
    }
    const Zipf colz(sp->col_law == 1 ? sp->col_a : 2.0, std::max<int64_t>(sp->cols, 1));
    parallel_blocks(sp->rows, threads, 4096, [&](int64_t b, int64_t e) {
        std::vector<int64_t> table;  // open addressing set of drawn ranks
        std::vector<int64_t> got;
        for (int64_t i = b; i < e; ++i) {
            const int64_t p0 = row_ptr[i], d = row_ptr[i + 1] - p0;
            Rng r(sp->seed, uint64_t(2 * i + 1));
            int64_t* ci = col_idx + p0;
            if (sp->row_law == 0) {
                Rng rd(sp->seed, uint64_t(2 * i));  // same skip process as the degree pass
                const double lq = std::log1p(-sp->row_p);
                int64_t j = -1, c = 0;
                for (;;) {
                    j += 1 + int64_t(std::floor(std::log(rd.uniform_open()) / lq));
                    if (j >= sp->cols) break;
                    ci[c++] = j;
                }
            } else if (sp->col_law == 1) {
                if (d * 2 >= sp->cols) {
                    // dense-ish row: draw distinct ranks by scanning a shuffled tail
                    std::vector<char> used(size_t(sp->cols), 0);
                    int64_t c = 0;
                    while (c < d) {
                        const int64_t k = colz(r) - 1;
                        if (!used[size_t(k)]) { used[size_t(k)] = 1; ci[c++] = perm[size_t(k)]; }
                    }
                } else {
                    size_t cap = 16;
                    while (cap < size_t(4 * d)) cap <<= 1;
                    table.assign(cap, -1);
                    int64_t c = 0;
                    while (c < d) {
                        const int64_t k = colz(r);
                        size_t h = size_t((uint64_t(k) * 0x9E3779B97F4A7C15ULL) >> 20) & (cap - 1);
                        bool dup = false;
                        while (table[h] != -1) {
                            if (table[h] == k) { dup = true; break; }
                            h = (h + 1) & (cap - 1);
                        }
                        if (dup) continue;
                        table[h] = k;
                        ci[c++] = perm[size_t(k - 1)];
                    }
                }
                std::sort(ci, ci + d);
            } else {
                // uniform distinct columns (Floyd's algorithm)
                got.clear();
                size_t cap = 16;
                while (cap < size_t(4 * d)) cap <<= 1;
                table.assign(cap, -1);
                int64_t c = 0;
                while (c < d) {
                    const int64_t k = int64_t(r.next() % uint64_t(sp->cols));
                    size_t h = size_t((uint64_t(k) * 0x9E3779B97F4A7C15ULL) >> 20) & (cap - 1);
                    bool dup = false;
                    while (table[h] != -1) {
                        if (table[h] == k) { dup = true; break; }
                        h = (h + 1) & (cap - 1);
                    }
                    if (dup) continue;
                    table[h] = k;
                    ci[c++] = k;
                }
                std::sort(ci, ci + d);
            }
            for (int64_t t = 0; t < d; ++t) values[p0 + t] = draw_value(sp->val_law, r);
        }
    });
    return 0;
}

}  // extern "C"
