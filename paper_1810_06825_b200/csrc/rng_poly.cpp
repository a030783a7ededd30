// Host-side GF(2) polynomial algebra for MT19937-64 jump-ahead (the device
// Omega generator, rng.cu).
//
// The state window x[t .. t+311] of std::mt19937_64 advances by one word per
// output; that transition T is linear over GF(2). Its characteristic
// polynomial P (degree 19937) is recovered once per process with
// Berlekamp-Massey from the engine's own output bits, and the jump
// polynomials g_a(x) = x^(J * 2^a) mod P are built by repeated squaring, so
// that T^(J*2^a) s = sum_i g_a[i] T^i s (evaluated on the device by Horner).
// The 31 never-used low bits of the oldest state word are the only part of the
// state outside P's invariant subspace; they never influence an output.
#include <cstdint>
#include <cstring>
#include <mutex>
#include <random>
#include <stdexcept>
#include <vector>

namespace fb {

namespace {

using Bits = std::vector<uint64_t>;

inline int getb(const Bits& b, int64_t i) { return int((b[size_t(i >> 6)] >> (i & 63)) & 1u); }
inline void flipb(Bits& b, int64_t i) { b[size_t(i >> 6)] ^= (uint64_t(1) << (i & 63)); }

// 64 bits of `b` starting at bit offset `off` (bits beyond the end read as 0)
inline uint64_t get64(const Bits& b, int64_t off) {
    const int64_t w = off >> 6, s = off & 63;
    const uint64_t lo = size_t(w) < b.size() ? b[size_t(w)] : 0;
    if (s == 0) return lo;
    const uint64_t hi = size_t(w + 1) < b.size() ? b[size_t(w + 1)] : 0;
    return (lo >> s) | (hi << (64 - s));
}

// dst ^= src << shift (bit shift), dst sized to hold the result
void xor_shifted(Bits& dst, const Bits& src, int64_t src_bits, int64_t shift) {
    const int64_t ws = shift >> 6, bs = shift & 63;
    const int64_t nw = (src_bits + 63) >> 6;
    for (int64_t i = 0; i < nw; ++i) {
        const uint64_t v = src[size_t(i)];
        if (!v) continue;
        if (size_t(i + ws) >= dst.size()) break;
        dst[size_t(i + ws)] ^= v << bs;
        if (bs && size_t(i + ws + 1) < dst.size()) dst[size_t(i + ws + 1)] ^= v >> (64 - bs);
    }
}

struct Poly {
    int L = 0;       // degree of P
    Bits P;          // P(x), bits 0..L
};

Poly characteristic_polynomial() {
    // output bit sequence: LSB of successive mt19937_64 outputs
    const int64_t N = 2 * 19937 + 256;
    std::mt19937_64 eng(5489u);
    Bits s(size_t((N + 63) / 64), 0);
    for (int64_t i = 0; i < N; ++i)
        if (eng() & 1u) flipb(s, i);
    // reversed sequence R_j = s_{N-1-j}: then s_{n-i} = R_{N-1-n+i}
    Bits R(s.size(), 0);
    for (int64_t j = 0; j < N; ++j)
        if (getb(s, N - 1 - j)) flipb(R, j);
    const size_t W = size_t((N + 64) / 64) + 2;
    Bits C(W, 0), B(W, 0), T;
    C[0] = B[0] = 1;
    int64_t L = 0, m = 1;
    for (int64_t n = 0; n < N; ++n) {
        // d = sum_{i=0..L} C_i s_{n-i}
        uint64_t acc = 0;
        const int64_t base = N - 1 - n;
        for (int64_t w = 0; w * 64 <= L; ++w) {
            uint64_t cw = C[size_t(w)];
            if (w * 64 + 63 > L) {
                const int64_t keep = L - w * 64 + 1;
                if (keep < 64) cw &= (uint64_t(1) << keep) - 1;
            }
            acc ^= cw & get64(R, base + w * 64);
        }
        const int d = __builtin_parityll(acc);
        if (!d) {
            ++m;
        } else if (2 * L <= n) {
            T = C;
            xor_shifted(C, B, int64_t(B.size()) * 64, m);
            L = n + 1 - L;
            B = T;
            m = 1;
        } else {
            xor_shifted(C, B, int64_t(B.size()) * 64, m);
            ++m;
        }
    }
    Poly p;
    p.L = int(L);
    p.P.assign(size_t(L / 64 + 1), 0);
    for (int64_t i = 0; i <= L; ++i)
        if (getb(C, L - i)) flipb(p.P, i);
    return p;
}

// g <- g^2 mod P  (g has < L bits)
void square_mod(const Poly& p, Bits& g) {
    const int64_t L = p.L;
    Bits sq(size_t((2 * L + 63) / 64 + 1), 0);
    for (int64_t i = 0; i < L; ++i)
        if (getb(g, i)) flipb(sq, 2 * i);
    for (int64_t d = 2 * L - 2; d >= L; --d)
        if (getb(sq, d)) xor_shifted(sq, p.P, L + 1, d - L);
    g.assign(size_t((L + 63) / 64), 0);
    for (int64_t w = 0; w < int64_t(g.size()); ++w) g[size_t(w)] = sq[size_t(w)];
    const int64_t tail = L & 63;
    if (tail) g.back() &= (uint64_t(1) << tail) - 1;
}

// g <- g * h mod P  (both < L bits)
void mul_mod(const Poly& p, Bits& g, const Bits& h) {
    const int64_t L = p.L;
    Bits pr(size_t((2 * L + 63) / 64 + 2), 0);
    for (int64_t i = 0; i < L; ++i)
        if (getb(g, i)) xor_shifted(pr, h, L, i);
    for (int64_t d = 2 * L - 2; d >= L; --d)
        if (getb(pr, d)) xor_shifted(pr, p.P, L + 1, d - L);
    g.assign(size_t((L + 63) / 64), 0);
    for (int64_t w = 0; w < int64_t(g.size()); ++w) g[size_t(w)] = pr[size_t(w)];
    const int64_t tail = L & 63;
    if (tail) g.back() &= (uint64_t(1) << tail) - 1;
}

const Poly& char_poly() {
    static std::once_flag once;
    static Poly poly;
    std::call_once(once, [] { poly = characteristic_polynomial(); });
    if (poly.L != 19937) throw std::runtime_error("mt19937_64: unexpected characteristic polynomial degree");
    return poly;
}

}  // namespace

// Jump polynomials of a 16-ary jump tree for segments of J = 156 * 2^log2_steps
// words (a whole number of the device generator's 156-word steps): level a
// holds x^(J q 16^a) mod P for q = 1..15, so segment k = q 16^a + r starts at
// T^(J q 16^a) applied to the start of segment r < 16^a.
// Returned as 32-bit coefficient groups: out[((a * 15) + q - 1) * groups + g]
// bit b is the coefficient of x^(32 g + b). Also returns the degree L.
int mt64_jump_polys(int log2_steps, int levels, std::vector<uint32_t>& out, int& groups) {
    const Poly& poly = char_poly();
    const int64_t L = poly.L;
    groups = int((L + 31) / 32);
    Bits base(size_t((L + 63) / 64) + 1, 0);
    base[0] = 1;  // x^0
    for (int e = 0; e < 156; ++e) {  // base <- x * base mod P
        uint64_t carry = 0;
        for (auto& w : base) { const uint64_t nc = w >> 63; w = (w << 1) | carry; carry = nc; }
        if (getb(base, L)) xor_shifted(base, poly.P, L + 1, 0);
    }
    base.resize(size_t((L + 63) / 64));
    for (int e = 0; e < log2_steps; ++e) square_mod(poly, base);  // x^J
    out.assign(size_t(levels) * 15 * size_t(groups), 0);
    for (int a = 0; a < levels; ++a) {
        Bits g = base;  // x^(J 16^a)
        for (int q = 1; q <= 15; ++q) {
            if (q > 1) mul_mod(poly, g, base);
            uint32_t* dst = out.data() + (size_t(a) * 15 + size_t(q - 1)) * size_t(groups);
            for (int gi = 0; gi < groups; ++gi) dst[gi] = uint32_t(g[size_t(gi / 2)] >> ((gi & 1) * 32));
        }
        if (a + 1 < levels)
            for (int e = 0; e < 4; ++e) square_mod(poly, base);  // x^(J 16^(a+1))
    }
    return int(L);
}

// std::mt19937_64 seeding (the standard's initialization recurrence).
void mt64_seed_state(uint64_t seed, uint64_t* state312) {
    state312[0] = seed;
    for (int i = 1; i < 312; ++i)
        state312[i] = 6364136223846793005ULL * (state312[i - 1] ^ (state312[i - 1] >> 62)) + uint64_t(i);
}

}  // namespace fb
