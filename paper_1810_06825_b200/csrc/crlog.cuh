// Correctly rounded natural log on (0, 1] for the polar method of the Omega
// stream (rng.cu k_emit; libstdc++'s normal_distribution calls std::log on
// r2 = x^2 + y^2). Shared by the device generator and the host checks
// (tests/cpp/log_check.cpp), so every operation is an explicitly rounded
// double op (no contraction on either side).
//
//  - cr_log: double-double evaluation of 2 atanh((m-1)/(m+1)), ~2^-73
//    relative, one rounding at the end (the slow, robust path).
//  - fast_log: table-driven log x = k ln2 - log(c_i) + log1p(z c_i - 1) with
//    z c_i - 1 exact, ~2^-68 relative; when the result lies within that bound
//    of a rounding midpoint (probability ~2^-14) it defers to cr_log (Ziv).
#pragma once

#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define FB_HD __host__ __device__ __forceinline__
#else
#define FB_HD inline
#endif

namespace fb {
namespace crlog {

#ifdef __CUDA_ARCH__
FB_HD double add(double a, double b) { return __dadd_rn(a, b); }
FB_HD double sub(double a, double b) { return __dsub_rn(a, b); }
FB_HD double mul(double a, double b) { return __dmul_rn(a, b); }
FB_HD double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
FB_HD double div_(double a, double b) { return __ddiv_rn(a, b); }
FB_HD uint64_t bits(double x) { return static_cast<uint64_t>(__double_as_longlong(x)); }
FB_HD double from_bits(uint64_t u) { return __longlong_as_double(static_cast<long long>(u)); }
#else
// host: compiled with -ffp-contract=off, so these are single IEEE operations
FB_HD double add(double a, double b) { return a + b; }
FB_HD double sub(double a, double b) { return a - b; }
FB_HD double mul(double a, double b) { return a * b; }
FB_HD double fma_(double a, double b, double c) { return __builtin_fma(a, b, c); }
FB_HD double div_(double a, double b) { return a / b; }
FB_HD uint64_t bits(double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; }
FB_HD double from_bits(uint64_t u) { double x; std::memcpy(&x, &u, 8); return x; }
#endif

struct dd { double hi, lo; };
FB_HD dd two_sum(double a, double b) {
    const double s = add(a, b);
    const double bb = sub(s, a);
    return {s, add(sub(a, sub(s, bb)), sub(b, bb))};
}
FB_HD dd fast_two_sum(double a, double b) {
    const double s = add(a, b);
    return {s, sub(b, sub(s, a))};
}
FB_HD dd two_prod(double a, double b) {
    const double p = mul(a, b);
    return {p, fma_(a, b, -p)};
}
FB_HD dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    s.lo = add(s.lo, add(a.lo, b.lo));
    return fast_two_sum(s.hi, s.lo);
}
FB_HD dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = fma_(a.hi, b.lo, p.lo);
    p.lo = fma_(a.lo, b.hi, p.lo);
    return fast_two_sum(p.hi, p.lo);
}

FB_HD double cr_log(double x) {
    if (x == 1.0) return 0.0;
    // x = m 2^e, m in [1/sqrt2, sqrt2) (x is normal here: r2 >= 2^-128)
    int e = int((bits(x) >> 52) & 0x7ff) - 1022;
    double m = from_bits((bits(x) & 0x000fffffffffffffull) | 0x3fe0000000000000ull);  // [0.5, 1)
    if (m < 0.70710678118654752440) { m = mul(m, 2.0); e -= 1; }
    // log m = 2 atanh(s), s = (m - 1) / (m + 1), |s| < 0.172
    const double num = sub(m, 1.0);  // exact (Sterbenz)
    const dd den = two_sum(m, 1.0);
    // s = num / den to ~2^-104: one division, residual by FMA
    const double rcp = div_(1.0, den.hi);
    const double q1 = mul(num, rcp);
    const double rem = sub(fma_(-q1, den.hi, num), mul(q1, den.lo));
    const double q2 = mul(rem, rcp);
    const dd s = fast_two_sum(q1, q2);
    const dd s2 = dd_mul(s, s);
    // tail sum_{k>=4} s2^(k-4) / (2k+1) in double (relative weight < 1e-6)
    double t = 1.0 / 45.0;
    for (int k = 21; k >= 4; --k) t = fma_(t, s2.hi, 1.0 / double(2 * k + 1));
    // 1 + s2/3 + s2^2/5 + s2^3/7 + s2^4 t, in double-double
    const dd c3{0x1.5555555555555p-2, 0x1.5555555555555p-56};   // 1/3
    const dd c5{0x1.999999999999ap-3, -0x1.999999999999ap-57};  // 1/5
    const dd c7{0x1.2492492492492p-3, 0x1.2492492492492p-57};   // 1/7
    dd p{t, 0.0};
    p = dd_add(dd_mul(p, s2), c7);
    p = dd_add(dd_mul(p, s2), c5);
    p = dd_add(dd_mul(p, s2), c3);
    p = dd_add(dd_mul(p, s2), {1.0, 0.0});
    dd lm = dd_mul(p, s);
    lm.hi = mul(lm.hi, 2.0);
    lm.lo = mul(lm.lo, 2.0);
    const dd ln2{0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
    const dd el = dd_mul({double(e), 0.0}, ln2);
    const dd r = dd_add(el, lm);
    return add(r.hi, r.lo);
}

// ---- table-driven fast path ------------------------------------------------
// z in [0.6875, 1.375) is split into 256 subintervals by the top 8 mantissa
// bits of (bits(x) - bits(0.6875)); c_i ~ 1/center_i with 9 significant
// bits so that r = z c_i - 1 is exact in one FMA (|r| < 2^-8); the two
// subintervals touching 1 use c = 1 (no cancellation for x -> 1).
constexpr int kLogTab = 256;
constexpr uint64_t kLogOff = 0x3fe6000000000000ull;  // 0.6875
struct LogEntry { double c, lhi, llo; };              // -log(c) = lhi + llo

FB_HD double fast_log(double x, const LogEntry* tab) {
    if (x == 1.0) return 0.0;
    const uint64_t ix = bits(x);
    const uint64_t tmp = ix - kLogOff;
    const int i = int((tmp >> 44) & 255u);
    const int k = int(static_cast<int64_t>(tmp) >> 52);
    const double z = from_bits(ix - (tmp & (0xfffull << 52)));
    const LogEntry t = tab[i];
    const double r = fma_(z, t.c, -1.0);  // exact
    // log1p(r) = r - r^2/2 + r^3 (1/3 - r/4 + ... - r^7/10)
    const dd r2 = two_prod(r, r);
    double p = -0.1;
    p = fma_(p, r, 1.0 / 9.0);
    p = fma_(p, r, -0.125);
    p = fma_(p, r, 1.0 / 7.0);
    p = fma_(p, r, -1.0 / 6.0);
    p = fma_(p, r, 0.2);
    p = fma_(p, r, -0.25);
    // r^3/3 carries 2^-18 of the value: its leading part in double-double
    const dd r3 = dd_mul(r2, {r, 0.0});
    const dd c3{0x1.5555555555555p-2, 0x1.5555555555555p-56};
    const dd t3 = dd_mul(r3, c3);
    const double tail = mul(mul(r3.hi, r), p);  // r^4 (p)
    // k ln2 + lhi + r - r2/2 (big parts, exact sums) ...
    const double ln2hi = 0x1.62e42fefa3800p-1, ln2lo = 0x1.ef35793c76730p-45;
    const dd a = two_sum(mul(double(k), ln2hi), t.lhi);  // k ln2hi exact (|k| < 2^11)
    const dd b = two_sum(a.hi, r);
    const dd c = two_sum(b.hi, mul(-0.5, r2.hi));
    // ... and the small parts in double
    double lo = add(mul(double(k), ln2lo), t.llo);
    lo = add(lo, a.lo);
    lo = add(lo, b.lo);
    lo = add(lo, c.lo);
    lo = add(lo, mul(-0.5, r2.lo));
    lo = add(lo, t3.hi);
    lo = add(lo, add(t3.lo, tail));
    const dd res = fast_two_sum(c.hi, lo);
    // Ziv: res.hi = RN(res.hi + res.lo); the true value rounds to res.hi unless
    // it is within the error bound of the midpoint ulp/2 away from res.hi
    const uint64_t hb = bits(res.hi) & 0x7fffffffffffffffull;
    const double half_ulp = from_bits(((hb >> 52) - 53) << 52);
    const double err = mul(from_bits(hb), 0x1.0p-66);
    const double lo_abs = from_bits(bits(res.lo) & 0x7fffffffffffffffull);
    if (sub(half_ulp, lo_abs) > err && (hb & 0x000fffffffffffffull) != 0) return res.hi;
    return cr_log(x);
}

// Host: the table, -log(c_i) to ~2^-100 by the atanh series in double-double.
inline dd dd_div_exact(double a, double b) {  // a / b to ~2^-106
    const double q1 = div_(a, b);
    const double r = fma_(-q1, b, a);
    return fast_two_sum(q1, div_(r, b));
}
inline dd log_dd(double c) {  // c in [0.5, 2], c - 1 and c + 1 exact
    const dd s = dd_div_exact(sub(c, 1.0), add(c, 1.0));
    const dd s2 = dd_mul(s, s);
    dd acc{0.0, 0.0};
    for (int k = 40; k >= 0; --k) acc = dd_add(dd_mul(acc, s2), dd_div_exact(1.0, double(2 * k + 1)));
    dd r = dd_mul(acc, s);
    return {mul(r.hi, 2.0), mul(r.lo, 2.0)};
}
inline void build_log_table(LogEntry* tab) {
    for (int i = 0; i < kLogTab; ++i) {
        const double zlo = from_bits(kLogOff + (uint64_t(i) << 44));
        const double zhi = from_bits(kLogOff + (uint64_t(i + 1) << 44));
        double c = 1.0;
        if (!(zhi == 1.0 || zlo == 1.0)) {
            const double inv = 1.0 / (0.5 * (zlo + zhi));
            int e = int((bits(inv) >> 52) & 0x7ff) - 1023;  // inv in [2^e, 2^(e+1))
            const double scale = from_bits(uint64_t(1023 + 8 - e) << 52);
            const double unscale = from_bits(uint64_t(1023 - 8 + e) << 52);
            c = __builtin_nearbyint(inv * scale) * unscale;  // 9 significant bits
        }
        const dd l = log_dd(c);
        tab[i] = {c, -l.hi, -l.lo};
    }
}

}  // namespace crlog
}  // namespace fb
