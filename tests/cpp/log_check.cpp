// Host check of the Omega generator's correctly rounded log
// (paper_1810_06825_b200/csrc/crlog.cuh): fast_log (table + Ziv fallback) and
// cr_log against an independent quad-precision reference, on inputs drawn like
// the polar method's r2 plus edge cases. Built and run by
// tests/test_host_cpu.py::test_correctly_rounded_log.
#include <quadmath.h>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_1810_06825_b200/csrc/crlog.cuh"

using namespace fb::crlog;

static double ref_log(double x) { return (double)logq((__float128)x); }

int main(int argc, char** argv) {
    const long n = argc > 1 ? atol(argv[1]) : 2000000;
    std::vector<LogEntry> tab(kLogTab);
    build_log_table(tab.data());
    // r = z c - 1 exact and |r| < 2^-8 at both ends of every subinterval
    long bad_tab = 0;
    for (int i = 0; i < kLogTab; ++i) {
        for (int end = 0; end < 2; ++end) {
            const double z = from_bits(kLogOff + ((uint64_t(i) + end) << 44)) * (end ? (1 - 0x1p-53) : 1.0);
            const long double exact = (long double)z * (long double)tab[i].c - 1.0L;
            const double r = fma_(z, tab[i].c, -1.0);
            if ((long double)r != exact || __builtin_fabs(r) >= 0x1p-8) ++bad_tab;
        }
    }
    std::mt19937_64 g(12345);
    long bad_fast = 0, bad_cr = 0, fallback = 0, diff = 0;
    for (long t = 0; t < n; ++t) {
        double x;
        const int kind = int(t % 8);
        if (kind < 5) {  // polar r2 = x^2 + y^2 from two 64-bit draws
            const double u = 2.0 * ((double)g() * 0x1p-64) - 1.0, v = 2.0 * ((double)g() * 0x1p-64) - 1.0;
            x = u * u + v * v;
            if (x > 1.0 || x == 0.0) continue;
        } else if (kind == 5) {  // near 1
            x = 1.0 - (double)(g() >> 11) * 0x1p-60;
        } else if (kind == 6) {  // tiny
            x = (double)((g() >> 11) | 1) * 0x1p-53 * 0x1p-60;
        } else {  // subinterval edges
            const int i = int(g() & 255);
            x = from_bits(kLogOff + (uint64_t(i) << 44) + (g() & 3) - 1) * 0.5;
        }
        const double f = fast_log(x, tab.data()), c = cr_log(x), r = ref_log(x);
        bad_fast += f != r;
        bad_cr += c != r;
        diff += f != c;
        (void)fallback;
    }
    printf("table_bad %ld fast_bad %ld cr_bad %ld fast_vs_cr %ld of %ld\n", bad_tab, bad_fast, bad_cr, diff, n);
    return (bad_tab || bad_fast) ? 1 : 0;
}
