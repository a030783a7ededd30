// Host check of the sketch's log (paper_1810_06825_b200/csrc/glibc_log.cuh):
// the restatement of glibc's log must equal this host's std::log bitwise on
// inputs drawn like the polar method's r2 = x^2 + y^2 (libstdc++'s
// normal_distribution, dense_kernels.hpp:19-28), near 1 (the second
// polynomial), at every subinterval edge of the table, and on uniform bit
// patterns over [2^-106, 1]. Built with -ffp-contract=off and run by
// tests/test_host_cpu.py::test_glibc_log_restatement.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "../../paper_1810_06825_b200/csrc/glibc_log.cuh"

using fb::glibc_log::log_polar;

static double (*volatile host_log)(double) = static_cast<double (*)(double)>(std::log);

static double from_bits(uint64_t u) {
    double x;
    std::memcpy(&x, &u, 8);
    return x;
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? atol(argv[1]) : 4000000;
    long bad = 0, tested = 0, near1 = 0;
    auto check = [&](double x) {
        ++tested;
        const double a = log_polar(x), b = host_log(x);
        if (std::memcmp(&a, &b, 8) != 0) {
            if (bad < 10) std::printf("mismatch x=%a glibc=%a restated=%a\n", x, b, a);
            ++bad;
        }
        if (x >= 1 - 0x1p-4 && x < 1 + 0x1.09p-4) ++near1;
    };
    std::mt19937_64 g(20181016);
    for (long t = 0; t < n; ++t) {
        // polar r2 from two canonical draws (generate_canonical<double, 53>
        // of a 64-bit engine: one word times 2^-64)
        const double u = 2.0 * (double(g()) * 0x1p-64) - 1.0, v = 2.0 * (double(g()) * 0x1p-64) - 1.0;
        const double x = u * u + v * v;
        if (x > 1.0 || x == 0.0) continue;
        check(x);
    }
    for (long t = 0; t < n / 4; ++t) {   // uniform bit patterns in [2^-106, 1]
        const uint64_t lo = 0x3950000000000000ull, hi = 0x3ff0000000000000ull;
        check(from_bits(lo + g() % (hi - lo + 1)));
    }
    for (long t = 0; t < n / 4; ++t)     // dense near 1: [1 - 2^-4, 1]
        check(1.0 - double(g() >> 11) * 0x1p-57);
    for (int e = -106; e <= 0; ++e)      // every subinterval edge, each binade
        for (uint64_t i = 0; i <= 128; ++i) {
            const uint64_t b = 0x3fe6000000000000ull + (i << 45);
            for (int d = -2; d <= 2; ++d) {
                const double x = std::ldexp(from_bits(b + uint64_t(int64_t(d))), e);
                if (x > 0 && x <= 1.0) check(x);
            }
        }
    check(1.0);
    std::printf("tested %ld near1 %ld bad %ld\n", tested, near1, bad);
    return bad == 0 ? 0 : 1;
}
