// glibc's log, restated operation for operation, for the sketch's polar
// transform.
//
// The reference draws Omega with libstdc++'s polar normal_distribution
// (dense_kernels.hpp:19-28), which calls std::log, i.e. glibc's log. On
// x86-64 hosts with FMA and AVX2 (the GPU box's host and this image) the ifunc
// resolves `log` to the FMA build of glibc's table-driven log (ARM's
// optimized-routines algorithm: 128 subintervals, a degree-6 polynomial for
// log1p(r) - r, and a degree-12 one for inputs within ~1/16 of 1). It is not
// correctly rounded (0.52 ulp), so the device evaluates the same operations
// in the same order, with the FMA contractions that build makes. The order
// below is read from `objdump -d` of that function (libm.so.6 of this image,
// the target of the `log` PLT slot); the constants are generated from the
// same library by tools/gen_glibc_log.py into glibc_log_data.h.
//
// Domain: the polar method's r2 = x*x + y*y, 0 < r2 <= 1, r2 >= 2^-106
// (u = 2c - 1 is a multiple of 2^-53 near 0), so no subnormal, negative,
// infinite or NaN input reaches it; those branches of glibc's log are not
// restated. Pinned bitwise against the host library by
// tests/cpp/glibc_log_check.cpp (CPU) and test_gpu_rng.py (device).
#pragma once
#include <cstdint>
#include <cstring>
#include <cmath>
#include "glibc_log_data.h"

namespace fb {
namespace glibc_log {

#if defined(__CUDACC__)
#define GL_HD __host__ __device__ __forceinline__
#else
#define GL_HD inline
#endif
#if defined(__CUDA_ARCH__)
#define GL_ADD(a, b) __dadd_rn((a), (b))
#define GL_SUB(a, b) __dsub_rn((a), (b))
#define GL_MUL(a, b) __dmul_rn((a), (b))
#define GL_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
// host: the including file must be compiled without FP contraction
// (-ffp-contract=off) so these stay separately rounded
#define GL_ADD(a, b) ((a) + (b))
#define GL_SUB(a, b) ((a) - (b))
#define GL_MUL(a, b) ((a) * (b))
#define GL_FMA(a, b, c) std::fma((a), (b), (c))
#endif

constexpr double kTab[256] = FB_GLIBC_LOG_TAB_INIT;
#if defined(__CUDACC__)
__device__ const double kTabDev[256] = FB_GLIBC_LOG_TAB_INIT;
#endif

GL_HD uint64_t as_u64(double x) {
#if defined(__CUDA_ARCH__)
    return uint64_t(__double_as_longlong(x));
#else
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
#endif
}
GL_HD double as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double x;
    std::memcpy(&x, &u, 8);
    return x;
#endif
}

// log(x) for 2^-1022 <= x < +inf, bitwise equal to glibc's FMA build.
GL_HD double log_polar(double x) {
    const uint64_t ix = as_u64(x);
    constexpr uint64_t LO = 0x3fee000000000000ull;   // 1 - 2^-4
    constexpr uint64_t HI = 0x3ff1090000000000ull;   // 1 + 0x1.09p-4
    if (ix - LO < HI - LO) {
        // |x - 1| small: log1p(r) = r - r^2/2 + r^3 * P(r), with r^2/2 split
        // exactly (rhi has 26 significant bits).
        if (ix == 0x3ff0000000000000ull) return 0.0;
        const double r = GL_SUB(x, 1.0);
        const double r2 = GL_MUL(r, r);
        const double r3 = GL_MUL(r, r2);
        const double p12 = GL_FMA(r2, kB3, GL_FMA(r, kB2, kB1));             // B1 + r B2 + r2 B3
        const double p45 = GL_FMA(r2, kB6, GL_FMA(r, kB5, kB4));             // B4 + r B5 + r2 B6
        double p7 = GL_FMA(r2, kB9, GL_FMA(r, kB8, kB7));                    // B7 + r B8 + r2 B9
        p7 = GL_FMA(r3, kB10, p7);                                           //  + r3 B10
        const double p = GL_FMA(GL_FMA(p7, r3, p45), r3, p12);               // y = r3 * p below
        const double t = GL_FMA(r, 0x1p27, r);                               // r + r*2^27
        const double rhi = GL_FMA(-0x1p27, r, t);                            // (r + w) - w
        const double rlo = GL_SUB(r, rhi);
        const double rh2 = GL_MUL(rhi, rhi);
        const double hi = GL_FMA(rh2, kB0, r);                               // r + rhi^2 * B0
        double lo = GL_FMA(rh2, kB0, GL_SUB(r, hi));                         // r - hi + w
        lo = GL_FMA(GL_MUL(kB0, rlo), GL_ADD(r, rhi), lo);                   // + B0 rlo (rhi + r)
        const double y = GL_FMA(p, r3, lo);
        return GL_ADD(hi, y);
    }
    // x = 2^k z, z in [0x1.6p-1, 0x1.6p0); c (near the centre of z's
    // subinterval i) carries invc = 1/c and logc = log(c).
    constexpr uint64_t OFF = 0x3fe6000000000000ull;
    const uint64_t tmp = ix - OFF;
    const int i = int((tmp >> 45) & 127);
    const int k = int(int64_t(tmp) >> 52);
    const uint64_t iz = ix - (tmp & (0xfffull << 52));
#if defined(__CUDA_ARCH__)
    const double invc = __ldg(&kTabDev[2 * i]), logc = __ldg(&kTabDev[2 * i + 1]);
#else
    const double invc = kTab[2 * i], logc = kTab[2 * i + 1];
#endif
    const double z = as_f64(iz);
    const double kd = double(k);
    const double r = GL_FMA(z, invc, -1.0);                                  // z/c - 1
    const double w = GL_FMA(kd, kLn2hi, logc);                               // k ln2hi + log c
    const double hi = GL_ADD(r, w);
    const double lo = GL_FMA(kd, kLn2lo, GL_ADD(GL_SUB(w, hi), r));          // w - hi + r + k ln2lo
    const double r2 = GL_MUL(r, r);
    const double a12 = GL_FMA(r, kA2, kA1);
    const double a34 = GL_FMA(r, kA4, kA3);
    const double q = GL_FMA(a34, r2, a12);                                   // A1 + r A2 + r2 (A3 + r A4)
    const double y = GL_FMA(GL_MUL(r, r2), q, GL_FMA(r2, kA0, lo));        // lo + r2 A0 + r^3 q
    return GL_ADD(y, hi);
}

#undef GL_HD
#undef GL_ADD
#undef GL_SUB
#undef GL_MUL
#undef GL_FMA

}  // namespace glibc_log
}  // namespace fb
