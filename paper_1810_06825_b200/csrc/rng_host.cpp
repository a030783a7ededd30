// Host Omega generator: dense_kernels.hpp:19-28 verbatim in semantics —
// std::mt19937_64(seed) + libstdc++ std::normal_distribution<double>(0, 1)
// (Marsaglia polar with a cached second value), stream order. Compiled by g++
// with -O3 -ffp-contract=off and no -march (no FMA), the arithmetic of the
// reference's own x86-64 build. Used when FRPCA_FLAG_HOST_OMEGA is set; the
// default path draws the same stream on the device (rng.cu).
#include <cstdint>
#include <random>

namespace fb {

void gaussian_stream_host(uint64_t seed, int64_t count, double* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> normal(0.0, 1.0);
    for (int64_t i = 0; i < count; ++i) out[i] = normal(rng);
}

}  // namespace fb
