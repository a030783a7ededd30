// Device Omega generator (placeholder until the bit-compatible MT19937-64 +
// polar generator lands; callers pass FRPCA_FLAG_HOST_OMEGA meanwhile).
#include "internal.cuh"

namespace fb {

void gaussian_stream_device(Ctx&, uint64_t, int64_t, double*) {
    throw InvalidArgument("frpca_b200: device Omega generator not available in this build; "
                          "set FRPCA_FLAG_HOST_OMEGA");
}

}  // namespace fb
