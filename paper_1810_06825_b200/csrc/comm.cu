// Collectives of the sharded path: one process per GPU, NCCL over
// NVLink 5 / NVSwitch. The only exchange steps of frPCA are sums: the n x l
// A^T*Y partials (frpcat, row-block sharding), the m x l A*X partials (frpca,
// column-block sharding) and the l x l Gram partials. Everything else is
// replicated (identical on every rank) or rank-local.
#include <nccl.h>

#include "driver.cuh"

namespace fb {

#define FB_NCCL(expr)                                                                \
    do {                                                                             \
        ncclResult_t _r = (expr);                                                    \
        if (_r != ncclSuccess)                                                       \
            throw CudaError(std::string(#expr) + ": " + ncclGetErrorString(_r));     \
    } while (0)

void comm_unique_id(void* out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    FB_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
}

void comm_init(Ctx& c, int rank, int world, const void* id128) {
    c.rank = rank;
    c.world = world;
    if (world <= 1) return;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    FB_NCCL(ncclCommInitRank(&comm, world, id, rank));
    c.comm = comm;
}

void comm_destroy(Ctx& c) {
    if (c.comm) ncclCommDestroy(c.comm);
    c.comm = nullptr;
}

// Chunked so very large partials (e.g. 32 GB) stay within NCCL's count type
// and so a later version can overlap chunks with the producing SpMM.
void allreduce_sum(Ctx& c, double* x, int64_t count) {
    if (c.world <= 1 || count == 0) return;
    Prof prof(c, "allreduce", 8.0 * count * 2.0 * (c.world - 1) / c.world, double(count));
    const int64_t chunk = int64_t(1) << 28;
    for (int64_t off = 0; off < count; off += chunk) {
        const size_t n = size_t(std::min(chunk, count - off));
        FB_NCCL(ncclAllReduce(x + off, x + off, n, ncclFloat64, ncclSum, c.comm, c.stream));
    }
}

}  // namespace fb
