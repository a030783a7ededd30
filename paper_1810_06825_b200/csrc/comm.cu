// Collectives of the sharded path: one process per GPU, NCCL over
// NVLink 5 / NVSwitch. The only exchange steps of frPCA are sums: the n x l
// A^T*Y partials (frpcat, row-block sharding), the m x l A*X partials (frpca,
// column-block sharding) and the l x l Gram partials. Everything else is
// replicated (identical on every rank) or rank-local.
//
// NCCL is resolved at run time (dlopen) and only for world > 1: the process
// may already hold PyTorch's bundled libnccl.so.2 (a newer release with the
// same soname), and linking the system copy eagerly would shadow it.
#include <dlfcn.h>

#include <mutex>
#include <nccl.h>

#include "driver.cuh"

namespace fb {
namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* candidates[] = {
            "libnccl.so.2",  // already loaded (e.g. by torch) or on the search path
            "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
            "/usr/lib/x86_64-linux-gnu/libnccl.so.2",
        };
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        for (const char* c : candidates) {
            if (h) break;
            h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) return;
        n.h = h;
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(dlsym(h, "ncclAllReduce"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!n.h || !n.GetUniqueId || !n.CommInitRank || !n.AllReduce || !n.CommDestroy)
        throw CudaError("frpca_b200: libnccl.so.2 could not be loaded");
    return n;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw CudaError(std::string(what) + ": " +
                        (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error"));
}

}  // namespace

void comm_unique_id(void* out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

void comm_init(Ctx& c, int rank, int world, const void* id128) {
    c.rank = rank;
    c.world = world;
    if (world <= 1) return;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    check(nccl().CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
    c.comm = comm;
}

void comm_destroy(Ctx& c) {
    if (c.comm) nccl().CommDestroy(c.comm);
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
        check(nccl().AllReduce(x + off, x + off, n, ncclFloat64, ncclSum, c.comm, c.stream),
              "ncclAllReduce");
    }
}

}  // namespace fb
