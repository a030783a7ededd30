// Collectives of the sharded path. The only exchange steps of
// frPCA are sums: the n x l A^T*Y partials (frpcat, row-block sharding), the
// m x l A*X partials (frpca, column-block sharding) and the l x l Gram
// partials. Everything else is replicated (identical on every rank) or
// rank-local. Reference loops these replace: randsvd.hpp:255-258, :307-310
// (the reference itself is single-process).
//
// Two implementations of the same in-place sum over ranks:
//  - NcclColl: NCCL over NVLink 5 / NVSwitch, one communicator per rank,
//    from ncclCommInitRank (one process per GPU) or ncclCommInitAll (one
//    process driving several GPUs, frpca_group_create). Stream-ordered.
//  - Loopback: ranks that are contexts of ONE process, possibly on the same
//    device (testing the sharded path on a single GPU, where NCCL refuses a
//    duplicate device). Host-staged: each rank finishes its stream, the ranks
//    meet at a host barrier, rank 0 adds the buffers in rank order (fixed,
//    deterministic), and every rank copies the sum back. No kernel ever waits
//    on another rank's kernel; the ranks only meet on the host.
//
// NCCL is resolved at run time (dlopen) and only for world > 1: the process
// may already hold PyTorch's bundled libnccl.so.2 (a newer release with the
// same soname), and linking the system copy eagerly would shadow it.
#include <dlfcn.h>

#include <condition_variable>
#include <mutex>
#include <nccl.h>

#include "driver.cuh"

namespace fb {
namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
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
        n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
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

// Chunks keep every call within NCCL's count type and let a caller overlap
// them with the producing kernels (allreduce_sum_async).
constexpr int64_t kNcclChunk = int64_t(1) << 28;

struct NcclColl final : Collective {
    ncclComm_t comm = nullptr;
    explicit NcclColl(ncclComm_t c) : comm(c) {}
    ~NcclColl() override {
        if (comm) nccl().CommDestroy(comm);
    }
    void allreduce_sum(Ctx& c, double* x, int64_t count, cudaStream_t s) override {
        for (int64_t off = 0; off < count; off += kNcclChunk) {
            const size_t n = size_t(std::min(kNcclChunk, count - off));
            check(nccl().AllReduce(x + off, x + off, n, ncclFloat64, ncclSum, comm, s), "ncclAllReduce");
        }
        (void)c;
    }
};

__global__ void k_add_into(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        dst[i] += src[i];
}

}  // namespace

// Host-staged sum over the contexts of one process (see the header comment).
struct LoopbackGroup {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t generation = 0;
    std::vector<double*> buf;
    std::vector<int> dev;
    std::vector<int64_t> count;
    bool failed = false;
    explicit LoopbackGroup(int w) : world(w), buf(size_t(w)), dev(size_t(w)), count(size_t(w)) {}

    // all ranks arrive; returns false when a rank reported a failure
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const int64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen || failed; });
        }
        return !failed;
    }
    // a rank that cannot reach the next exchange releases the others
    void fail() {
        std::lock_guard<std::mutex> lk(mu);
        failed = true;
        cv.notify_all();
    }
};

void loopback_fail(LoopbackGroup& g) { g.fail(); }

// called with every rank idle (the start of a group run)
void loopback_reset(LoopbackGroup& g) {
    std::lock_guard<std::mutex> lk(g.mu);
    g.failed = false;
    g.arrived = 0;
}

namespace {

struct LoopbackColl final : Collective {
    std::shared_ptr<LoopbackGroup> g;
    int rank;
    LoopbackColl(std::shared_ptr<LoopbackGroup> grp, int r) : g(std::move(grp)), rank(r) {}
    void allreduce_sum(Ctx& c, double* x, int64_t count, cudaStream_t s) override {
        FB_CUDA(cudaStreamSynchronize(s));
        {
            std::lock_guard<std::mutex> lk(g->mu);
            g->buf[size_t(rank)] = x;
            g->dev[size_t(rank)] = c.device;
            g->count[size_t(rank)] = count;
        }
        if (!g->barrier()) throw CudaError("loopback allreduce: another rank failed");
        std::string err;
        if (rank == 0) {
            try {
                for (int r = 1; r < g->world; ++r)
                    if (g->count[size_t(r)] != count) throw CudaError("loopback allreduce: ranks disagree on the count");
                // rank 0 adds the other ranks' buffers in rank order on its
                // own stream (peer copies when the ranks sit on other devices)
                DBuf<double> tmp;
                for (int r = 1; r < g->world; ++r) {
                    const double* src = g->buf[size_t(r)];
                    if (g->dev[size_t(r)] != c.device) {
                        if (!tmp.get()) tmp.alloc(size_t(count), s);
                        FB_CUDA(cudaMemcpyPeerAsync(tmp.get(), c.device, src, g->dev[size_t(r)],
                                                    sizeof(double) * size_t(count), s));
                        src = tmp.get();
                    }
                    const int grid = int(std::min<int64_t>(4 * c.num_sms, (count + 255) / 256));
                    k_add_into<<<std::max(grid, 1), 256, 0, s>>>(x, src, count);
                    FB_LAUNCH_CHECK();
                }
                FB_CUDA(cudaStreamSynchronize(s));
            } catch (const std::exception& e) {
                err = e.what();
                g->fail();
            }
        }
        if (!g->barrier()) throw CudaError(err.empty() ? "loopback allreduce: rank 0 failed" : err);
        if (rank != 0) {
            FB_CUDA(cudaMemcpyPeerAsync(x, c.device, g->buf[0], g->dev[0], sizeof(double) * size_t(count), s));
            FB_CUDA(cudaStreamSynchronize(s));
        }
        if (!g->barrier()) throw CudaError("loopback allreduce: another rank failed");  // rank 0's buffer is free again
    }
};

}  // namespace

std::shared_ptr<LoopbackGroup> loopback_group(int world) { return std::make_shared<LoopbackGroup>(world); }

void comm_attach_loopback(Ctx& c, const std::shared_ptr<LoopbackGroup>& g, int rank) {
    c.rank = rank;
    c.world = g->world;
    c.coll = std::make_shared<LoopbackColl>(g, rank);
}

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
    c.coll = std::make_shared<NcclColl>(comm);
}

void comm_init_all(std::vector<Ctx*>& ctxs, const std::vector<int>& devices) {
    const int n = int(ctxs.size());
    if (!nccl().CommInitAll) throw CudaError("frpca_b200: ncclCommInitAll not available");
    std::vector<ncclComm_t> comms(static_cast<size_t>(n));
    check(nccl().CommInitAll(comms.data(), n, devices.data()), "ncclCommInitAll");
    for (int r = 0; r < n; ++r) {
        ctxs[size_t(r)]->rank = r;
        ctxs[size_t(r)]->world = n;
        ctxs[size_t(r)]->coll = std::make_shared<NcclColl>(comms[size_t(r)]);
    }
}

void comm_destroy(Ctx& c) { c.coll.reset(); }

void allreduce_sum(Ctx& c, double* x, int64_t count) {
    if (c.world <= 1 || count == 0) return;
    Prof prof(c, "allreduce", 8.0 * count * 2.0 * (c.world - 1) / c.world, double(count));
    c.coll->allreduce_sum(c, x, count, c.stream);
}

}  // namespace fb
