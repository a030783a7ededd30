#include <chrono>
// extern "C" boundary (include/frpca_b200.h). Exceptions never cross it:
// each entry point maps fb::InvalidArgument -> 2, fb::NumericalError -> 4,
// CUDA/NCCL/cuSOLVER failures -> 5 and keeps the message for
// frpca_last_error(), which the C++ drop-in rethrows as the reference's
// std::invalid_argument / frpca::NumericalError.
#include <algorithm>
#include <cstring>
#include <string>

#include <exception>
#include <thread>

#include "driver.cuh"

using namespace fb;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return FRPCA_OK;
    } catch (const InvalidArgument& e) {
        g_err = e.what();
        return FRPCA_ERR_INVALID;
    } catch (const NumericalError& e) {
        g_err = e.what();
        return FRPCA_ERR_NUMERICAL;
    } catch (const IoError& e) {
        g_err = e.what();
        return FRPCA_ERR_IO;
    } catch (const CudaError& e) {
        g_err = e.what();
        return FRPCA_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        g_err = "frpca_b200: host allocation failed";
        return FRPCA_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FRPCA_ERR_CUDA;
    }
}

void check_ctx(const frpca_ctx* c) { require(c != nullptr, "frpca_b200: null context"); }

}  // namespace

struct frpca_ctx : fb::Ctx {};
struct frpca_dmat : fb::DMat {};
// Single-process multi-GPU: one context (rank) per listed device.
struct frpca_group {
    std::vector<frpca_ctx*> ctx;
    std::vector<int> devices;
    std::shared_ptr<fb::LoopbackGroup> loop;  // host-staged collective (a device listed twice)
    int comm = 0;                             // FRPCA_COMM_NCCL / FRPCA_COMM_LOOPBACK
};

namespace fb {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

cudaEvent_t Ctx::get_event() {
    if (!event_pool.empty()) {
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    FB_CUDA(cudaEventCreate(&e));
    return e;
}

void Ctx::flush_profile() {
    if (pending.empty()) return;
    FB_CUDA(cudaStreamSynchronize(stream));
    for (auto& p : pending) {
        float ms = 0.f;
        FB_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        ProfAgg& g = agg[p.name];
        g.launches += 1;
        g.ms += ms;
        g.bytes += p.bytes;
        g.flops += p.flops;
        event_pool.push_back(p.a);
        event_pool.push_back(p.b);
    }
    pending.clear();
}

Prof::Prof(Ctx& ctx, const char* name, double bytes, double flops) : c(ctx) {
    if (!c.prof) return;
    Ctx::Pending p;
    p.name = name;
    p.a = c.get_event();
    p.b = c.get_event();
    p.bytes = bytes;
    p.flops = flops;
    cudaEventRecord(p.a, c.stream);
    idx = c.pending.size();
    c.pending.push_back(p);
}

Prof::~Prof() {
    if (idx != size_t(-1) && idx < c.pending.size()) cudaEventRecord(c.pending[idx].b, c.stream);
}

}  // namespace fb

namespace {

// host column-major (rows x cols, ld) -> device row-major rows x cols
void upload_colmajor(Ctx& c, const double* h, int64_t rows, int64_t cols, int64_t ld, double* d_rm) {
    DBuf<double> t(size_t(rows * cols), c.stream);
    if (ld == rows) {
        FB_CUDA(cudaMemcpyAsync(t.get(), h, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, c.stream));
    } else {
        FB_CUDA(cudaMemcpy2DAsync(t.get(), sizeof(double) * rows, h, sizeof(double) * ld,
                                  sizeof(double) * rows, cols, cudaMemcpyHostToDevice, c.stream));
    }
    transpose_device(c, t.get(), cols, rows, d_rm);
}

// device row-major rows x cols -> host column-major
void download_colmajor(Ctx& c, const double* d_rm, int64_t rows, int64_t cols, double* h) {
    DBuf<double> t(size_t(rows * cols), c.stream);
    transpose_device(c, d_rm, rows, cols, t.get());
    FB_CUDA(cudaMemcpyAsync(h, t.get(), sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, c.stream));
    FB_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace

extern "C" {

const char* frpca_last_error(void) { return g_err.c_str(); }
int frpca_version(void) { return 10000; }

int frpca_ctx_create(int device, frpca_ctx** out) {
    return guarded([&] {
        require(out != nullptr, "frpca_ctx_create: null output");
        FB_CUDA(cudaSetDevice(device));
        auto* c = new frpca_ctx;
        c->device = device;
        try {
            FB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            if (cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS)
                throw CudaError("cusolverDnCreate failed");
            cusolverDnSetStream(c->solver, c->stream);
            FB_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
            // keep freed stream-ordered allocations pooled between calls
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
                uint64_t thr = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int frpca_nccl_unique_id(void* out128) {
    return guarded([&] { comm_unique_id(out128); });
}

int frpca_ctx_create_dist(int device, int rank, int world, const void* nccl_id128, frpca_ctx** out) {
    return guarded([&] {
        require(world >= 1 && rank >= 0 && rank < world, "frpca_ctx_create_dist: bad rank/world");
        int st = frpca_ctx_create(device, out);
        if (st != FRPCA_OK) throw CudaError(g_err);
        comm_init(**out, rank, world, nccl_id128);
    });
}

int frpca_group_create(const int* devices, int ndev, int comm, frpca_group** out) {
    return guarded([&] {
        require(devices != nullptr && ndev >= 1 && out != nullptr, "frpca_group_create: bad arguments");
        require(comm == FRPCA_COMM_AUTO || comm == FRPCA_COMM_NCCL || comm == FRPCA_COMM_LOOPBACK,
                "frpca_group_create: unknown collective");
        std::vector<int> dv(devices, devices + ndev);
        std::vector<int> sorted = dv;
        std::sort(sorted.begin(), sorted.end());
        const bool dup = std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end();
        require(!(dup && comm == FRPCA_COMM_NCCL), "frpca_group_create: NCCL needs distinct devices");
        const int kind = (comm == FRPCA_COMM_LOOPBACK || (comm == FRPCA_COMM_AUTO && dup)) ? FRPCA_COMM_LOOPBACK
                                                                                          : FRPCA_COMM_NCCL;
        auto g = std::make_unique<frpca_group>();
        g->devices = dv;
        g->comm = kind;
        try {
            for (int r = 0; r < ndev; ++r) {
                frpca_ctx* c = nullptr;
                if (frpca_ctx_create(dv[size_t(r)], &c) != FRPCA_OK) throw CudaError(g_err);
                g->ctx.push_back(c);
            }
            if (ndev > 1) {
                if (kind == FRPCA_COMM_LOOPBACK) {
                    g->loop = loopback_group(ndev);
                    for (int r = 0; r < ndev; ++r) comm_attach_loopback(*g->ctx[size_t(r)], g->loop, r);
                } else {
                    std::vector<Ctx*> cs(g->ctx.begin(), g->ctx.end());
                    comm_init_all(cs, dv);
                }
            }
        } catch (...) {
            for (auto* c : g->ctx) frpca_ctx_destroy(c);
            throw;
        }
        *out = g.release();
    });
}

int frpca_group_size(const frpca_group* g, int* n) {
    return guarded([&] {
        require(g != nullptr && n != nullptr, "frpca_group_size: null argument");
        *n = int(g->ctx.size());
    });
}

int frpca_group_ctx(frpca_group* g, int rank, frpca_ctx** out) {
    return guarded([&] {
        require(g != nullptr && out != nullptr, "frpca_group_ctx: null argument");
        require(rank >= 0 && rank < int(g->ctx.size()), "frpca_group_ctx: rank out of range");
        *out = g->ctx[size_t(rank)];
    });
}

int frpca_group_destroy(frpca_group* g) {
    return guarded([&] {
        if (!g) return;
        for (auto* c : g->ctx) frpca_ctx_destroy(c);
        delete g;
    });
}

int frpca_shard_cuts(int64_t rows, int64_t cols, const int64_t* row_ptr, const int64_t* col_idx, int32_t col_shard,
                     int32_t world, int64_t* cuts) {
    return guarded([&] {
        require(rows >= 0 && cols >= 0 && row_ptr != nullptr && cuts != nullptr, "frpca_shard_cuts: bad arguments");
        require(!col_shard || row_ptr[rows] == 0 || col_idx != nullptr, "frpca_shard_cuts: bad arguments");
        shard_cuts(rows, cols, row_ptr, col_idx, col_shard, world, cuts);
    });
}

int frpca_shard_cols_count(int64_t rows, const int64_t* row_ptr, const int64_t* col_idx, int64_t c0, int64_t c1,
                           int64_t* nnz_local) {
    return guarded([&] {
        require(row_ptr != nullptr && nnz_local != nullptr && c0 <= c1, "frpca_shard_cols: bad arguments");
        int64_t t = 0;
        for (int64_t i = 0; i < rows; ++i) {
            const int64_t* a = col_idx + row_ptr[i];
            const int64_t* b = col_idx + row_ptr[i + 1];
            t += int64_t(std::lower_bound(a, b, c1) - std::lower_bound(a, b, c0));
        }
        *nnz_local = t;
    });
}

int frpca_shard_cols(int64_t rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values, int64_t c0,
                     int64_t c1, int64_t* l_row_ptr, int64_t* l_col_idx, double* l_values) {
    return guarded([&] {
        require(row_ptr != nullptr && l_row_ptr != nullptr && c0 <= c1, "frpca_shard_cols: bad arguments");
        std::vector<int64_t> lrp, lci;
        std::vector<double> lva;
        shard_extract_cols(rows, row_ptr, col_idx, values, c0, c1, lrp, lci, lva);
        std::memcpy(l_row_ptr, lrp.data(), sizeof(int64_t) * lrp.size());
        if (!lci.empty()) {
            std::memcpy(l_col_idx, lci.data(), sizeof(int64_t) * lci.size());
            std::memcpy(l_values, lva.data(), sizeof(double) * lva.size());
        }
    });
}

int frpca_ctx_destroy(frpca_ctx* c) {
    return guarded([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        comm_destroy(*c);
        for (auto& p : c->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
        for (auto e : c->event_pool) cudaEventDestroy(e);
        if (c->timer_a) cudaEventDestroy(c->timer_a);
        if (c->timer_b) cudaEventDestroy(c->timer_b);
        if (c->solver) cusolverDnDestroy(c->solver);
        for (auto& b : c->slots) b.release();
        if (c->side) {
            for (auto& b : c->side->slots) b.release();
            c->side->omega_stage.release();
            c->side->dflag.release();
            cudaStreamSynchronize(c->side->stream);
            cudaStreamDestroy(c->side->stream);
            c->side.reset();
        }
        c->omega_stage.release();  // stream-ordered frees before the stream goes
        if (c->tside) {
            cudaStreamSynchronize(c->tside->stream);
            cudaStreamDestroy(c->tside->stream);
            c->tside.reset();
        }
        c->dflag.release();
        c->wcount.release();
        if (c->copy) {
            cudaStreamSynchronize(c->copy);
            cudaStreamDestroy(c->copy);
        }
        if (c->comm_stream) {
            cudaStreamSynchronize(c->comm_stream);
            cudaStreamDestroy(c->comm_stream);
        }
        if (c->aux) {
            cudaStreamSynchronize(c->aux);
            cudaStreamDestroy(c->aux);
            cudaEventDestroy(c->ev_fork);
            cudaEventDestroy(c->ev_join);
        }
        if (c->stream) {
            cudaStreamSynchronize(c->stream);
            cudaStreamDestroy(c->stream);
        }
        delete c;
    });
}

int frpca_ctx_sync(frpca_ctx* c) {
    return guarded([&] {
        check_ctx(c);
        FB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int frpca_host_alloc(uint64_t bytes, void** out) {
    return guarded([&] { FB_CUDA(cudaMallocHost(out, bytes ? bytes : 1)); });
}
int frpca_host_free(void* p) {
    return guarded([&] { if (p) FB_CUDA(cudaFreeHost(p)); });
}

int frpca_dmat_upload(frpca_ctx* c, int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                      const int64_t* col_idx, const double* values, frpca_dmat** out) {
    return frpca_dmat_upload_shard(c, rows, cols, 0, 0, rows, cols, nnz, row_ptr, col_idx, values, out);
}

int frpca_dmat_upload_shard(frpca_ctx* c, int64_t grows, int64_t gcols, int32_t col_shard,
                            int64_t offset, int64_t rows, int64_t cols, int64_t nnz,
                            const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                            frpca_dmat** out) {
    return guarded([&] {
        check_ctx(c);
        require(out != nullptr, "frpca_dmat_upload: null output");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        if (col_shard) {
            require(rows == grows && offset >= 0 && offset + cols <= gcols,
                    "frpca_dmat_upload_shard: column block out of range");
        } else {
            require(cols == gcols && offset >= 0 && offset + rows <= grows,
                    "frpca_dmat_upload_shard: row block out of range");
        }
        auto* M = new frpca_dmat;
        M->ctx = c;
        M->grows = grows;
        M->gcols = gcols;
        M->offset = offset;
        M->col_shard = col_shard;
        try {
            dcsr_upload_build(*c, *M, rows, cols, nnz, row_ptr, col_idx, values);
        } catch (...) {
            delete M;
            throw;
        }
        *out = M;
    });
}

int frpca_dmat_destroy(frpca_dmat* M) {
    return guarded([&] {
        if (!M) return;
        cudaSetDevice(M->ctx->device);
        delete M;
    });
}

int frpca_dmat_info(const frpca_dmat* M, int64_t* rows, int64_t* cols, int64_t* nnz) {
    return guarded([&] {
        require(M != nullptr, "frpca_dmat_info: null matrix");
        if (rows) *rows = M->A.rows;
        if (cols) *cols = M->A.cols;
        if (nnz) *nnz = M->A.nnz;
    });
}

int frpca_dmat_pass_count(const frpca_dmat* M, uint64_t* out) {
    return guarded([&] {
        require(M != nullptr && out != nullptr, "frpca_dmat_pass_count: null argument");
        *out = M->passes.load(std::memory_order_relaxed);
    });
}

int frpca_dmat_reset_pass_count(frpca_dmat* M) {
    return guarded([&] {
        require(M != nullptr, "frpca_dmat_reset_pass_count: null matrix");
        M->passes.store(0, std::memory_order_relaxed);
    });
}

int frpca_dmat_get_transpose(const frpca_dmat* M, int64_t* rp, int64_t* ci, double* v) {
    return guarded([&] {
        require(M != nullptr, "frpca_dmat_get_transpose: null matrix");
        Ctx& c = *M->ctx;
        std::lock_guard<std::mutex> lk(c.mu);
        FB_CUDA(cudaSetDevice(c.device));
        download_csr(c, M->At, rp, ci, v);
    });
}

int frpca_spmm(frpca_ctx* c, frpca_dmat* M, int transpose, const double* X, int64_t ldx,
               int64_t ncols, double* Y) {
    return guarded([&] {
        check_ctx(c);
        require(M != nullptr, "spmm: null matrix");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        const DCsr& A = transpose ? M->At : M->A;
        const int64_t nin = A.cols, nout = A.rows;
        require(ncols >= 0, "spmm: negative column count");
        require(ncols == 0 || ldx >= nin, "spmm: leading dimension too small");
        if (ncols == 0 || nout == 0) {
            M->passes.fetch_add(1);
            return;
        }
        DBuf<double> dX(size_t(std::max<int64_t>(nin, 1) * ncols), c->stream);
        DBuf<double> dY(size_t(nout * ncols), c->stream);
        if (nin) upload_colmajor(*c, X, nin, ncols, ldx, dX.get());
        spmm_pass(*c, *M, transpose != 0, dX.get(), ncols, dY.get());
        download_colmajor(*c, dY.get(), nout, ncols, Y);
    });
}

int frpca_gaussian_matrix(frpca_ctx* c, int64_t rows, int64_t cols, uint64_t seed, double* out) {
    return guarded([&] {
        check_ctx(c);
        require(rows >= 1 && cols >= 1, "gaussian_matrix: dimensions must be >= 1");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        DBuf<double> d(size_t(rows * cols), c->stream);
        with_checks(*c, [&] { gaussian_stream_device(*c, seed, rows * cols, d.get()); });
        FB_CUDA(cudaMemcpyAsync(out, d.get(), sizeof(double) * rows * cols, cudaMemcpyDeviceToHost,
                                c->stream));
        FB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int frpca_gaussian_window(frpca_ctx* c, int64_t count, int64_t period, int64_t w0, int64_t w1, uint64_t seed,
                          double* out) {
    return guarded([&] {
        check_ctx(c);
        require(count >= 1 && period >= 1 && 0 <= w0 && w0 < w1 && w1 <= period, "gaussian_window: bad window");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        const int64_t per = w1 - w0, full = count / period, rem = count % period;
        const int64_t n = full * per + std::max<int64_t>(0, std::min(rem, w1) - w0);
        DBuf<double> d(size_t(std::max<int64_t>(n, 1)), c->stream);
        with_checks(*c, [&] { gaussian_stream_window(*c, seed, count, period, w0, w1, d.get()); });
        if (n) FB_CUDA(cudaMemcpyAsync(out, d.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        FB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int frpca_gaussian_window_rows(frpca_ctx* c, int64_t count, int64_t period, int64_t w0, int64_t w1, uint64_t seed,
                               double* out) {
    return guarded([&] {
        check_ctx(c);
        require(count >= 1 && period >= 1 && 0 <= w0 && w0 < w1 && w1 <= period, "gaussian_window: bad window");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        const int64_t n = (w1 - w0) * ((count + period - 1) / period);
        DBuf<double> d(size_t(n), c->stream);
        FB_CUDA(cudaMemcpyAsync(d.get(), out, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        with_checks(*c, [&] { gaussian_stream_window(*c, seed, count, period, w0, w1, d.get(), true); });
        FB_CUDA(cudaMemcpyAsync(out, d.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        FB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int frpca_lu_basis(frpca_ctx* c, int64_t m, int64_t l, const double* Mh, double* X) {
    return guarded([&] {
        check_ctx(c);
        require(m >= l && l >= 1, "lu_basis: input must be tall (rows >= cols >= 1)");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        DBuf<double> W(size_t(m * l), c->stream);
        upload_colmajor(*c, Mh, m, l, m, W.get());
        with_checks(*c, [&] { lu_basis_device(*c, W.get(), m, l); });
        download_colmajor(*c, W.get(), m, l, X);
    });
}

struct frpca_mtx {
    fb::MtxData d;
};

int frpca_mtx_read(const char* path, frpca_mtx** out, int64_t* rows, int64_t* cols, int64_t* n) {
    return guarded([&] {
        require(path != nullptr && out != nullptr, "frpca_mtx_read: null argument");
        auto* h = new frpca_mtx;
        try {
            mtx_read(path, h->d);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
        if (rows) *rows = h->d.rows;
        if (cols) *cols = h->d.cols;
        if (n) *n = int64_t(h->d.v.size());
    });
}

int frpca_mtx_entries(const frpca_mtx* h, int64_t* r, int64_t* c, double* v) {
    return guarded([&] {
        require(h != nullptr, "frpca_mtx_entries: null handle");
        const size_t n = h->d.v.size();
        if (r) std::memcpy(r, h->d.r.data(), sizeof(int64_t) * n);
        if (c) std::memcpy(c, h->d.c.data(), sizeof(int64_t) * n);
        if (v) std::memcpy(v, h->d.v.data(), sizeof(double) * n);
    });
}

void frpca_mtx_free(frpca_mtx* h) { delete h; }

int frpca_mtx_write(const char* path, int64_t rows, int64_t cols, const int64_t* row_ptr, const int64_t* col_idx,
                    const double* values) {
    return guarded([&] {
        require(path != nullptr && row_ptr != nullptr, "frpca_mtx_write: null argument");
        mtx_write(path, rows, cols, row_ptr, col_idx, values);
    });
}

int frpca_csr_from_triplets(frpca_ctx* c, int64_t rows, int64_t cols, int64_t n, const int64_t* r,
                            const int64_t* ci, const double* v, int64_t* nnz, int64_t* row_ptr, int64_t* col_idx,
                            double* values) {
    return guarded([&] {
        check_ctx(c);
        require(rows >= 0 && cols >= 0, "from_triplets: negative dimension");
        require(n >= 0 && (n == 0 || (r && ci && v)) && nnz && row_ptr, "from_triplets: null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        csr_from_triplets_device(*c, rows, cols, n, r, ci, v, nnz, row_ptr, col_idx, values);
    });
}

int frpca_low_rank_error(frpca_ctx* c, frpca_dmat* M, int64_t k, const double* U, const double* S, const double* V,
                         int norm, uint64_t entry_limit, double* out) {
    return guarded([&] {
        check_ctx(c);
        require(M != nullptr && out != nullptr && k >= 0, "low_rank_error: null argument");
        require(norm == FRPCA_NORM_FROBENIUS || norm == FRPCA_NORM_SPECTRAL, "low_rank_error: unknown norm");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        const int64_t m = M->A.rows, n = M->A.cols;
        cudaStream_t s = c->stream;
        DBuf<double> dU(size_t(std::max<int64_t>(m * k, 1)), s), dS(size_t(std::max<int64_t>(k, 1)), s),
            dV(size_t(std::max<int64_t>(n * k, 1)), s);
        if (k) {
            FB_CUDA(cudaMemcpyAsync(dU.get(), U, sizeof(double) * m * k, cudaMemcpyHostToDevice, s));
            FB_CUDA(cudaMemcpyAsync(dS.get(), S, sizeof(double) * k, cudaMemcpyHostToDevice, s));
            FB_CUDA(cudaMemcpyAsync(dV.get(), V, sizeof(double) * n * k, cudaMemcpyHostToDevice, s));
        }
        *out = low_rank_error_device(*c, *M, k, dU.get(), dS.get(), dV.get(), norm, entry_limit);
    });
}

int frpca_pc_correlation(frpca_ctx* c, int64_t m, int64_t k, const double* Ut, const double* Ur, double* corr) {
    return guarded([&] {
        check_ctx(c);
        require(m >= 0 && k >= 0 && corr != nullptr, "pc_correlation: null argument");
        require(m >= 2, "pc_correlation: need at least two samples");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        DBuf<double> a(size_t(std::max<int64_t>(m * k, 1)), c->stream), b(size_t(std::max<int64_t>(m * k, 1)), c->stream);
        if (k) {
            FB_CUDA(cudaMemcpyAsync(a.get(), Ut, sizeof(double) * m * k, cudaMemcpyHostToDevice, c->stream));
            FB_CUDA(cudaMemcpyAsync(b.get(), Ur, sizeof(double) * m * k, cudaMemcpyHostToDevice, c->stream));
        }
        pc_correlation_device(*c, m, k, a.get(), b.get(), corr);
    });
}

int frpca_projector_distance(frpca_ctx* c, int64_t m, int64_t k1, const double* Q1, int64_t k2, const double* Q2,
                             double* out) {
    return guarded([&] {
        check_ctx(c);
        require(m >= 1 && k1 >= 0 && k2 >= 0 && out != nullptr, "projector_distance: null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        DBuf<double> a(size_t(std::max<int64_t>(m * k1, 1)), c->stream), b(size_t(std::max<int64_t>(m * k2, 1)), c->stream);
        if (k1) FB_CUDA(cudaMemcpyAsync(a.get(), Q1, sizeof(double) * m * k1, cudaMemcpyHostToDevice, c->stream));
        if (k2) FB_CUDA(cudaMemcpyAsync(b.get(), Q2, sizeof(double) * m * k2, cudaMemcpyHostToDevice, c->stream));
        *out = projector_distance_device(*c, m, k1, a.get(), k2, b.get());
    });
}

int frpca_orth(frpca_ctx* c, int64_t m, int64_t l, const double* Mh, double* Q) {
    return guarded([&] {
        check_ctx(c);
        require(m >= l && l >= 1, "orth: input must be tall (rows >= cols >= 1)");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        DBuf<double> W(size_t(m * l), c->stream);
        upload_colmajor(*c, Mh, m, l, m, W.get());
        with_checks(*c, [&] { orth_device(*c, W.get(), m, l); });
        download_colmajor(*c, W.get(), m, l, Q);
    });
}

int frpca_eig_svd(frpca_ctx* c, int64_t m, int64_t n, const double* Ah, double* U, double* S,
                  double* V) {
    return guarded([&] {
        check_ctx(c);
        require(m >= n && n >= 1, "eig_svd: input must be tall (rows >= cols >= 1)");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        DBuf<double> W(size_t(m * n), c->stream), Ud(size_t(m * n), c->stream);
        upload_colmajor(*c, Ah, m, n, m, W.get());
        EigWork e;
        with_checks(*c, [&] { e.run(*c, W.get(), m, n, /*row_sharded=*/false); });
        DBuf<double> Mf(size_t(n * n), c->stream), Sd(size_t(n), c->stream);
        e.factor(*c, 0, int(n), int(n), false, true, Mf.get());
        gemm_device(*c, W.get(), m, n, Mf.get(), n, Ud.get(), n, false);
        e.singular_values(*c, 0, int(n), false, Sd.get());
        FB_CUDA(cudaMemcpyAsync(S, Sd.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        FB_CUDA(cudaMemcpyAsync(V, e.B.get(), sizeof(double) * n * n, cudaMemcpyDeviceToHost, c->stream));
        download_colmajor(*c, Ud.get(), m, n, U);
    });
}

// FRPCA_DEBUG_TIMELINE (with profiling on): the call's event brackets on the
// main stream (and the upload builder's), start / end relative to the first
// one (diagnostic)
static void print_timeline(Ctx& c, size_t p0) {
    static const bool tl = std::getenv("FRPCA_DEBUG_TIMELINE") != nullptr;
    if (!tl || !c.prof || c.pending.size() <= p0) return;
    const cudaEvent_t base = c.pending[p0].a;
    for (size_t i = p0; i < c.pending.size(); ++i) {
        float t0 = 0.f, t1 = 0.f;
        cudaEventElapsedTime(&t0, base, c.pending[i].a);
        cudaEventElapsedTime(&t1, base, c.pending[i].b);
        std::fprintf(stderr, "[timeline] %9.2f %9.2f %s\n", t0, t1, c.pending[i].name.c_str());
    }
    if (c.tside)
        for (size_t i = c.tside->tl_mark; i < c.tside->pending.size(); ++i) {
            float t0 = 0.f, t1 = 0.f;
            cudaEventElapsedTime(&t0, base, c.tside->pending[i].a);
            cudaEventElapsedTime(&t1, base, c.tside->pending[i].b);
            std::fprintf(stderr, "[timeline] %9.2f %9.2f   builder: %s\n", t0, t1, c.tside->pending[i].name.c_str());
        }
}

int frpca_run(frpca_ctx* c, frpca_dmat* M, int algorithm, const frpca_config* cfg, const double* omega,
              int64_t omega_rows, int64_t omega_cols, double* U, double* S, double* V, double* basis,
              frpca_stats* stats, int* dispatched) {
    return guarded([&] {
        check_ctx(c);
        require(M != nullptr && cfg != nullptr, "frpca_run: null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        RunArgs a;
        a.cfg = *cfg;
        a.omega = omega;
        a.omega_rows = omega_rows;
        a.omega_cols = omega_cols;
        a.U = U; a.S = S; a.V = V; a.basis = basis;
        a.device_io = (cfg->flags & FRPCA_FLAG_DEVICE_IO) != 0;
        int algo = algorithm;
        if (algo == FRPCA_ALGO_AUTO) algo = (M->grows < M->gcols) ? FRPCA_ALGO_FRPCA : FRPCA_ALGO_FRPCAT;
        require(algo == FRPCA_ALGO_FRPCA || algo == FRPCA_ALGO_FRPCAT || algo == FRPCA_ALGO_BASIC_RPCA ||
                    algo == FRPCA_ALGO_BASIC_RPCAT,
                "frpca_run: unknown algorithm");
        if (dispatched) *dispatched = algo;
        const size_t p0 = c->pending.size();
        run_algorithm(*c, *M, a, stats, algo);
        print_timeline(*c, p0);
    });
}

// One-shot run from a host CSR: upload + run + release, with the sketch (which
// depends only on the seed and the shape) generated on a second stream by a
// second host thread while the CSR is uploaded and the device transpose built.
// FRPCA_DEBUG_E2E: host timestamps of frpca_run_csr's phases (diagnostic)
static void dbg_mark(const char* what, bool start = false) {
    static const bool on = std::getenv("FRPCA_DEBUG_E2E") != nullptr;
    if (!on) return;
    static thread_local std::chrono::steady_clock::time_point t0;
    const auto now = std::chrono::steady_clock::now();
    if (start) t0 = now;
    std::fprintf(stderr, "[e2e] %8.2f ms %s\n", std::chrono::duration<double, std::milli>(now - t0).count(), what);
}

int frpca_run_csr(frpca_ctx* c, int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                  const int64_t* col_idx, const double* values, int algorithm, const frpca_config* cfg,
                  const double* omega, int64_t omega_rows, int64_t omega_cols, double* U, double* S, double* V,
                  double* basis, frpca_stats* stats, int* dispatched) {
    return guarded([&] {
        check_ctx(c);
        require(cfg != nullptr, "frpca_run: null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        FB_CUDA(cudaSetDevice(c->device));
        dbg_mark("start", true);
        const size_t p0 = c->pending.size();
        int algo = algorithm;
        if (algo == FRPCA_ALGO_AUTO) algo = (rows < cols) ? FRPCA_ALGO_FRPCA : FRPCA_ALGO_FRPCAT;
        // shape of the sketch each algorithm draws (randsvd.hpp:110, :150, :239, :291)
        const int64_t l = cfg->k + cfg->oversample, q = cfg->passes;
        int64_t orow = 0, ocol = 0;
        bool ok = !omega && !(cfg->flags & FRPCA_FLAG_HOST_OMEGA) && c->world == 1 && cfg->k >= 1 &&
                  cfg->oversample >= 0 && l >= 1 && rows >= 1 && cols >= 1;
        if (ok) {
            if (algo == FRPCA_ALGO_FRPCA) {
                ok = rows <= cols && q >= 2 && l <= rows;
                if (q % 2 == 0) { orow = cols; ocol = l; } else { orow = rows; ocol = l; }
            } else if (algo == FRPCA_ALGO_FRPCAT) {
                ok = rows >= cols && q >= 2 && l <= cols;
                if (q % 2 == 0) { orow = l; ocol = rows; } else { orow = cols; ocol = l; }
            } else if (algo == FRPCA_ALGO_BASIC_RPCA) {
                ok = cfg->power >= 0 && l <= std::min(rows, cols);
                orow = cols; ocol = l;
            } else if (algo == FRPCA_ALGO_BASIC_RPCAT) {
                ok = cfg->power >= 0 && l <= std::min(rows, cols);
                orow = l; ocol = rows;
            } else {
                ok = false;
            }
        }
        DBuf<double>* pre = nullptr;
        bool pre_rm = false;
        std::exception_ptr side_err;
        std::thread side_thread;
        if (ok) {
            if (!c->side) {
                auto sd = std::make_unique<Ctx>();
                sd->device = c->device;
                sd->num_sms = c->num_sms;
                sd->omega_sync = true;  // checked on its own thread (off the critical path)
                FB_CUDA(cudaStreamCreateWithFlags(&sd->stream, cudaStreamNonBlocking));
                c->side = std::move(sd);
            }
            Ctx* side = c->side.get();
            const uint64_t seed = mix_seed(cfg->seed, 0xA11CEull);
            const int64_t count = orow * ocol;
            // frpca and odd-q frpcat read the sketch row-major: generated so
            const bool rm = algo == FRPCA_ALGO_FRPCA || (algo == FRPCA_ALGO_FRPCAT && q % 2 == 1);
            pre_rm = rm;
            side_thread = std::thread([side, seed, count, orow, rm, &pre, &side_err] {
                try {
                    FB_CUDA(cudaSetDevice(side->device));
                    pre = &side->slot(0, size_t(count));  // kept: swapped with the run's slot
                    gaussian_stream_window(*side, seed, count, orow, 0, orow, pre->get(), rm);
                    FB_CUDA(cudaStreamSynchronize(side->stream));
                } catch (...) {
                    side_err = std::current_exception();
                }
            });
        }
        std::unique_ptr<frpca_dmat> M;
        try {
            M.reset(new frpca_dmat);
            M->ctx = c;
            M->grows = rows;
            M->gcols = cols;
            // the panel plan of the run's A^T*Y width is built while the
            // values are still crossing PCIe
            const int64_t whint = (algo == FRPCA_ALGO_FRPCA || algo == FRPCA_ALGO_FRPCAT) ? cfg->k + cfg->oversample : 0;
            // frpca / frpcat: the first A*X starts on the values as they land
            const char* pe = std::getenv("FRPCA_UPLOAD_PIPELINE");  // A/B knob
            const bool pipe = whint > 0 && c->world == 1 && !(pe && pe[0] == '0');
            dcsr_upload_build(*c, *M, rows, cols, nnz, row_ptr, col_idx, values, whint, pipe);
        } catch (...) {
            if (side_thread.joinable()) side_thread.join();
            throw;
        }
        dbg_mark("upload returned");
        if (side_thread.joinable()) side_thread.join();
        dbg_mark("side joined");
        if (side_err) std::rethrow_exception(side_err);
        RunArgs a;
        a.cfg = *cfg;
        a.omega = omega;
        a.omega_rows = omega_rows;
        a.omega_cols = omega_cols;
        a.U = U; a.S = S; a.V = V; a.basis = basis;
        a.device_io = (cfg->flags & FRPCA_FLAG_DEVICE_IO) != 0;
        a.pre = ok ? pre : nullptr;
        a.pre_rowmajor = pre_rm;
        if (dispatched) *dispatched = algo;
        require(algo == FRPCA_ALGO_FRPCA || algo == FRPCA_ALGO_FRPCAT || algo == FRPCA_ALGO_BASIC_RPCA ||
                    algo == FRPCA_ALGO_BASIC_RPCAT,
                "frpca_run: unknown algorithm");
        run_algorithm(*c, *M, a, stats, algo);
        dbg_mark("run returned");
        FB_CUDA(cudaStreamSynchronize(c->stream));
        dbg_mark("synced");
        M.reset();
        dbg_mark("matrix released");
        print_timeline(*c, p0);
    });
}

// Sharded run of a host CSR over a group (the single-process
// callers of the reference, frpca_cli.cpp:158-183, with every GPU of the box):
// frpcat takes row blocks, frpca column blocks (shard_cuts); each rank uploads
// its shard and runs on its own host thread; the collectives sum the partials.
// U / V / S land in the caller's full column-major matrices: each rank writes
// its rows of the sharded factor, rank 0 the replicated one and S.
int frpca_group_run_csr(frpca_group* g, int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* values, int algorithm, const frpca_config* cfg,
                        double* U, double* S, double* V, frpca_stats* stats, int* dispatched) {
    return guarded([&] {
        require(g != nullptr && cfg != nullptr && row_ptr != nullptr, "frpca_run: null argument");
        require(rows >= 0 && cols >= 0 && nnz == row_ptr[rows], "frpca_group_run_csr: row_ptr[rows] must equal nnz");
        require(!(cfg->flags & FRPCA_FLAG_DEVICE_IO), "frpca_group_run_csr: host buffers only");
        int algo = algorithm;
        if (algo == FRPCA_ALGO_AUTO) algo = (rows < cols) ? FRPCA_ALGO_FRPCA : FRPCA_ALGO_FRPCAT;
        require(algo == FRPCA_ALGO_FRPCA || algo == FRPCA_ALGO_FRPCAT,
                "frpca_group_run_csr: only frpca / frpcat run sharded");
        if (dispatched) *dispatched = algo;
        const int world = int(g->ctx.size());
        const int col_shard = algo == FRPCA_ALGO_FRPCA ? 1 : 0;
        std::vector<int64_t> cuts(size_t(world) + 1);
        shard_cuts(rows, cols, row_ptr, col_idx, col_shard, world, cuts.data());
        if (g->loop) loopback_reset(*g->loop);  // a failed earlier run left the flag set
        std::vector<std::exception_ptr> errs(static_cast<size_t>(world));
        std::vector<frpca_stats> st(static_cast<size_t>(world));
        auto rank_main = [&](int r) {
            frpca_ctx* c = g->ctx[size_t(r)];
            try {
                std::lock_guard<std::mutex> lk(c->mu);
                FB_CUDA(cudaSetDevice(c->device));
                const int64_t a0 = cuts[size_t(r)], a1 = cuts[size_t(r) + 1];
                std::vector<int64_t> lrp, lci;
                std::vector<double> lva;
                const int64_t *prp, *pci;
                const double* pva;
                int64_t lrows, lcols;
                if (!col_shard) {
                    lrp.resize(size_t(a1 - a0) + 1);
                    for (int64_t i = a0; i <= a1; ++i) lrp[size_t(i - a0)] = row_ptr[i] - row_ptr[a0];
                    prp = lrp.data();
                    pci = col_idx + row_ptr[a0];
                    pva = values + row_ptr[a0];
                    lrows = a1 - a0;
                    lcols = cols;
                } else {
                    shard_extract_cols(rows, row_ptr, col_idx, values, a0, a1, lrp, lci, lva);
                    prp = lrp.data();
                    pci = lci.data();
                    pva = lva.data();
                    lrows = rows;
                    lcols = a1 - a0;
                }
                std::unique_ptr<frpca_dmat> M(new frpca_dmat);
                M->ctx = c;
                M->grows = rows;
                M->gcols = cols;
                M->offset = a0;
                M->col_shard = col_shard;
                dcsr_upload_build(*c, *M, lrows, lcols, prp[lrows], prp, pci, pva);
                RunArgs a;
                a.cfg = *cfg;
                if (!col_shard) {   // frpcat: U row-sharded, V replicated
                    a.U = U ? U + a0 : nullptr;
                    a.u_ld = rows;
                    a.V = r == 0 ? V : nullptr;
                } else {            // frpca: V row-sharded (columns of A), U replicated
                    a.V = V ? V + a0 : nullptr;
                    a.v_ld = cols;
                    a.U = r == 0 ? U : nullptr;
                }
                a.S = r == 0 ? S : nullptr;
                run_algorithm(*c, *M, a, &st[size_t(r)], algo);
                FB_CUDA(cudaStreamSynchronize(c->stream));
            } catch (...) {
                errs[size_t(r)] = std::current_exception();
                if (g->loop) loopback_fail(*g->loop);
            }
        };
        std::vector<std::thread> th;
        for (int r = 0; r < world; ++r) th.emplace_back(rank_main, r);
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        if (stats) *stats = st[0];
    });
}

int frpca_profile_enable(frpca_ctx* c, int enable) {
    return guarded([&] {
        check_ctx(c);
        c->flush_profile();
        c->prof = enable != 0;
    });
}

int frpca_profile_reset(frpca_ctx* c) {
    return guarded([&] {
        check_ctx(c);
        c->flush_profile();
        c->agg.clear();
    });
}

int frpca_profile_count(frpca_ctx* c, int* n) {
    return guarded([&] {
        check_ctx(c);
        c->flush_profile();
        c->agg_names.clear();
        for (auto& kv : c->agg) c->agg_names.push_back(kv.first);
        *n = int(c->agg_names.size());
    });
}

int frpca_profile_get(frpca_ctx* c, int idx, const char** name, int64_t* launches, double* ms,
                      double* bytes, double* flops) {
    return guarded([&] {
        check_ctx(c);
        require(idx >= 0 && idx < int(c->agg_names.size()), "frpca_profile_get: index out of range");
        const std::string& k = c->agg_names[size_t(idx)];
        const ProfAgg& g = c->agg.at(k);
        if (name) *name = k.c_str();
        if (launches) *launches = g.launches;
        if (ms) *ms = g.ms;
        if (bytes) *bytes = g.bytes;
        if (flops) *flops = g.flops;
    });
}

int frpca_timer_begin(frpca_ctx* c) {
    return guarded([&] {
        check_ctx(c);
        if (!c->timer_a) FB_CUDA(cudaEventCreate(&c->timer_a));
        if (!c->timer_b) FB_CUDA(cudaEventCreate(&c->timer_b));
        FB_CUDA(cudaEventRecord(c->timer_a, c->stream));
    });
}

int frpca_timer_end(frpca_ctx* c, double* ms) {
    return guarded([&] {
        check_ctx(c);
        require(c->timer_a != nullptr, "frpca_timer_end: no frpca_timer_begin");
        FB_CUDA(cudaEventRecord(c->timer_b, c->stream));
        FB_CUDA(cudaEventSynchronize(c->timer_b));
        float f = 0.f;
        FB_CUDA(cudaEventElapsedTime(&f, c->timer_a, c->timer_b));
        *ms = f;
    });
}

int frpca_launch_count(uint64_t* out) {
    return guarded([&] { *out = g_launches.load(std::memory_order_relaxed); });
}

}  // extern "C"
