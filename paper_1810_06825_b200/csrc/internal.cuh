// Internal types shared by the translation units of libfrpca_b200.so.
#pragma once

#include <cusolverDn.h>

#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "mtx.hpp"

namespace fb {

struct Ctx;
// In-place fp64 sum over the ranks of a sharded run (comm.cu: NCCL or the
// host-staged loopback of contexts in one process), ordered on stream s.
struct Collective {
    virtual ~Collective() = default;
    virtual void allreduce_sum(Ctx& c, double* x, int64_t count, cudaStream_t s) = 0;
};

// One unit of SpMM work for one warp (see spmm.cu). r1 >= 0: the consecutive
// short rows [r0, r1), each summed sequentially in CSR order straight into the
// output row. r1 < 0: nonzeros [p0, p1) of the long row r0, summed
// sequentially into partial slot -(r1 + 1); partials of one row are then
// added in slot order (fixed, deterministic combine).
struct WorkItem {
    int64_t p0, p1;
    int32_t r0, r1;
};
struct Combine {
    int32_t row, s0, s1, pad;
};

// A load-balanced SpMM work list (built once at load, see csr.cu).
struct ItemList {
    DBuf<WorkItem> items;
    DBuf<Combine> comb;
    int64_t nitems = 0, ncomb = 0, nslots = 0, chunk = 0;
    // kCuts row ranges at item boundaries (a long row's chunks stay together),
    // for a product whose output rows are handed on chunk by chunk (the
    // sharded allreduce overlapped with the rest of the product): chunk k is
    // rows [cut_row[k], cut_row[k+1]), items [cut_item[k], ..), combines
    // [cut_comb[k], ..)
    std::vector<int64_t> cut_row, cut_item, cut_comb;
};
constexpr int kCuts = 8;

// Panelled A^T*Y (csr.cu build_panels, spmm.cu spmm_panelled): when the
// gathered operand Y (rows x l) is much larger than L2, the entries of the
// "hot" rows of A^T (popular columns of A) are cut at panel boundaries of Y's
// rows (`pr` rows per panel) and the chunks are executed panel-major, so the Y
// rows they gather are L2-resident while a panel is being worked on; the
// chunk partials are added per row in entry order. The other ("cold") rows
// keep the plain gather list.
struct PanelPlan {
    int64_t pr = 0, npanels = 0, thot = 0, nhot = 0;
    DBuf<uint8_t> skip;  // hot rows (skipped by the cold list)
    ItemList hot;        // chunk items, panel-major; slots per row in entry order
    ItemList cold;       // work list of the other rows
    DBuf<int32_t> counter;
    DBuf<double> part;   // chunk partials, kept with the plan (grown on demand)
};

// Values of a CSR still crossing PCIe (frpca_run_csr's pipelined upload,
// csr.cu dcsr_upload_build): the copy stream records ev[j] when values chunk j
// has landed; item chunk k of A's work list (ItemList::cut_*) needs chunk
// need[k]. Meanwhile the builder thread builds A^T (structure, work list,
// panel plan, then its values behind the last chunk) and A's column ranks on
// its own stream and records `all`. The first product over the matrix
// consumes it (spmm.cu): A*X chunk by chunk as the values land; anything else
// joins the builder and waits for `all` (consume_pending).
struct DCsr;
struct PendingValues {
    std::vector<cudaEvent_t> ev;
    std::vector<int> need;
    cudaEvent_t all = nullptr;
    std::thread builder;
    std::exception_ptr err;
    bool joined = false;
    DCsr* a = nullptr;                  // receives the ranks at the join
    DBuf<int32_t> perm;                 // A^T entry k = nonzero perm[k] of A (the values gather)
    DBuf<int32_t> rank_of, rank_ids;    // A's column ranks, built by the builder
    PendingValues() = default;
    PendingValues(const PendingValues&) = delete;
    PendingValues& operator=(const PendingValues&) = delete;
    void join();  // joins the builder, installs the ranks, rethrows its error
    ~PendingValues() {
        // never free a buffer the builder or the copy stream still uses
        if (builder.joinable()) builder.join();
        if (all) cudaEventSynchronize(all);
        for (auto e : ev) cudaEventDestroy(e);
        if (all) cudaEventDestroy(all);
    }
};

// Device CSR: int64 row_ptr (8 B/row), int32 col ids, fp64 values (12 B/nnz).
struct DCsr {
    int64_t rows = 0, cols = 0, nnz = 0;
    DBuf<int64_t> rowptr;
    DBuf<int32_t> col;
    DBuf<double> val;
    ItemList L;  // work list over all rows
    // Column encodings of A (A only): popularity rank of every column (nnz,
    // ties to the lower id) and its inverse rank_ids. The sx_h top-ranked
    // columns are encoded as kColHot | rank (X rows staged in shared memory
    // by the sliced A*X, spmm.cu k_spmm_sx); the following ones up to hint_h
    // carry the sign bit (X rows kept in L2 with evict_last, MODE_HINT).
    // Re-encoded in place by ensure_encoding when a call needs other counts.
    DBuf<int32_t> rank_of, rank_ids;
    int64_t hint_h = 0, sx_h = 0;
    PanelPlan pan;  // on A^T only
    // last member, so it is destroyed (and waited for) before the buffers
    std::shared_ptr<PendingValues> pend;
};
// one device word read back through the context's mapped host words (no
// device->host copy queued behind large uploads)
int64_t read_i64(Ctx& c, const int64_t* d);
// waits (on c.stream) for every pending value of A and drops the record
void consume_pending(Ctx& c, DCsr& A);
constexpr int32_t kColMask = 0x7fffffff;  // id under the L2-hint sign bit
constexpr int32_t kColHot = 0x40000000;   // shared-memory-staged column: kColHot | rank
constexpr int32_t kRankMask = 0x3fffffff;

struct ProfAgg {
    int64_t launches = 0;
    double ms = 0, bytes = 0, flops = 0;
};

// Pinned, device-mapped host words for scalar read-backs: a kernel stores the
// value, the host reads it after a stream synchronisation. No device->host
// copy is queued behind the multi-GB host->device copies of an upload
// (measured: a copy-based read waited up to 65 ms behind the values).
struct MappedSlots {
    uint64_t* h = nullptr;
    uint64_t* d = nullptr;
    MappedSlots() = default;
    MappedSlots(const MappedSlots&) = delete;
    MappedSlots& operator=(const MappedSlots&) = delete;
    ~MappedSlots() {
        if (h) cudaFreeHost(h);
    }
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cusolverDnHandle_t solver = nullptr;
    int rank = 0, world = 1;
    std::shared_ptr<Collective> coll;  // world > 1
    int num_sms = 148;
    std::mutex mu;  // the ABI serialises calls on one context
    cudaEvent_t timer_a = nullptr, timer_b = nullptr;
    // Deferred errors: kernels record the first failure of a call here
    // (atomicCAS from 0; codes kErr*), read once when the call finishes, so a
    // run has no host round trip between its stages (err_reset / err_check).
    DBuf<int> dflag;
    bool force_cusolver = false;  // re-run after the small eigensolver did not converge
    bool omega_sync = false;      // Omega batches checked on the host (re-run after a shortfall; side stream)
    bool checked = false;         // inside with_checks: deferred errors will be read
    DBuf<double> omega_stage;  // normals staging of the Omega generator, kept (grown on demand)
    MappedSlots mapped;        // csr.cu read_scalar
    std::unique_ptr<Ctx> side;  // second stream for work overlapped with the upload (frpca_run_csr)
    std::unique_ptr<Ctx> tside;  // builder of A^T beside the first A*X (pipelined upload)
    cudaStream_t copy = nullptr;  // device->host copies of results overlapped with the output GEMMs
    // sharded runs: the allreduce of a product's finished row chunks runs here
    // while the next chunks are computed (spmm.cu *_reduced)
    cudaStream_t comm_stream = nullptr;
    // A^T*Y cold rows run beside the panel chunks (spmm.cu spmm_t_device)
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    DBuf<int32_t> wcount;  // SpMM work counters (main stream, aux stream)
    // Run workspaces by role, kept between runs and grown on demand: a fresh
    // multi-GB allocation per run makes the stream-ordered pool remap memory
    // (measured 0.8 s for a 16 GB output buffer at C4).
    static constexpr int kSlots = 8;
    DBuf<double> slots[kSlots];  // fixed storage: references handed out stay valid
    DBuf<double>& slot(int i, size_t n) {
        if (i < 0 || i >= kSlots) throw CudaError("workspace slot out of range");
        DBuf<double>& b = slots[i];
        if (b.n < n) {
            b.release();
            b.alloc(n, stream);
        }
        b.s = stream;
        return b;
    }

    // profiling: events around each launch, folded into per-kernel aggregates
    bool prof = false;
    size_t tl_mark = 0;  // first bracket of the current call (timeline diagnostics)
    struct Pending {
        std::string name;
        cudaEvent_t a, b;
        double bytes, flops;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    std::map<std::string, ProfAgg> agg;
    std::vector<std::string> agg_names;  // stable storage for frpca_profile_get

    cudaEvent_t get_event();
    void flush_profile();  // synchronises the stream
};

// RAII launch bracket: records events on ctx.stream when profiling is on.
struct Prof {
    Ctx& c;
    size_t idx = size_t(-1);
    Prof(Ctx& ctx, const char* name, double bytes, double flops);
    ~Prof();
};

struct DMat {
    Ctx* ctx = nullptr;
    DCsr A;   // local rows (or local column block) of the matrix
    DCsr At;  // its transpose, built on the device at load
    int64_t grows = 0, gcols = 0;  // global shape (== local shape on 1 GPU)
    int64_t offset = 0;            // first global row (row shard) or column (col shard)
    int col_shard = 0;
    std::atomic<uint64_t> passes{0};
    DMat() = default;
    ~DMat() {
        // the builder of a pipelined upload writes into At: finish it first
        std::shared_ptr<PendingValues> p = A.pend ? A.pend : At.pend;
        A.pend.reset();
        At.pend.reset();
        p.reset();
    }
};

// ---- csr.cu
// width_hint > 0: the A^T*Y panel plan for that width is built at load too
void dcsr_upload_build(Ctx& c, DMat& M, int64_t rows, int64_t cols, int64_t nnz,
                       const int64_t* h_rowptr, const int64_t* h_col, const double* h_val,
                       int64_t width_hint = 0, bool pipelined = false);
void download_csr(Ctx& c, const DCsr& A, int64_t* rp, int64_t* ci, double* v);
// work list of A's rows (rows with skip[r] != 0 left out), chunk size ch
void build_items(Ctx& c, const DCsr& A, const uint8_t* skip, ItemList& L, int64_t ch);
// sign-bit L2 hints on A's column ids for an A*X of width w (<= 256)
void ensure_hint(Ctx& c, DCsr& A, int64_t w);
// A's column ids encoded for hint_h L2-hinted and sx_h shared-memory columns
void ensure_encoding(Ctx& c, DCsr& A, int64_t hint_h, int64_t sx_h);
// panel plan of T (== A^T) for panels of pr rows of the gathered operand
void ensure_panels(Ctx& c, DCsr& T, int64_t pr, int64_t slot_cap);

// ---- spmm.cu : Y (rows x ncols, row-major ldy) = A * X (row-major ldx)
// panel rows / partial-slot cap of the panelled A^T*Y of width ncols on T
// (false: that A^T*Y runs unpanelled)
bool panel_rows_for(const DCsr& T, int64_t ncols, int64_t& pr, int64_t& cap);
void spmm_device(Ctx& c, const DCsr& A, const double* X, int64_t ldx, int64_t ncols, double* Y,
                 int64_t ldy, const char* tag);
// Z = A^T Y on T = the transposed CSR of A (panelled for large Y, spmm.cu)
void spmm_t_device(Ctx& c, DCsr& T, const double* Y, int64_t ncols, double* Z, const char* tag);
// The same products followed by the in-place sum of the output over the
// ranks, overlapped: each chunk of output rows (ItemList::cut_*) is summed on
// Ctx::comm_stream as soon as it is final, while the next chunk is computed.
// ldy == ncols. One GPU: the plain product.
void spmm_device_reduced(Ctx& c, const DCsr& A, const double* X, int64_t ncols, double* Y, const char* tag);
// comm.cu: in-place sum over ranks on the ctx stream (no-op on one GPU)
void allreduce_sum(Ctx& c, double* x, int64_t count);
void spmm_t_device_reduced(Ctx& c, DCsr& T, const double* Y, int64_t ncols, double* Z, const char* tag);

// ---- dense.cu
// B (n x n, column-major, full symmetric) = W^T W for row-major W (r x n, ld n).
void gram_device(Ctx& c, const double* W, int64_t r, int64_t n, double* B);
// C = W (r x K row-major, ld K) * M (K x N row-major, ld N). col_major_out: C is
// column-major (ldc >= r) else row-major (ldc >= N).
void gemm_device(Ctx& c, const double* W, int64_t r, int64_t K, const double* M, int64_t N,
                 double* C, int64_t ldc, bool col_major_out);
// out (cols x rows, row-major) = transpose of in (rows x cols row-major) ==
// column-major <-> row-major conversion of an r x c matrix.
void transpose_device(Ctx& c, const double* in, int64_t rows, int64_t cols, double* out);
double maxabs_device(Ctx& c, const double* x, int64_t n);
// max |x| into *out (bit pattern of a non-negative double), no host round trip
void maxabs_device_async(Ctx& c, const double* x, int64_t n, unsigned long long* out);

// ---- deferred errors (driver.cu)
constexpr int kErrLuPivot = 1, kErrEigRank = 2, kErrEigNoConv = 3, kErrOmegaShort = 4, kErrEigFail = 5,
              kErrOrthRank = 6;
int* err_flag(Ctx& c);
void err_reset(Ctx& c);
// waits for the stream; throws the first recorded error (NumericalError with
// the reference's message), or RetryCall when the call must be repeated with
// a slower path: cuSOLVER after a small-eigensolver non-convergence, the
// host-checked Omega loop after a (probability ~1e-15) stream shortfall
void err_check(Ctx& c);
struct RetryCall : std::runtime_error {
    int code;
    explicit RetryCall(int cd) : std::runtime_error("retry"), code(cd) {}
};

// ---- eig.cu : symmetric eigensolve of column-major n x n B (lower used):
// V (column-major) eigenvectors, D ascending eigenvalues (device), D copied to h_D.
void syevd_device(Ctx& c, double* B_inout_V, int64_t n, double* d_D, bool final_step = false);

// ---- csr.cu : from_triplets (sparse_matrix.hpp:62-95) on the device; host
// outputs row_ptr (rows + 1), col_idx / values (>= nnz entries; n suffices).
void csr_from_triplets_device(Ctx& c, int64_t rows, int64_t cols, int64_t n, const int64_t* r, const int64_t* ci,
                              const double* v, int64_t* nnz, int64_t* row_ptr, int64_t* col_idx, double* values);

// ---- orth.cu : in place: W (r x l row-major) -> Q of its Householder QR.
void orth_device(Ctx& c, double* W, int64_t r, int64_t l);

// ---- lu.cu : in place: W (m x l row-major) -> P^T L (row-major), lu_basis.
void lu_basis_device(Ctx& c, double* W, int64_t m, int64_t l);

// ---- rng.cu : Omega stream (dense_kernels.hpp:19-28) into `out` (count
// doubles, stream order), generated on the device.
void gaussian_stream_device(Ctx& c, uint64_t seed, int64_t count, double* out);
// the positions p < count of the same stream with (p mod P) in [w0, w1), into
// out[(p / P) (w1 - w0) + (p mod P - w0)]: a rank's slice of the sketch
// (randsvd.hpp:246-247 sharded; only that slice is written)
// rowmajor: the window's rows as a row-major (w1 - w0) x ceil(count / P) matrix
// (the transposed layout the products gather from) instead of column-major
void gaussian_stream_window(Ctx& c, uint64_t seed, int64_t count, int64_t P, int64_t w0, int64_t w1, double* out,
                            bool rowmajor = false);
void gaussian_stream_host(uint64_t seed, int64_t count, double* out);

}  // namespace fb
