// Driver-level declarations (driver.cu, comm.cu, abi.cu).
#pragma once

#include "internal.cuh"

namespace fb {

struct RunArgs {
    frpca_config cfg{};
    const double* omega = nullptr;
    int64_t omega_rows = 0, omega_cols = 0;
    double *U = nullptr, *S = nullptr, *V = nullptr, *basis = nullptr;
    // leading dimensions of U / V in the caller's memory (0: their row count);
    // a group run writes each rank's rows of the sharded factor into the
    // caller's full matrix
    int64_t u_ld = 0, v_ld = 0;
    bool device_io = false;
    // Omega generated ahead (frpca_run_csr), moved into the run's slot by the
    // first sketch_into of the call; a repeated call (run_algorithm's retry)
    // regenerates it
    DBuf<double>* pre = nullptr;
    bool pre_rowmajor = false;  // `pre` holds the row-major (transposed) layout
};

// eig_svd pipeline state: Gram -> (allreduce) -> syevd (B becomes V) -> rank check.
// `row_sharded`: W holds this rank's rows of a row-distributed matrix, so the
// Gram partials are summed over ranks; a replicated W (identical on every
// rank, e.g. Z after its allreduce) is not summed.
struct EigWork {
    DBuf<double> B, D;
    int64_t l = 0;
    // keep_gram (n x n, optional): a copy of the Gram matrix before syevd overwrites it
    void run(Ctx& c, const double* W, int64_t r, int64_t n, bool row_sharded, double* keep_gram = nullptr);
    void factor(Ctx& c, int s, int k, int ncols, bool rev, bool scale, double* M);
    void singular_values(Ctx& c, int s, int k, bool rev, double* S);
};

void eig_svd_U(Ctx& c, const double* W, int64_t r, int64_t n, double* Uout);
void spmm_pass(Ctx& c, DMat& M, bool transpose, const double* X, int64_t ncols, double* Y);
void spmm_pass_reduced(Ctx& c, DMat& M, bool transpose, const double* X, int64_t ncols, double* Y);
void run_frpcat(Ctx& c, DMat& M, const RunArgs& a, frpca_stats* st);
void run_frpca(Ctx& c, DMat& M, const RunArgs& a, frpca_stats* st);
// basic_rpca (left = false) / basic_rpcat (left = true), randsvd.hpp:95-175
void run_basic(Ctx& c, DMat& M, const RunArgs& a, frpca_stats* st, bool left);
// one of the four algorithms with the deferred-error protocol: reset, run,
// check; a small-eigensolver non-convergence re-runs the call with cuSOLVER
void run_algorithm(Ctx& c, DMat& M, const RunArgs& a, frpca_stats* st, int algo);
// f() under the deferred-error protocol (the standalone kernel entry points)
template <class F>
void with_checks(Ctx& c, F&& f) {
    for (int attempt = 0;; ++attempt) {
        try {
            err_reset(c);
            c.checked = true;
            f();
            c.checked = false;
            err_check(c);
            break;
        } catch (const RetryCall& r) {
            c.checked = false;
            if (attempt >= 2) {
                c.force_cusolver = c.omega_sync = false;
                throw CudaError("deferred-error retry did not succeed");
            }
            if (r.code == kErrEigNoConv) c.force_cusolver = true;
            else c.omega_sync = true;
        } catch (...) {
            c.checked = c.force_cusolver = c.omega_sync = false;
            throw;
        }
    }
    c.force_cusolver = c.omega_sync = false;
}
uint64_t mix_seed(uint64_t seed, uint64_t tag);

// validation.cu (validation.hpp:125-282); U, S, V, Q device, column-major
double low_rank_error_device(Ctx& c, DMat& M, int64_t k, const double* U, const double* S, const double* V,
                             int norm, uint64_t entry_limit);
void pc_correlation_device(Ctx& c, int64_t m, int64_t k, const double* Ut, const double* Ur, double* corr_host);
double projector_distance_device(Ctx& c, int64_t m, int64_t k1, const double* Q1, int64_t k2, const double* Q2);

// comm.cu: in-place sum over ranks (no-op on one GPU).
void allreduce_sum(Ctx& c, double* x, int64_t count);
void comm_init(Ctx& c, int rank, int world, const void* id128);       // NCCL, one process per GPU
void comm_init_all(std::vector<Ctx*>& ctxs, const std::vector<int>& devices);  // NCCL, one process
struct LoopbackGroup;
std::shared_ptr<LoopbackGroup> loopback_group(int world);
void comm_attach_loopback(Ctx& c, const std::shared_ptr<LoopbackGroup>& g, int rank);
void loopback_fail(LoopbackGroup& g);
void loopback_reset(LoopbackGroup& g);

// group.cu: host-side shard plan of a CSR over `world` ranks.
// Row blocks (frpcat) balanced by nnz + rows; column blocks (frpca) balanced by
// column nnz + 1. cuts: world + 1 boundaries.
void shard_cuts(int64_t rows, int64_t cols, const int64_t* row_ptr, const int64_t* col_idx, int col_shard,
                int world, int64_t* cuts);
// the local CSR of columns [c0, c1) (local column ids); row_ptr rows + 1
void shard_extract_cols(int64_t rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                        int64_t c0, int64_t c1, std::vector<int64_t>& lrp, std::vector<int64_t>& lci,
                        std::vector<double>& lva);
void comm_destroy(Ctx& c);
void comm_unique_id(void* out128);

}  // namespace fb
