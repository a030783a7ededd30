/*
 * frpca_b200.h — C ABI of the B200-native frPCA / frPCAt hot path
 * (arXiv 1810.06825; reference: /root/reference/proj/include/frpca/*.hpp).
 *
 * The reference has no FFI: its boundary is the header-only C++ template API
 * of randsvd.hpp (frpca :229-232, frpcat :281-284, auto_pca :339-341) over
 * SparseMatrixCsr<double> (sparse_matrix.hpp:19-150). This header is the thin
 * C layer the drop-in C++ API (include/frpca/frpca.hpp) and the Python host
 * mirror (paper_1810_06825_b200/) call; every entry point names the
 * reference interface it replaces. Plain pointers and sizes only.
 *
 * Conventions
 *  - Host dense matrices are COLUMN-MAJOR (Eigen's layout, types.hpp:12-16).
 *    Device-resident variants (FRPCA_FLAG_DEVICE_IO) use the same layout.
 *  - Sparse input is the reference CSR: int64 row_ptr (rows+1), int64
 *    col_idx (nnz, strictly increasing per row), double values (nnz).
 *  - Status: 0 ok; 2 invalid argument (std::invalid_argument via
 *    detail::require, types.hpp:45-47); 3 I/O; 4 numerical
 *    (frpca::NumericalError, types.hpp:27-30); 5 CUDA/NCCL failure.
 *    These equal the reference CLI's exit codes (frpca_cli.cpp:33-35).
 *    The message is available from frpca_last_error() (thread-local).
 */
#ifndef FRPCA_B200_H
#define FRPCA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FRPCA_OK 0
#define FRPCA_ERR_INVALID 2
#define FRPCA_ERR_IO 3
#define FRPCA_ERR_NUMERICAL 4
#define FRPCA_ERR_CUDA 5

/* PcaAlgorithm (randsvd.hpp:14): only the fast algorithms are on the path. */
#define FRPCA_ALGO_FRPCA 0  /* Alg. 5, rows <= cols (randsvd.hpp:224-276) */
#define FRPCA_ALGO_FRPCAT 1 /* Alg. 6, rows >= cols (randsvd.hpp:278-328) */
#define FRPCA_ALGO_AUTO 2   /* shape dispatch (randsvd.hpp:330-351) */
#define FRPCA_ALGO_BASIC_RPCA 3  /* baseline, sketch on the right (randsvd.hpp:95-134) */
#define FRPCA_ALGO_BASIC_RPCAT 4 /* baseline, sketch on the left (randsvd.hpp:136-175) */

/* frpca_run flags */
#define FRPCA_FLAG_DEVICE_IO 1u   /* omega/U/S/V/basis pointers are device pointers */
#define FRPCA_FLAG_HOST_OMEGA 2u  /* draw Omega with the host libstdc++ generator
                                     (default: bit-compatible device generator) */

typedef struct frpca_ctx frpca_ctx;   /* device, stream, cuSOLVER handle, NCCL comm */
typedef struct frpca_dmat frpca_dmat; /* device CSR + transposed CSR, built at load */

/* PcaConfig (randsvd.hpp:28-40); `deterministic` is unused by the reference
 * algorithms too (kernels here are always deterministic). */
typedef struct {
    int64_t k;
    int64_t oversample;
    int64_t passes; /* q >= 2, total passes over A */
    int64_t power;  /* baselines' p; unused on this path */
    uint64_t seed;
    int32_t deterministic;
    uint32_t flags; /* FRPCA_FLAG_* */
} frpca_config;

/* RunStats (randsvd.hpp:42-53) + load time of the upload that built dmat. */
typedef struct {
    double sketch_seconds;
    double power_seconds;
    double finalize_seconds;
    uint64_t passes_over_matrix;
} frpca_stats;

/* ---- library / context ---------------------------------------------------- */
const char* frpca_last_error(void);
int frpca_version(void);
int frpca_ctx_create(int device, frpca_ctx** out);
/* Multi-GPU: one process per GPU; `nccl_id` is the 128-byte ncclUniqueId from
 * frpca_nccl_unique_id() on rank 0, broadcast by the caller. */
int frpca_nccl_unique_id(void* out128);
int frpca_ctx_create_dist(int device, int rank, int world, const void* nccl_id128,
                          frpca_ctx** out);
int frpca_ctx_destroy(frpca_ctx* ctx);

/* Single-process multi-GPU (the reference's callers are single-process,
 * frpca_cli.cpp:158-183): one context (rank) per listed device. Distinct
 * devices exchange through NCCL (ncclCommInitAll); a device listed more than
 * once selects the host-staged loopback collective (ranks sharing a GPU, for
 * testing the sharded path on one device). comm: FRPCA_COMM_*. */
#define FRPCA_COMM_AUTO 0
#define FRPCA_COMM_NCCL 1
#define FRPCA_COMM_LOOPBACK 2
typedef struct frpca_group frpca_group;
int frpca_group_create(const int* devices, int ndev, int comm, frpca_group** out);
int frpca_group_size(const frpca_group* g, int* n);
/* the rank's context (owned by the group): shards can also be uploaded and run
 * per rank from the caller's own threads (frpca_dmat_upload_shard, frpca_run) */
int frpca_group_ctx(frpca_group* g, int rank, frpca_ctx** out);
int frpca_group_destroy(frpca_group* g);
/* frpca / frpcat / auto over the group from a host CSR: row blocks (frpcat) or
 * column blocks (frpca) from frpca_shard_cuts, one host thread per rank; U, S,
 * V are the caller's full column-major matrices (rows x k, k, cols x k).
 * Errors as frpca_run. */
int frpca_group_run_csr(frpca_group* g, int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* values, int algorithm, const frpca_config* cfg,
                        double* U, double* S, double* V, frpca_stats* stats, int* dispatched);

/* Shard plan (host only, no device): world + 1 boundaries of row blocks
 * (col_shard = 0; balanced by nnz + rows) or column blocks (col_shard = 1;
 * balanced by column nnz + 1). frpca_shard_cols extracts the local CSR of
 * columns [c0, c1) with local column ids (capacity from frpca_shard_cols_count). */
int frpca_shard_cuts(int64_t rows, int64_t cols, const int64_t* row_ptr, const int64_t* col_idx, int32_t col_shard,
                     int32_t world, int64_t* cuts);
int frpca_shard_cols_count(int64_t rows, const int64_t* row_ptr, const int64_t* col_idx, int64_t c0, int64_t c1,
                           int64_t* nnz_local);
int frpca_shard_cols(int64_t rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values, int64_t c0,
                     int64_t c1, int64_t* l_row_ptr, int64_t* l_col_idx, double* l_values);
int frpca_ctx_sync(frpca_ctx* ctx);
/* Pinned host memory helpers (for zero-staging host buffers). */
int frpca_host_alloc(uint64_t bytes, void** out);
int frpca_host_free(void* p);

/* ---- sparse matrix (replaces SparseMatrixCsr<double>, sparse_matrix.hpp:19-150)
 * Uploads and validates (same checks and messages as validate(), :125-142),
 * then builds the transposed CSR on the device (sparse_matrix.hpp:242-267,
 * moved to load time) and the load-balanced work lists of both. Host arrays
 * may be pageable or pinned. */
int frpca_dmat_upload(frpca_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz,
                      const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                      frpca_dmat** out);
/* Multi-GPU shard: this rank holds rows [row0, row0+rows) of a global
 * (grows x gcols) matrix (frpcat row-block sharding), or, with
 * col_shard = 1, columns [col0, col0+cols) of a (grows x gcols) matrix given
 * as a local CSR with LOCAL column ids (frpca column-block sharding). */
int frpca_dmat_upload_shard(frpca_ctx* ctx, int64_t grows, int64_t gcols, int32_t col_shard,
                            int64_t offset, int64_t rows, int64_t cols, int64_t nnz,
                            const int64_t* row_ptr, const int64_t* col_idx,
                            const double* values, frpca_dmat** out);
int frpca_dmat_destroy(frpca_dmat* A);
int frpca_dmat_info(const frpca_dmat* A, int64_t* rows, int64_t* cols, int64_t* nnz);
/* passCount()/resetPassCount() (sparse_matrix.hpp:119-122). */
int frpca_dmat_pass_count(const frpca_dmat* A, uint64_t* out);
int frpca_dmat_reset_pass_count(frpca_dmat* A);
/* Copies the device transposed CSR back (test helper, mirrors transpose()). */
int frpca_dmat_get_transpose(const frpca_dmat* A, int64_t* t_row_ptr, int64_t* t_col_idx,
                             double* t_values);

/* ---- load step ------------------------------------------------
 * load_matrix_market (matrix_market.hpp:27-93) up to from_triplets: parses a
 * coordinate real/integer, general/symmetric file (symmetric off-diagonal
 * entries also yield the mirrored entry) into an opaque handle; rows, cols and
 * the number of triplets n are returned. Errors: FRPCA_ERR_IO with the
 * reference's message. frpca_mtx_entries copies the 0-based triplets (file
 * order) into caller arrays of length n. */
typedef struct frpca_mtx frpca_mtx;
int frpca_mtx_read(const char* path, frpca_mtx** out, int64_t* rows, int64_t* cols, int64_t* n);
int frpca_mtx_entries(const frpca_mtx* h, int64_t* r, int64_t* c, double* v);
void frpca_mtx_free(frpca_mtx* h);
/* write_matrix_market (matrix_market.hpp:95-116): general, %.17g values. */
int frpca_mtx_write(const char* path, int64_t rows, int64_t cols, const int64_t* row_ptr,
                    const int64_t* col_idx, const double* values);
/* SparseMatrixCsr::from_triplets (sparse_matrix.hpp:62-95) on the device:
 * sort by (row, col), sum duplicates, drop exact-zero sums. Outputs (host):
 * nnz, row_ptr (rows + 1), col_idx and values (capacity n). Out-of-bounds
 * entries -> FRPCA_ERR_INVALID "from_triplets: entry out of bounds". */
int frpca_csr_from_triplets(frpca_ctx* ctx, int64_t rows, int64_t cols, int64_t n, const int64_t* r,
                            const int64_t* c, const double* v, int64_t* nnz, int64_t* row_ptr,
                            int64_t* col_idx, double* values);

/* ---- kernels (sparse_matrix.hpp:177-240, dense_kernels.hpp:16-174) --------- */
/* Y = A*X (transpose=0, spmm :177-206) or Y = A^T*X (transpose=1,
 * spmm_transpose :208-240). X: (A.cols or A.rows) x ncols column-major with
 * leading dimension ldx; Y column-major. One pass over A. */
int frpca_spmm(frpca_ctx* ctx, frpca_dmat* A, int transpose, const double* X, int64_t ldx,
               int64_t ncols, double* Y);
/* gaussian_matrix (dense_kernels.hpp:16-28): column-major rows x cols from
 * mt19937_64(seed) + libstdc++ normal_distribution, drawn on the device. */
int frpca_gaussian_matrix(frpca_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed,
                          double* out);
/* A rank's slice of the same stream (the sharded sketch): the positions
 * p < count with (p mod period) in [w0, w1), packed in order into out
 * (out[(p / period) (w1 - w0) + p mod period - w0]). */
int frpca_gaussian_window(frpca_ctx* ctx, int64_t count, int64_t period, int64_t w0, int64_t w1, uint64_t seed,
                          double* out);
/* The same window in the layout the products gather from: rows [w0, w1) of
 * the column-major stream as a row-major (w1 - w0) x ceil(count / period)
 * matrix (out[(p mod period - w0) ceil(count / period) + p / period]); positions
 * >= count are not written. Replaces gaussian_matrix + transpose for the
 * row-major sketch panels (randsvd.hpp:246-247, :298-299). */
int frpca_gaussian_window_rows(frpca_ctx* ctx, int64_t count, int64_t period, int64_t w0, int64_t w1,
                               uint64_t seed, double* out);
/* lu_basis (dense_kernels.hpp:50-116): X = P^T L of M (m x l, m >= l). */
int frpca_lu_basis(frpca_ctx* ctx, int64_t m, int64_t l, const double* M, double* X);
/* orth (dense_kernels.hpp:30-48): Q (m x l, column-major) of the Householder
 * QR of M; rank deficiency (|diag R| <= m eps max) -> FRPCA_ERR_NUMERICAL. */
int frpca_orth(frpca_ctx* ctx, int64_t m, int64_t l, const double* M, double* Q);
/* eig_svd (dense_kernels.hpp:145-174): U m x n, S ascending (n), V n x n. */
int frpca_eig_svd(frpca_ctx* ctx, int64_t m, int64_t n, const double* A, double* U, double* S,
                  double* V);

/* ---- algorithms (randsvd.hpp:224-351) -------------------------------------
 * algorithm: FRPCA_ALGO_*. omega: optional injected sketch (column-major,
 * omega_rows x omega_cols; the shape check of sketch_matrix, randsvd.hpp:68-74).
 * Outputs: U rows x k, S k (descending), V cols x k, column-major; basis
 * (nullable) receives Q (RunStats::capture_basis). stats, dispatched nullable.
 * With a distributed ctx, each rank passes its shard; U (frpcat) / V (frpca)
 * receive the rank's local rows, the replicated factor is written on every rank. */
int frpca_run(frpca_ctx* ctx, frpca_dmat* A, int algorithm, const frpca_config* cfg,
              const double* omega, int64_t omega_rows, int64_t omega_cols, double* U,
              double* S, double* V, double* basis, frpca_stats* stats, int* dispatched);

/* ---- validation metrics (validation.hpp:125-282) ------------
 * Host column-major inputs. low_rank_error: |A - U diag(S) V^T| (U rows x k,
 * S k, V cols x k) in FRPCA_NORM_FROBENIUS (dense residual when rows*cols <=
 * entry_limit, else the cross-term identity) or FRPCA_NORM_SPECTRAL (power
 * iteration through the SpMM kernels; counts passes over A like the
 * reference). pc_correlation: |Pearson| of matching columns (m x k each).
 * projector_distance: |Q1 Q1^T - Q2 Q2^T|_2 for orthonormal Q1 (m x k1),
 * Q2 (m x k2). Messages and error codes as the reference. */
#define FRPCA_NORM_FROBENIUS 0
#define FRPCA_NORM_SPECTRAL 1
#define FRPCA_ORACLE_ENTRY_LIMIT 4000000ull /* kDefaultOracleEntryLimit, validation.hpp:26 */
int frpca_low_rank_error(frpca_ctx* ctx, frpca_dmat* A, int64_t k, const double* U, const double* S,
                         const double* V, int norm, uint64_t entry_limit, double* out);
int frpca_pc_correlation(frpca_ctx* ctx, int64_t m, int64_t k, const double* U_test, const double* U_ref,
                         double* corr);
int frpca_projector_distance(frpca_ctx* ctx, int64_t m, int64_t k1, const double* Q1, int64_t k2,
                             const double* Q2, double* out);

/* One-shot run from a host CSR (upload, run, release): the reference-facing
 * call for a matrix that is not kept on the device. The sketch depends only on
 * the seed and the shape, so it is generated on a second stream while the CSR
 * is uploaded and validated and the transpose is built. Same arguments,
 * outputs and errors as frpca_dmat_upload + frpca_run; single GPU. */
int frpca_run_csr(frpca_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                  const int64_t* col_idx, const double* values, int algorithm, const frpca_config* cfg,
                  const double* omega, int64_t omega_rows, int64_t omega_cols, double* U, double* S,
                  double* V, double* basis, frpca_stats* stats, int* dispatched);

/* ---- timing helpers (device-side events on the ctx stream) ---------------- */
/* Last-run per-kernel accounting: name, launches, total device ms, algorithmic
 * bytes and flops (for the roofline report). idx out of range -> 2. */
int frpca_profile_enable(frpca_ctx* ctx, int enable);
int frpca_profile_count(frpca_ctx* ctx, int* n);
int frpca_profile_get(frpca_ctx* ctx, int idx, const char** name, int64_t* launches,
                      double* ms, double* bytes, double* flops);
int frpca_profile_reset(frpca_ctx* ctx);
/* Device-time bracket on the ctx stream (CUDA events): begin, then end returns
 * the elapsed milliseconds between the two events. */
int frpca_timer_begin(frpca_ctx* ctx);
int frpca_timer_end(frpca_ctx* ctx, double* ms);
/* Number of kernels this library has launched in this process (all contexts). */
int frpca_launch_count(uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* FRPCA_B200_H */
