// Drop-in C++ API of the B200 frPCA / frPCAt hot path.
//
// Mirrors the reference's public interface for this path
// (/root/reference/proj/include/frpca/{types,sparse_matrix,dense_kernels,randsvd}.hpp)
// for Scalar = double: same namespace, names, argument conventions and
// exceptions, so code written against the reference's frpca(), frpcat(),
// auto_pca(), basic_rpca(), basic_rpcat(), spmm(), spmm_transpose(),
// lu_basis(), orth(), eig_svd(), load_matrix_market(), write_matrix_market(),
// gaussian_matrix() compiles against this header and runs on a B200.
//
// What differs, by necessity: Eigen is not available, so Matrix<double> /
// Vector<double> are a minimal column-major stand-in exposing the surface the
// hot path uses (rows(), cols(), data(), operator(), size()). All compute goes
// through the C ABI (include/frpca_b200.h, libfrpca_b200.so); there is no CPU
// path. Link with -L<pkg>/lib -lfrpca_b200.
#pragma once

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../frpca_b200.h"

namespace frpca {

using Index = std::int64_t;  // types.hpp:10 (Eigen::Index)

// ---- types.hpp:19-30 --------------------------------------------------------
class IoError : public std::runtime_error {
public:
    explicit IoError(const std::string& what) : std::runtime_error(what) {}
};
class NumericalError : public std::runtime_error {
public:
    explicit NumericalError(const std::string& what) : std::runtime_error(what) {}
};
class DeviceError : public std::runtime_error {
public:
    explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
inline void require(bool condition, const char* message) {  // types.hpp:45-47
    if (!condition) throw std::invalid_argument(message);
}
inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t tag) {  // types.hpp:52-57
    std::uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// Status of the C ABI -> the reference's exception types.
inline void check(int status) {
    if (status == FRPCA_OK) return;
    const std::string msg = frpca_last_error();
    switch (status) {
        case FRPCA_ERR_INVALID: throw std::invalid_argument(msg);
        case FRPCA_ERR_NUMERICAL: throw NumericalError(msg);
        case FRPCA_ERR_IO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}
}  // namespace detail

// ---- Matrix / Vector: column-major dense storage (types.hpp:12-16) --------
template <typename Scalar>
class Matrix {
public:
    Matrix() = default;
    Matrix(Index r, Index c) : rows_(r), cols_(c), d_(std::size_t(r) * std::size_t(c), Scalar(0)) {}
    static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
    static Matrix Identity(Index r, Index c) {
        Matrix m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = Scalar(1);
        return m;
    }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    Index outerStride() const { return rows_; }
    Scalar* data() { return d_.data(); }
    const Scalar* data() const { return d_.data(); }
    Scalar& operator()(Index i, Index j) { return d_[std::size_t(i + j * rows_)]; }
    Scalar operator()(Index i, Index j) const { return d_[std::size_t(i + j * rows_)]; }
    Scalar& operator()(Index i) { return d_[std::size_t(i)]; }
    Scalar operator()(Index i) const { return d_[std::size_t(i)]; }
    void resize(Index r, Index c) { rows_ = r; cols_ = c; d_.assign(std::size_t(r) * std::size_t(c), Scalar(0)); }
    bool operator==(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_ && d_ == o.d_; }
    bool operator!=(const Matrix& o) const { return !(*this == o); }

private:
    Index rows_ = 0, cols_ = 0;
    std::vector<Scalar> d_;
};

template <typename Scalar>
class Vector : public Matrix<Scalar> {
public:
    Vector() = default;
    explicit Vector(Index n) : Matrix<Scalar>(n, 1) {}
};

// SvdResult (types.hpp:34-41)
template <typename Scalar>
struct SvdResult {
    Matrix<Scalar> U;
    Vector<Scalar> S;
    Matrix<Scalar> V;
    Index rank() const { return S.size(); }
};

// ---- device context ----------------------------------------------------------
namespace b200 {
class Context {
public:
    explicit Context(int device = 0) { detail::check(frpca_ctx_create(device, &h_)); }
    ~Context() { if (h_) frpca_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    frpca_ctx* get() const { return h_; }
    static Context& default_context() {
        static Context c(0);
        return c;
    }

private:
    frpca_ctx* h_ = nullptr;
};

// Devices the drop-in runs frpca / frpcat on (the reference's
// callers are single-process, frpca_cli.cpp:158-183). Default: the list in
// FRPCA_DEVICES ("0,1,2,3"), else device 0 alone. With several devices the
// calls shard A over a group (frpca_group_run_csr: row blocks for frpcat,
// column blocks for frpca, NCCL between the GPUs); a device listed twice uses
// the host-staged loopback collective (testing the sharded path on one GPU).
class Group {
public:
    explicit Group(const std::vector<int>& devices) {
        frpca::detail::check(frpca_group_create(devices.data(), int(devices.size()), FRPCA_COMM_AUTO, &h_));
    }
    ~Group() { if (h_) frpca_group_destroy(h_); }
    Group(const Group&) = delete;
    Group& operator=(const Group&) = delete;
    frpca_group* get() const { return h_; }

private:
    frpca_group* h_ = nullptr;
};

namespace internal {
struct DeviceSet {
    std::mutex mu;
    std::vector<int> devices;
    std::unique_ptr<Group> group;
    DeviceSet() {
        if (const char* e = std::getenv("FRPCA_DEVICES")) {
            std::string s(e);
            std::size_t pos = 0;
            while (pos < s.size()) {
                const std::size_t q = s.find(',', pos);
                const std::string t = s.substr(pos, q == std::string::npos ? std::string::npos : q - pos);
                if (!t.empty()) devices.push_back(std::stoi(t));
                if (q == std::string::npos) break;
                pos = q + 1;
            }
        }
        if (devices.empty()) devices.push_back(0);
    }
    static DeviceSet& get() {
        static DeviceSet d;
        return d;
    }
};
}  // namespace internal

inline void set_devices(std::vector<int> devices) {
    frpca::detail::require(!devices.empty(), "set_devices: empty device list");
    auto& d = internal::DeviceSet::get();
    std::lock_guard<std::mutex> lk(d.mu);
    d.devices = std::move(devices);
    d.group.reset();
}

inline std::vector<int> devices() {
    auto& d = internal::DeviceSet::get();
    std::lock_guard<std::mutex> lk(d.mu);
    return d.devices;
}

// the group over devices() (created on first use; null for one device)
inline Group* default_group() {
    auto& d = internal::DeviceSet::get();
    std::lock_guard<std::mutex> lk(d.mu);
    if (d.devices.size() < 2) return nullptr;
    if (!d.group) d.group = std::make_unique<Group>(d.devices);
    return d.group.get();
}
}  // namespace b200

// ---- SparseMatrixCsr<double> (sparse_matrix.hpp:19-150) --------------------
template <typename Scalar>
class SparseMatrixCsr {
    static_assert(std::is_same_v<Scalar, double>, "the B200 path is fp64 (SparseMatrixCsr<double>)");

public:
    struct Triplet {
        Index row;
        Index col;
        Scalar value;
    };

    SparseMatrixCsr() : rows_(0), cols_(0), row_ptr_{0} {}
    SparseMatrixCsr(Index rows, Index cols, std::vector<Index> row_ptr, std::vector<Index> col_idx,
                    std::vector<Scalar> values)
        : rows_(rows), cols_(cols), row_ptr_(std::move(row_ptr)), col_idx_(std::move(col_idx)),
          values_(std::move(values)) {
        validate();
    }
    SparseMatrixCsr(const SparseMatrixCsr& o)
        : rows_(o.rows_), cols_(o.cols_), row_ptr_(o.row_ptr_), col_idx_(o.col_idx_), values_(o.values_) {}
    SparseMatrixCsr& operator=(const SparseMatrixCsr& o) {
        rows_ = o.rows_; cols_ = o.cols_; row_ptr_ = o.row_ptr_; col_idx_ = o.col_idx_; values_ = o.values_;
        dev_.reset();
        return *this;
    }
    SparseMatrixCsr(SparseMatrixCsr&&) noexcept = default;
    SparseMatrixCsr& operator=(SparseMatrixCsr&&) noexcept = default;

    // sparse_matrix.hpp:62-95
    static SparseMatrixCsr from_triplets(Index rows, Index cols, std::vector<Triplet> entries) {
        detail::require(rows >= 0 && cols >= 0, "from_triplets: negative dimension");
        for (const Triplet& t : entries)
            detail::require(t.row >= 0 && t.row < rows && t.col >= 0 && t.col < cols,
                            "from_triplets: entry out of bounds");
        std::stable_sort(entries.begin(), entries.end(), [](const Triplet& a, const Triplet& b) {
            return a.row != b.row ? a.row < b.row : a.col < b.col;
        });
        std::vector<Index> row_ptr(std::size_t(rows) + 1, 0), col_idx;
        std::vector<Scalar> values;
        std::size_t i = 0;
        while (i < entries.size()) {
            const Index r = entries[i].row, c = entries[i].col;
            Scalar sum = Scalar(0);
            while (i < entries.size() && entries[i].row == r && entries[i].col == c) sum += entries[i++].value;
            if (sum != Scalar(0)) {
                col_idx.push_back(c);
                values.push_back(sum);
                ++row_ptr[std::size_t(r) + 1];
            }
        }
        for (Index r = 0; r < rows; ++r) row_ptr[std::size_t(r) + 1] += row_ptr[std::size_t(r)];
        return SparseMatrixCsr(rows, cols, std::move(row_ptr), std::move(col_idx), std::move(values));
    }

    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index nonZeros() const { return Index(values_.size()); }
    const std::vector<Index>& rowPtr() const { return row_ptr_; }
    const std::vector<Index>& colIdx() const { return col_idx_; }
    const std::vector<Scalar>& values() const { return values_; }

    Matrix<Scalar> toDense() const {
        Matrix<Scalar> d(rows_, cols_);
        for (Index i = 0; i < rows_; ++i)
            for (Index p = row_ptr_[std::size_t(i)]; p < row_ptr_[std::size_t(i) + 1]; ++p)
                d(i, col_idx_[std::size_t(p)]) = values_[std::size_t(p)];
        return d;
    }

    // Pass counter (sparse_matrix.hpp:119-122), kept by the device copy.
    std::uint64_t passCount() const {
        std::uint64_t v = 0;
        if (dev_) detail::check(frpca_dmat_pass_count(dev_->h, &v));
        return v + passes_offset_;
    }
    void resetPassCount() const {
        if (dev_) detail::check(frpca_dmat_reset_pass_count(dev_->h));
        passes_offset_ = 0;
    }
    // passes made by a sharded run (the group's shards, not this device copy)
    void recordPasses(std::uint64_t n) const { passes_offset_ += n; }

    // The device copy (CSR + transposed CSR + work lists), built on first use.
    frpca_dmat* device(b200::Context& ctx = b200::Context::default_context()) const {
        std::lock_guard<std::mutex> lk(*mu_);
        if (!dev_ || dev_->ctx != &ctx) {
            auto d = std::make_shared<Dev>();
            d->ctx = &ctx;
            detail::check(frpca_dmat_upload(ctx.get(), rows_, cols_, nonZeros(), row_ptr_.data(),
                                            col_idx_.data(), values_.data(), &d->h));
            if (dev_) passes_offset_ += passCount();
            dev_ = d;
        }
        return dev_->h;
    }

private:
    void validate() const {  // sparse_matrix.hpp:125-142
        detail::require(rows_ >= 0 && cols_ >= 0, "csr: negative dimension");
        detail::require(row_ptr_.size() == std::size_t(rows_) + 1, "csr: row_ptr length must be rows + 1");
        detail::require(row_ptr_.front() == 0, "csr: row_ptr[0] must be 0");
        detail::require(row_ptr_.back() == Index(values_.size()), "csr: row_ptr[rows] must equal nnz");
        detail::require(col_idx_.size() == values_.size(), "csr: col_idx/values length mismatch");
        for (Index i = 0; i < rows_; ++i) {
            detail::require(row_ptr_[std::size_t(i)] <= row_ptr_[std::size_t(i) + 1],
                            "csr: row_ptr must be non-decreasing");
            for (Index p = row_ptr_[std::size_t(i)]; p < row_ptr_[std::size_t(i) + 1]; ++p) {
                detail::require(col_idx_[std::size_t(p)] >= 0 && col_idx_[std::size_t(p)] < cols_,
                                "csr: column index out of range");
                if (p > row_ptr_[std::size_t(i)])
                    detail::require(col_idx_[std::size_t(p) - 1] < col_idx_[std::size_t(p)],
                                    "csr: column indices must be strictly increasing within a row");
            }
        }
    }

    struct Dev {
        frpca_dmat* h = nullptr;
        b200::Context* ctx = nullptr;
        ~Dev() { if (h) frpca_dmat_destroy(h); }
    };
    Index rows_, cols_;
    std::vector<Index> row_ptr_, col_idx_;
    std::vector<Scalar> values_;
    mutable std::shared_ptr<Dev> dev_;
    mutable std::uint64_t passes_offset_ = 0;
    mutable std::shared_ptr<std::mutex> mu_ = std::make_shared<std::mutex>();
};

// ---- kernels (sparse_matrix.hpp:177-267, dense_kernels.hpp:16-174) ---------
template <typename Scalar>
Matrix<Scalar> spmm(const SparseMatrixCsr<Scalar>& A, const Matrix<Scalar>& X) {
    detail::require(X.rows() == A.cols(), "spmm: inner dimensions do not match");
    auto& ctx = b200::Context::default_context();
    Matrix<Scalar> Y(A.rows(), X.cols());
    detail::check(frpca_spmm(ctx.get(), A.device(ctx), 0, X.data(), std::max<Index>(X.rows(), 1),
                             X.cols(), Y.data()));
    return Y;
}

template <typename Scalar>
Matrix<Scalar> spmm_transpose(const SparseMatrixCsr<Scalar>& A, const Matrix<Scalar>& Y) {
    detail::require(Y.rows() == A.rows(), "spmm_transpose: inner dimensions do not match");
    auto& ctx = b200::Context::default_context();
    Matrix<Scalar> Z(A.cols(), Y.cols());
    detail::check(frpca_spmm(ctx.get(), A.device(ctx), 1, Y.data(), std::max<Index>(Y.rows(), 1),
                             Y.cols(), Z.data()));
    return Z;
}

template <typename Scalar>
SparseMatrixCsr<Scalar> transpose(const SparseMatrixCsr<Scalar>& A) {
    auto& ctx = b200::Context::default_context();
    std::vector<Index> rp(std::size_t(A.cols()) + 1), ci(std::size_t(A.nonZeros()));
    std::vector<Scalar> va(std::size_t(A.nonZeros()));
    detail::check(frpca_dmat_get_transpose(A.device(ctx), rp.data(), ci.data(), va.data()));
    return SparseMatrixCsr<Scalar>(A.cols(), A.rows(), std::move(rp), std::move(ci), std::move(va));
}

template <typename Scalar>
Matrix<Scalar> gaussian_matrix(Index rows, Index cols, std::uint64_t seed) {
    detail::require(rows >= 1 && cols >= 1, "gaussian_matrix: dimensions must be >= 1");
    Matrix<Scalar> G(rows, cols);
    detail::check(frpca_gaussian_matrix(b200::Context::default_context().get(), rows, cols, seed, G.data()));
    return G;
}

template <typename Scalar>
Matrix<Scalar> lu_basis(const Matrix<Scalar>& M) {
    detail::require(M.rows() >= M.cols() && M.cols() >= 1, "lu_basis: input must be tall (rows >= cols >= 1)");
    Matrix<Scalar> X(M.rows(), M.cols());
    detail::check(frpca_lu_basis(b200::Context::default_context().get(), M.rows(), M.cols(), M.data(), X.data()));
    return X;
}

// dense_kernels.hpp:30-48
template <typename Scalar>
Matrix<Scalar> orth(const Matrix<Scalar>& M) {
    detail::require(M.rows() >= M.cols() && M.cols() >= 1, "orth: input must be tall (rows >= cols >= 1)");
    Matrix<Scalar> Q(M.rows(), M.cols());
    detail::check(frpca_orth(b200::Context::default_context().get(), M.rows(), M.cols(), M.data(), Q.data()));
    return Q;
}

template <typename Scalar>
struct EigSvdResult {  // dense_kernels.hpp:136-143
    Matrix<Scalar> U;
    Vector<Scalar> S;  // ascending
    Matrix<Scalar> V;
};

template <typename Scalar>
EigSvdResult<Scalar> eig_svd(const Matrix<Scalar>& A) {
    detail::require(A.rows() >= A.cols() && A.cols() >= 1, "eig_svd: input must be tall (rows >= cols >= 1)");
    EigSvdResult<Scalar> r;
    r.U = Matrix<Scalar>(A.rows(), A.cols());
    r.S = Vector<Scalar>(A.cols());
    r.V = Matrix<Scalar>(A.cols(), A.cols());
    detail::check(frpca_eig_svd(b200::Context::default_context().get(), A.rows(), A.cols(), A.data(),
                                r.U.data(), r.S.data(), r.V.data()));
    return r;
}

// ---- matrix_market.hpp (the load step) -------------------------
// load_matrix_market (:27-93): the parse runs on the host (parallel chunks),
// from_triplets (sparse_matrix.hpp:62-95) on the device.
template <typename Scalar = double>
SparseMatrixCsr<Scalar> load_matrix_market(const std::string& path) {
    frpca_mtx* h = nullptr;
    int64_t rows = 0, cols = 0, n = 0;
    detail::check(frpca_mtx_read(path.c_str(), &h, &rows, &cols, &n));
    std::vector<int64_t> r(static_cast<size_t>(n)), c(static_cast<size_t>(n));
    std::vector<double> v(static_cast<size_t>(n));
    const int st = frpca_mtx_entries(h, r.data(), c.data(), v.data());
    frpca_mtx_free(h);
    detail::check(st);
    std::vector<Index> rp(static_cast<size_t>(rows) + 1), ci(static_cast<size_t>(std::max<int64_t>(n, 1)));
    std::vector<Scalar> va(static_cast<size_t>(std::max<int64_t>(n, 1)));
    int64_t nnz = 0;
    detail::check(frpca_csr_from_triplets(b200::Context::default_context().get(), rows, cols, n, r.data(),
                                          c.data(), v.data(), &nnz, rp.data(), ci.data(), va.data()));
    ci.resize(static_cast<size_t>(nnz));
    va.resize(static_cast<size_t>(nnz));
    return SparseMatrixCsr<Scalar>(rows, cols, std::move(rp), std::move(ci), std::move(va));
}

// write_matrix_market (:95-116): general coordinate, %.17g values
template <typename Scalar>
void write_matrix_market(const std::string& path, const SparseMatrixCsr<Scalar>& A) {
    detail::check(frpca_mtx_write(path.c_str(), A.rows(), A.cols(), A.rowPtr().data(), A.colIdx().data(),
                                  A.values().data()));
}

// ---- randsvd.hpp -------------------------------------------------------------
enum class PcaAlgorithm { BasicRpca, BasicRpcat, EigSvds, Frpca, Frpcat, Auto };  // :14

struct PcaConfig {  // :28-40
    Index k = 0;
    Index oversample = 5;
    Index passes = 2;
    Index power = 0;
    std::uint64_t seed = 0;
    bool deterministic = false;
    Index sketch_width() const { return k + oversample; }
};

template <typename Scalar>
struct RunStats {  // :42-53
    double sketch_seconds = 0.0;
    double power_seconds = 0.0;
    double finalize_seconds = 0.0;
    std::uint64_t passes_over_matrix = 0;
    bool capture_basis = false;
    Matrix<Scalar> basis;
};

template <typename Scalar>
struct AutoPcaResult {  // :331-334
    SvdResult<Scalar> svd;
    PcaAlgorithm dispatched = PcaAlgorithm::Auto;
};

namespace detail {
template <typename Scalar>
SvdResult<Scalar> run(int algo, const SparseMatrixCsr<Scalar>& A, const PcaConfig& cfg,
                      RunStats<Scalar>* stats, const Matrix<Scalar>* omega, int* dispatched) {
    frpca_config c{cfg.k, cfg.oversample, cfg.passes, cfg.power, cfg.seed, cfg.deterministic ? 1 : 0, 0u};
    const Index k = std::max<Index>(cfg.k, 0), l = cfg.k + cfg.oversample;
    int eff = algo == FRPCA_ALGO_AUTO ? (A.rows() < A.cols() ? FRPCA_ALGO_FRPCA : FRPCA_ALGO_FRPCAT) : algo;
    SvdResult<Scalar> out;
    out.U = Matrix<Scalar>(A.rows(), k);
    out.S = Vector<Scalar>(k);
    out.V = Matrix<Scalar>(A.cols(), k);
    Matrix<Scalar> basis;
    const bool want_basis = stats && stats->capture_basis && l >= 1;
    // several devices: the sharded group run (an injected sketch or a captured
    // basis keep the call on one device)
    if ((eff == FRPCA_ALGO_FRPCA || eff == FRPCA_ALGO_FRPCAT) && !omega && !want_basis) {
        if (b200::Group* g = b200::default_group()) {
            frpca_stats st{};
            detail::check(frpca_group_run_csr(g->get(), A.rows(), A.cols(), A.nonZeros(), A.rowPtr().data(),
                                              A.colIdx().data(), A.values().data(), algo, &c, out.U.data(),
                                              out.S.data(), out.V.data(), &st, dispatched));
            A.recordPasses(st.passes_over_matrix);
            if (stats) {
                stats->sketch_seconds = st.sketch_seconds;
                stats->power_seconds = st.power_seconds;
                stats->finalize_seconds = st.finalize_seconds;
                stats->passes_over_matrix = st.passes_over_matrix;
            }
            return out;
        }
    }
    auto& ctx = b200::Context::default_context();
    if (want_basis)
        basis = Matrix<Scalar>(eff == FRPCA_ALGO_FRPCA || eff == FRPCA_ALGO_BASIC_RPCA ? A.rows() : A.cols(), l);
    frpca_stats st{};
    detail::check(frpca_run(ctx.get(), A.device(ctx), algo, &c, omega ? omega->data() : nullptr,
                            omega ? omega->rows() : 0, omega ? omega->cols() : 0, out.U.data(),
                            out.S.data(), out.V.data(), want_basis ? basis.data() : nullptr, &st,
                            dispatched));
    if (stats) {
        stats->sketch_seconds = st.sketch_seconds;
        stats->power_seconds = st.power_seconds;
        stats->finalize_seconds = st.finalize_seconds;
        stats->passes_over_matrix = st.passes_over_matrix;
        if (want_basis) stats->basis = std::move(basis);
    }
    return out;
}
}  // namespace detail

// randsvd.hpp:99-102
template <typename Scalar>
SvdResult<Scalar> basic_rpca(const SparseMatrixCsr<Scalar>& A, const PcaConfig& cfg,
                             std::type_identity_t<RunStats<Scalar>>* stats = nullptr,
                             const std::type_identity_t<Matrix<Scalar>>* omega = nullptr) {
    return detail::run<Scalar>(FRPCA_ALGO_BASIC_RPCA, A, cfg, stats, omega, nullptr);
}

// randsvd.hpp:139-142
template <typename Scalar>
SvdResult<Scalar> basic_rpcat(const SparseMatrixCsr<Scalar>& A, const PcaConfig& cfg,
                              std::type_identity_t<RunStats<Scalar>>* stats = nullptr,
                              const std::type_identity_t<Matrix<Scalar>>* omega = nullptr) {
    return detail::run<Scalar>(FRPCA_ALGO_BASIC_RPCAT, A, cfg, stats, omega, nullptr);
}

// randsvd.hpp:229-232
template <typename Scalar>
SvdResult<Scalar> frpca(const SparseMatrixCsr<Scalar>& A, const PcaConfig& cfg,
                        std::type_identity_t<RunStats<Scalar>>* stats = nullptr,
                        const std::type_identity_t<Matrix<Scalar>>* omega = nullptr) {
    return detail::run<Scalar>(FRPCA_ALGO_FRPCA, A, cfg, stats, omega, nullptr);
}

// randsvd.hpp:281-284
template <typename Scalar>
SvdResult<Scalar> frpcat(const SparseMatrixCsr<Scalar>& A, const PcaConfig& cfg,
                         std::type_identity_t<RunStats<Scalar>>* stats = nullptr,
                         const std::type_identity_t<Matrix<Scalar>>* omega = nullptr) {
    return detail::run<Scalar>(FRPCA_ALGO_FRPCAT, A, cfg, stats, omega, nullptr);
}

// randsvd.hpp:336-351
template <typename Scalar>
AutoPcaResult<Scalar> auto_pca(const SparseMatrixCsr<Scalar>& A, const PcaConfig& cfg,
                               std::type_identity_t<RunStats<Scalar>>* stats = nullptr) {
    AutoPcaResult<Scalar> out;
    int d = -1;
    out.svd = detail::run<Scalar>(FRPCA_ALGO_AUTO, A, cfg, stats, nullptr, &d);
    out.dispatched = d == FRPCA_ALGO_FRPCA ? PcaAlgorithm::Frpca : PcaAlgorithm::Frpcat;
    return out;
}

// ---- validation.hpp: metrics on the GPU --------------------------
enum class ErrorNorm { Frobenius, Spectral };                      // :17
constexpr std::uint64_t kDefaultOracleEntryLimit = 4'000'000;      // :26

template <typename Scalar>
struct OracleSvd {  // :73-77 (computed by the caller; the metrics need S and U)
    Matrix<Scalar> U;
    Vector<Scalar> S;
    Matrix<Scalar> V;
};

// :170-203
template <typename Scalar>
Scalar low_rank_error(const SparseMatrixCsr<Scalar>& A, const SvdResult<Scalar>& r, ErrorNorm norm,
                      std::uint64_t entry_limit = kDefaultOracleEntryLimit) {
    detail::require(r.U.rows() == A.rows() && r.V.rows() == A.cols(), "low_rank_error: shape mismatch");
    detail::require(r.U.cols() == r.S.size() && r.V.cols() == r.S.size(),
                    "low_rank_error: inconsistent factor widths");
    auto& ctx = b200::Context::default_context();
    double out = 0.0;
    detail::check(frpca_low_rank_error(ctx.get(), A.device(ctx), r.S.size(), r.U.data(), r.S.data(), r.V.data(),
                                       norm == ErrorNorm::Spectral ? FRPCA_NORM_SPECTRAL : FRPCA_NORM_FROBENIUS,
                                       entry_limit, &out));
    return Scalar(out);
}

// :207-215
template <typename Scalar>
Scalar best_rank_k_error(const Vector<Scalar>& s, Index k, ErrorNorm norm) {
    detail::require(k >= 0, "best_rank_k_error: negative k");
    const Index n = s.size();
    if (k >= n) return Scalar(0);
    if (norm == ErrorNorm::Spectral) return s(k);
    Scalar acc = 0;
    for (Index i = k; i < n; ++i) acc += s(i) * s(i);
    return std::sqrt(acc);
}

// :228-246
template <typename Scalar>
Vector<Scalar> pc_correlation(const Matrix<Scalar>& U_test, const Matrix<Scalar>& U_ref) {
    detail::require(U_test.rows() == U_ref.rows() && U_test.cols() == U_ref.cols(), "pc_correlation: shape mismatch");
    detail::require(U_test.rows() >= 2, "pc_correlation: need at least two samples");
    Vector<Scalar> corr(U_test.cols());
    detail::check(frpca_pc_correlation(b200::Context::default_context().get(), U_test.rows(), U_test.cols(),
                                       U_test.data(), U_ref.data(), corr.data()));
    return corr;
}

// :264-282
template <typename Scalar>
Scalar projector_distance(const Matrix<Scalar>& Q1, const Matrix<Scalar>& Q2) {
    detail::require(Q1.rows() == Q2.rows(), "projector_distance: row mismatch");
    double out = 0.0;
    detail::check(frpca_projector_distance(b200::Context::default_context().get(), Q1.rows(), Q1.cols(), Q1.data(),
                                           Q2.cols(), Q2.data(), &out));
    return Scalar(out);
}

// :287-319 (to_json needs nlohmann::json, which this header does not pull in)
struct AccuracyReport {
    std::vector<double> singular_value_rel_err;
    double recon_err_frobenius = 0.0;
    double recon_err_spectral = 0.0;
    double best_rank_k_err = 0.0;
    double eps_equivalent = 0.0;
    std::vector<double> pc_correlations;
};

template <typename Scalar>
AccuracyReport make_accuracy_report(const SparseMatrixCsr<Scalar>& A, const SvdResult<Scalar>& r,
                                    const OracleSvd<Scalar>& oracle) {
    const Index k = r.S.size();
    detail::require(oracle.S.size() >= k, "make_accuracy_report: oracle has fewer values than k");
    AccuracyReport rep;
    rep.singular_value_rel_err.resize(static_cast<std::size_t>(k));
    for (Index i = 0; i < k; ++i) {
        const double ref = static_cast<double>(oracle.S(i));
        rep.singular_value_rel_err[static_cast<std::size_t>(i)] =
            ref == 0.0 ? std::abs(static_cast<double>(r.S(i))) : std::abs(static_cast<double>(r.S(i)) - ref) / ref;
    }
    rep.recon_err_frobenius = double(low_rank_error(A, r, ErrorNorm::Frobenius));
    rep.recon_err_spectral = double(low_rank_error(A, r, ErrorNorm::Spectral));
    rep.best_rank_k_err = double(best_rank_k_error(oracle.S, k, ErrorNorm::Spectral));
    rep.eps_equivalent = rep.best_rank_k_err == 0.0 ? 0.0 : rep.recon_err_spectral / rep.best_rank_k_err - 1.0;
    Matrix<Scalar> Uk(oracle.U.rows(), k);
    std::memcpy(Uk.data(), oracle.U.data(), sizeof(Scalar) * std::size_t(oracle.U.rows() * k));
    Vector<Scalar> corr = pc_correlation(r.U, Uk);
    rep.pc_correlations.assign(corr.data(), corr.data() + corr.size());
    return rep;
}

}  // namespace frpca
