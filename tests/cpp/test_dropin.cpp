// Drop-in check: reference-style code (the assertions of proj/tests/
// test_sparse.cpp, test_dense_kernels.cpp and test_randsvd.cpp for the hot
// path) compiled against include/frpca/frpca.hpp and run on the B200.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>
#include <algorithm>

#include "frpca/frpca.hpp"

using frpca::Index;
using Csr = frpca::SparseMatrixCsr<double>;
using Matrix = frpca::Matrix<double>;

static int failures = 0;
#define CHECK(c)                                                            \
    do {                                                                    \
        if (!(c)) { std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); ++failures; } \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try { f(); } catch (const E&) { return true; } catch (...) { return false; }
    return false;
}

static Csr diag_sparse(const std::vector<double>& v, Index rows, Index cols) {
    std::vector<Csr::Triplet> e;
    for (Index i = 0; i < Index(v.size()); ++i) e.push_back({i, i, v[size_t(i)]});
    return Csr::from_triplets(rows, cols, e);
}

static frpca::PcaConfig make_config(Index k, Index s, Index q, std::uint64_t seed = 0) {
    frpca::PcaConfig c;
    c.k = k; c.oversample = s; c.passes = q; c.seed = seed;
    return c;
}

int main() {
    // test_sparse.cpp:28-36
    Csr A = Csr::from_triplets(3, 3, {{1, 2, 3.0}, {0, 1, 1.0}, {1, 2, -1.0}, {0, 0, 2.0}, {2, 0, 5.0}, {2, 0, -5.0}});
    CHECK(A.nonZeros() == 3);
    CHECK((A.rowPtr() == std::vector<Index>{0, 2, 3, 3}));
    // test_sparse.cpp:38-44
    CHECK((throws<std::invalid_argument>([] { Csr(2, 2, {0, 2, 1}, {0, 1}, {1.0, 1.0}); })));
    CHECK((throws<std::invalid_argument>([] { Csr(2, 2, {0, 1, 2}, {0, 5}, {1.0, 1.0}); })));
    // test_sparse.cpp:68-81 (spmm_transpose hand expansion)
    Csr B = Csr::from_triplets(2, 3, {{0, 0, 1.0}, {0, 2, 2.0}, {1, 1, 3.0}});
    Matrix y(2, 1);
    y(0, 0) = 1; y(1, 0) = 1;
    Matrix z = frpca::spmm_transpose(B, y);
    CHECK(z(0, 0) == 1.0 && z(1, 0) == 3.0 && z(2, 0) == 2.0);
    // test_sparse.cpp:111-118 (pass counter)
    Csr R = diag_sparse({1, 2, 3, 4}, 4, 4);
    R.resetPassCount();
    Matrix X = Matrix::Identity(4, 2);
    frpca::spmm(R, X);
    frpca::spmm_transpose(R, X);
    CHECK(R.passCount() == 2);
    // test_dense_kernels.cpp:71-75, :104-109
    Matrix I53 = Matrix::Identity(5, 3);
    CHECK(frpca::lu_basis(I53) == I53);
    Matrix D(4, 2);
    for (int i = 0; i < 4; ++i) { D(i, 0) = 1.0 + i; D(i, 1) = -3.0 * (1.0 + i); }
    CHECK((throws<frpca::NumericalError>([&] { frpca::lu_basis(D); })));
    // test_dense_kernels.cpp:15-21
    CHECK(frpca::gaussian_matrix<double>(17, 9, 123) == frpca::gaussian_matrix<double>(17, 9, 123));
    CHECK(frpca::gaussian_matrix<double>(17, 9, 123) != frpca::gaussian_matrix<double>(17, 9, 124));
    // test_randsvd.cpp:71-85
    auto r1 = frpca::frpca(diag_sparse({5, 4, 3, 2, 1}, 5, 8), make_config(2, 3, 6));
    CHECK(std::abs(r1.S(0) - 5.0) < 1e-8 && std::abs(r1.S(1) - 4.0) < 1e-8);
    auto r2 = frpca::frpcat(diag_sparse({5, 4, 3, 2, 1}, 8, 5), make_config(2, 3, 11));
    CHECK(std::abs(r2.S(0) - 5.0) < 1e-8 && std::abs(r2.S(1) - 4.0) < 1e-8);
    // test_randsvd.cpp:106-111
    Csr Z = Csr::from_triplets(6, 6, {});
    CHECK((throws<frpca::NumericalError>([&] { frpca::frpcat(Z, make_config(2, 1, 4)); })));
    // test_randsvd.cpp:182-190 (auto dispatch), :192-209 (pass accounting)
    Csr W = diag_sparse({5, 4, 3, 2, 1, 0.5, 0.25}, 7, 9);
    CHECK(frpca::auto_pca(W, make_config(2, 2, 4)).dispatched == frpca::PcaAlgorithm::Frpca);
    for (Index q : {2, 3, 4, 5, 6, 9, 11}) {
        frpca::RunStats<double> st;
        frpca::frpca(W, make_config(2, 2, q), &st);
        CHECK(st.passes_over_matrix == std::uint64_t(q));
    }
    // test_randsvd.cpp:253-262 (preconditions)
    CHECK((throws<std::invalid_argument>([&] { frpca::frpca(W, make_config(7, 5, 4)); })));
    CHECK((throws<std::invalid_argument>([&] { frpca::frpca(W, make_config(2, 2, 1)); })));
    CHECK((throws<std::invalid_argument>([&] { frpca::frpcat(W, make_config(2, 2, 4)); })));
    // test_randsvd.cpp:264-271 (bitwise determinism)
    auto a = frpca::frpca(W, make_config(2, 2, 5, 2024));
    auto b = frpca::frpca(W, make_config(2, 2, 5, 2024));
    CHECK(a.S == b.S && a.U == b.U && a.V == b.V);
    // baselines (randsvd.hpp:95-175) and orth (dense_kernels.hpp:30-48)
    {
        frpca::PcaConfig cd = make_config(2, 3, 0);  // test_randsvd.cpp:55-69: q = 0, p = 2
        cd.power = 2;
        auto b1 = frpca::basic_rpca(diag_sparse({5, 4, 3, 2, 1}, 5, 5), cd);
        CHECK(std::abs(b1.S(0) - 5.0) < 1e-8 && std::abs(b1.S(1) - 4.0) < 1e-8);
        auto b2 = frpca::basic_rpcat(diag_sparse({5, 4, 3, 2, 1}, 5, 5), cd);
        CHECK(std::abs(b2.S(0) - 5.0) < 1e-8 && std::abs(b2.S(1) - 4.0) < 1e-8);
        frpca::RunStats<double> st;
        frpca::PcaConfig c = make_config(2, 2, 2);
        c.power = 3;
        frpca::basic_rpca(W, c, &st);
        CHECK(st.passes_over_matrix == 8u);
        frpca::Matrix<double> M(2, 1);
        M(0, 0) = 3.0;
        M(1, 0) = 4.0;
        auto Qm = frpca::orth(M);
        CHECK(std::abs(std::abs(Qm(0, 0)) - 0.6) < 1e-15 && std::abs(std::abs(Qm(1, 0)) - 0.8) < 1e-15);
        CHECK((throws<frpca::NumericalError>([&] { frpca::orth(frpca::Matrix<double>(4, 2)); })));
    }
    // Matrix Market round trip (matrix_market.hpp:27-116)
    {
        const std::string path = "/tmp/frpca_dropin_test.mtx";
        frpca::write_matrix_market(path, W);
        auto L = frpca::load_matrix_market<double>(path);
        CHECK(L.rows() == W.rows() && L.cols() == W.cols());
        CHECK(L.rowPtr() == W.rowPtr() && L.colIdx() == W.colIdx() && L.values() == W.values());
        CHECK((throws<frpca::IoError>([] { frpca::load_matrix_market<double>("/nonexistent/x.mtx"); })));
    }
    // validation metrics (validation.hpp:170-282): zero factors give |A|
    {
        Csr D2 = diag_sparse({3.0, 4.0}, 2, 2);
        frpca::SvdResult<double> z;
        z.U = frpca::Matrix<double>(2, 1);
        z.U(0, 0) = 1.0;
        z.S = frpca::Vector<double>(1);
        z.V = z.U;
        CHECK(std::abs(frpca::low_rank_error(D2, z, frpca::ErrorNorm::Frobenius) - 5.0) < 1e-12);
        CHECK(std::abs(frpca::low_rank_error(D2, z, frpca::ErrorNorm::Spectral) - 4.0) < 1e-8);
        frpca::Matrix<double> Q1(6, 2), Q2(6, 2);
        Q1(0, 0) = Q1(1, 1) = 1.0;
        Q2(2, 0) = Q2(3, 1) = 1.0;
        CHECK(std::abs(frpca::projector_distance(Q1, Q2) - 1.0) < 1e-10);
    }
    // several devices: the same calls shard A over a group. The
    // device listed twice selects the loopback collective, so the sharded
    // path runs on one GPU; results agree with the single-device run.
    {
        std::vector<Csr::Triplet> e;
        std::uint64_t st = 12345;
        auto next = [&] { st = st * 6364136223846793005ull + 1442695040888963407ull; return st >> 11; };
        for (int t = 0; t < 60000; ++t)
            e.push_back({Index(next() % 4000), Index(next() % 900), double(next() % 1000) / 250.0 - 2.0});
        Csr T = Csr::from_triplets(4000, 900, e);
        frpca::PcaConfig c = make_config(10, 10, 4, 7);
        auto one = frpca::frpcat(T, c);
        const auto p0 = T.passCount();
        frpca::b200::set_devices({0, 0});
        frpca::RunStats<double> rs;
        auto two = frpca::frpcat(T, c, &rs);
        CHECK(rs.passes_over_matrix == 4u && T.passCount() == p0 + 4);
        double smax = 0.0;
        for (Index i = 0; i < 10; ++i) smax = std::max(smax, std::abs(two.S(i, 0) - one.S(i, 0)) / one.S(i, 0));
        CHECK(smax <= 1e-10);
        // |U1^T U2| has singular values ~1: check the diagonal of the
        // cross-Gram after sign alignment is ~1 for the well-separated top PCs
        double d0 = 0.0;
        for (Index i = 0; i < T.rows(); ++i) d0 += one.U(i, 0) * two.U(i, 0);
        CHECK(std::abs(std::abs(d0) - 1.0) < 1e-8);
        auto Tt = frpca::transpose(T);
        auto onet = frpca::frpca(Tt, c);  // column-sharded frpca on the wide matrix
        frpca::b200::set_devices({0});
        auto onet1 = frpca::frpca(Tt, c);
        double s2 = 0.0;
        for (Index i = 0; i < 10; ++i) s2 = std::max(s2, std::abs(onet.S(i, 0) - onet1.S(i, 0)) / onet1.S(i, 0));
        CHECK(s2 <= 1e-10);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
