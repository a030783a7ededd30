// ARBITER — TEST INFRASTRUCTURE ONLY (like oracle.cpp; see its header).
//
// The frpca / frpcat pipelines of the reference (randsvd.hpp:224-328) computed
// in 80-bit long double (64-bit significand), from the same CSR and the same
// fp64 sketch Omega. It is the "truth" against which two fp64 evaluations of
// the algorithm (the GPU path and the oracle) are compared when they disagree
// with each other by more than a tolerance: each fp64 evaluation's distance
// from this pipeline is its own rounding error, so the one closer to it is the
// more accurate (tools/parity_full.py --arbiter, tests/test_gpu_fullsize.py).
//
// Every step follows the reference's algorithm (spmm :177-206, spmm_transpose
// :208-240, lu_basis dense_kernels.hpp:50-116 with the same pivot rule and
// tolerance, eig_svd :145-174) with long double arithmetic throughout; the
// l x l eigenproblem is cyclic Jacobi (as the oracle), in long double. Summation
// orders are plain sequential sums: at 64-bit precision their rounding is
// ~2^-11 of the fp64 differences being judged.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace arb {

using Index = int64_t;
using R = long double;

static int g_threads = 1;

template <class F>
static void parallel_for(Index b, Index e, F&& f) {
    const Index n = e - b;
    const int t = int(std::min<Index>(g_threads, n));
    if (t <= 1) { for (Index i = b; i < e; ++i) f(i); return; }
    std::vector<std::thread> pool;
    std::atomic<Index> next{b};
    for (int w = 0; w < t; ++w)
        pool.emplace_back([&] {
            for (Index i = next.fetch_add(1); i < e; i = next.fetch_add(1)) f(i);
        });
    for (auto& th : pool) th.join();
}

// row-major r x c
struct Mat {
    Index rows = 0, cols = 0;
    std::vector<R> d;
    Mat() = default;
    Mat(Index r, Index c) : rows(r), cols(c), d(size_t(r) * size_t(c), R(0)) {}
    R* row(Index i) { return d.data() + size_t(i) * size_t(cols); }
    const R* row(Index i) const { return d.data() + size_t(i) * size_t(cols); }
    R& operator()(Index i, Index j) { return d[size_t(i) * size_t(cols) + size_t(j)]; }
    R operator()(Index i, Index j) const { return d[size_t(i) * size_t(cols) + size_t(j)]; }
};

struct Csr {
    Index rows, cols;
    const int64_t *rp, *ci;
    const double* v;
};

// Y = A X (sparse_matrix.hpp:195-203: per entry a sum over the row in CSR order)
static Mat spmm(const Csr& A, const Mat& X) {
    Mat Y(A.rows, X.cols);
    const Index l = X.cols;
    parallel_for(0, (A.rows + 255) / 256, [&](Index b) {
        for (Index i = b * 256; i < std::min(A.rows, b * 256 + 256); ++i) {
            R* y = Y.row(i);
            for (Index p = A.rp[i]; p < A.rp[i + 1]; ++p) {
                const R vp = A.v[p];
                const R* x = X.row(A.ci[p]);
                for (Index c = 0; c < l; ++c) y[c] += vp * x[c];
            }
        }
    });
    return Y;
}

// Z = A^T Y (sparse_matrix.hpp:229-237: ascending rows, zeros of y skipped)
static Mat spmm_t(const Csr& A, const Mat& Y) {
    Mat Z(A.cols, Y.cols);
    const Index l = Y.cols;
    const Index W = std::max<Index>(4, (l + g_threads - 1) / g_threads);
    parallel_for(0, (l + W - 1) / W, [&](Index t) {
        const Index c0 = t * W, c1 = std::min(l, c0 + W);
        for (Index i = 0; i < A.rows; ++i) {
            const R* y = Y.row(i);
            for (Index p = A.rp[i]; p < A.rp[i + 1]; ++p) {
                R* z = Z.row(A.ci[p]);
                const R vp = A.v[p];
                for (Index c = c0; c < c1; ++c)
                    if (y[c] != 0) z[c] += vp * y[c];
            }
        }
    });
    return Z;
}

// lu_basis (dense_kernels.hpp:50-116): first-max pivots, tol = l eps max|M|
// (eps of double, as the reference's Scalar), returns P^T L.
static Mat lu_basis(const Mat& M) {
    const Index m = M.rows, l = M.cols;
    Mat W = M;
    std::vector<Index> perm{}; perm.resize(size_t(m));
    std::iota(perm.begin(), perm.end(), Index(0));
    R mx = 0;
    for (R x : W.d) mx = std::max(mx, std::fabs(x));
    const R tol = R(l) * R(std::numeric_limits<double>::epsilon()) * mx;
    for (Index j = 0; j < l; ++j) {
        Index piv = j;
        R best = std::fabs(W(j, j));
        for (Index i = j + 1; i < m; ++i) {
            const R v = std::fabs(W(i, j));
            if (v > best) { best = v; piv = i; }
        }
        if (best <= tol) throw std::runtime_error("arbiter lu_basis: zero pivot");
        if (piv != j) {
            std::swap_ranges(W.row(j), W.row(j) + l, W.row(piv));
            std::swap(perm[size_t(j)], perm[size_t(piv)]);
        }
        const R d = W(j, j);
        const R* uj = W.row(j);
        parallel_for(0, (m - j - 1 + 1023) / 1024, [&](Index b) {
            for (Index i = j + 1 + b * 1024; i < std::min(m, j + 1 + b * 1024 + 1024); ++i) {
                R* wi = W.row(i);
                wi[j] /= d;
                const R f = wi[j];
                for (Index c = j + 1; c < l; ++c) wi[c] -= f * uj[c];
            }
        });
    }
    Mat X(m, l);
    for (Index i = 0; i < m; ++i) {
        const Index r = perm[size_t(i)];
        for (Index j = 0; j < std::min(i + 1, l); ++j) X(r, j) = (j == i) ? R(1) : W(i, j);
    }
    return X;
}

// cyclic Jacobi on a symmetric n x n (row-major), eigenvalues ascending
static void eig_sym(Mat A, Mat& V, std::vector<R>& D) {
    const Index n = A.rows;
    V = Mat(n, n);
    for (Index i = 0; i < n; ++i) V(i, i) = 1;
    const R eps = std::numeric_limits<R>::epsilon();
    for (int sweep = 0; sweep < 80; ++sweep) {
        bool rotated = false;
        for (Index p = 0; p < n - 1; ++p)
            for (Index q = p + 1; q < n; ++q) {
                const R apq = A(p, q), app = A(p, p), aqq = A(q, q);
                if (std::fabs(apq) <= eps * std::sqrt(std::fabs(app * aqq))) continue;
                rotated = true;
                const R theta = (aqq - app) / (2 * apq);
                const R t = (theta >= 0 ? R(1) : R(-1)) / (std::fabs(theta) + std::sqrt(1 + theta * theta));
                const R c = 1 / std::sqrt(1 + t * t), s = t * c;
                for (Index k = 0; k < n; ++k) {
                    const R akp = A(k, p), akq = A(k, q);
                    A(k, p) = c * akp - s * akq;
                    A(k, q) = s * akp + c * akq;
                }
                for (Index k = 0; k < n; ++k) {
                    const R apk = A(p, k), aqk = A(q, k);
                    A(p, k) = c * apk - s * aqk;
                    A(q, k) = s * apk + c * aqk;
                }
                A(p, q) = A(q, p) = 0;
                for (Index k = 0; k < n; ++k) {
                    const R vkp = V(k, p), vkq = V(k, q);
                    V(k, p) = c * vkp - s * vkq;
                    V(k, q) = s * vkp + c * vkq;
                }
            }
        if (!rotated) break;
    }
    std::vector<Index> ord{}; ord.resize(size_t(n));
    std::iota(ord.begin(), ord.end(), Index(0));
    std::stable_sort(ord.begin(), ord.end(), [&](Index a, Index b) { return A(a, a) < A(b, b); });
    D.resize(size_t(n));
    Mat Vs(n, n);
    for (Index j = 0; j < n; ++j) {
        D[size_t(j)] = A(ord[size_t(j)], ord[size_t(j)]);
        for (Index i = 0; i < n; ++i) Vs(i, j) = V(i, ord[size_t(j)]);
    }
    V = std::move(Vs);
}

struct EigSvd {
    Mat U;  // r x l
    std::vector<R> S;
    Mat V;  // l x l
};

// eig_svd (dense_kernels.hpp:145-174): Gram, eigensolve, rank check, U = W V S^-1
static EigSvd eig_svd(const Mat& W) {
    const Index r = W.rows, n = W.cols;
    Mat B(n, n);
    const Index nb = std::max<Index>(1, std::min<Index>(g_threads * 4, (r + 4095) / 4096));
    std::vector<Mat> parts(size_t(nb), Mat(n, n));
    parallel_for(0, nb, [&](Index b) {
        Mat& P = parts[size_t(b)];
        for (Index i = r * b / nb; i < r * (b + 1) / nb; ++i) {
            const R* w = W.row(i);
            for (Index a = 0; a < n; ++a) {
                const R wa = w[a];
                R* pa = P.row(a);
                for (Index c = 0; c <= a; ++c) pa[c] += wa * w[c];
            }
        }
    });
    for (auto& P : parts)
        for (Index a = 0; a < n; ++a)
            for (Index c = 0; c <= a; ++c) B(a, c) += P(a, c);
    for (Index a = 0; a < n; ++a)
        for (Index c = a + 1; c < n; ++c) B(a, c) = B(c, a);
    EigSvd out;
    std::vector<R> D;
    eig_sym(B, out.V, D);
    if (D[size_t(n - 1)] <= 0 || D[0] <= R(n) * R(std::numeric_limits<double>::epsilon()) * D[size_t(n - 1)])
        throw std::runtime_error("arbiter eig_svd: rank deficient");
    out.S.resize(size_t(n));
    for (Index j = 0; j < n; ++j) out.S[size_t(j)] = std::sqrt(D[size_t(j)]);
    Mat Ms(n, n);
    for (Index i = 0; i < n; ++i)
        for (Index j = 0; j < n; ++j) Ms(i, j) = out.V(i, j) / out.S[size_t(j)];
    out.U = Mat(r, n);
    parallel_for(0, (r + 255) / 256, [&](Index b) {
        for (Index i = b * 256; i < std::min(r, b * 256 + 256); ++i) {
            const R* w = W.row(i);
            R* u = out.U.row(i);
            for (Index t = 0; t < n; ++t) {
                const R wt = w[t];
                const R* mt = Ms.row(t);
                for (Index j = 0; j < n; ++j) u[j] += wt * mt[j];
            }
        }
    });
    return out;
}

static Mat from_colmajor(const double* p, Index r, Index c) {
    Mat M(r, c);
    for (Index i = 0; i < r; ++i)
        for (Index j = 0; j < c; ++j) M(i, j) = p[i + j * r];
    return M;
}

static Mat matmul(const Mat& A, const Mat& B) {  // small right factor
    Mat C(A.rows, B.cols);
    parallel_for(0, (A.rows + 255) / 256, [&](Index b) {
        for (Index i = b * 256; i < std::min(A.rows, b * 256 + 256); ++i)
            for (Index t = 0; t < A.cols; ++t) {
                const R a = A(i, t);
                for (Index j = 0; j < B.cols; ++j) C(i, j) += a * B(t, j);
            }
    });
    return C;
}

// Output columns ind = s+k-1 ... s (randsvd.hpp:262-267 / :314-319)
static void out_cols(const Mat& M, Index s, Index k, double* dst) {
    for (Index t = 0; t < k; ++t)
        for (Index i = 0; i < M.rows; ++i) dst[i + t * M.rows] = double(M(i, s + k - 1 - t));
}

}  // namespace arb

using namespace arb;

static thread_local std::string g_err;

extern "C" {

const char* arb_last_error(void) { return g_err.c_str(); }
void arb_set_threads(int t) { g_threads = t < 1 ? 1 : t; }

// algo 0 = frpca (Alg. 5), 1 = frpcat (Alg. 6); omega: the fp64 sketch of the
// run (column-major, the shape sketch_matrix draws: randsvd.hpp:239-247 /
// :291-299); U (rows x k), S (k), V (cols x k) column-major, descending.
int arb_pca(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci, const double* v, int algo,
            int64_t k, int64_t s, int64_t q, const double* omega, double* U, double* S, double* V) {
    try {
        const Csr A{rows, cols, rp, ci, v};
        const Index l = k + s, loops = (q - 1) / 2;
        Mat Q;
        if (algo == 1) {  // frpcat, randsvd.hpp:278-328
            if (q % 2 == 0) {
                Mat OmT(rows, l);  // Omega is l x rows column-major == Omega^T row-major
                for (Index i = 0; i < rows; ++i)
                    for (Index c = 0; c < l; ++c) OmT(i, c) = omega[c + i * l];
                Mat Y = spmm_t(A, OmT);
                Q = (q == 2) ? eig_svd(Y).U : lu_basis(Y);
            } else {
                Q = from_colmajor(omega, cols, l);
            }
            for (Index i = 1; i <= loops; ++i) {
                Mat Z = spmm_t(A, spmm(A, Q));
                Q = (i == loops) ? eig_svd(Z).U : lu_basis(Z);
            }
            EigSvd f = eig_svd(spmm(A, Q));
            out_cols(f.U, s, k, U);
            out_cols(matmul(Q, f.V), s, k, V);
            for (Index t = 0; t < k; ++t) S[t] = double(f.S[size_t(s + k - 1 - t)]);
        } else {  // frpca, randsvd.hpp:224-276
            if (q % 2 == 0) {
                Mat Y = spmm(A, from_colmajor(omega, cols, l));
                Q = (q > 2) ? lu_basis(Y) : eig_svd(Y).U;
            } else {
                Q = from_colmajor(omega, rows, l);
            }
            for (Index i = 1; i <= loops; ++i) {
                Mat Y = spmm(A, spmm_t(A, Q));
                Q = (i == loops) ? eig_svd(Y).U : lu_basis(Y);
            }
            EigSvd f = eig_svd(spmm_t(A, Q));
            out_cols(matmul(Q, f.V), s, k, U);
            out_cols(f.U, s, k, V);
            for (Index t = 0; t < k; ++t) S[t] = double(f.S[size_t(s + k - 1 - t)]);
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

}  // extern "C"
