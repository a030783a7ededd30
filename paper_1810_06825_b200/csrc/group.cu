// Host-side shard plan of the sharded path, shared by the
// single-process group run (abi.cu frpca_group_run_csr) and the one-process-
// per-GPU launch (paper_1810_06825_b200/shard.py calls these through the C ABI).
//
// frpcat (rows >= cols): contiguous row blocks balanced by nnz + rows (the SpMM
// work of a row is its nnz plus one output-row write); the n x l A^T*Y
// partials and the l x l Gram partials are summed across ranks.
// frpca (rows <= cols): column blocks (a row-block sharding of A^T) balanced by
// column nnz + 1, shipped as local CSRs with local column ids; the m x l A*X
// partials and the Gram partials are summed across ranks.
#include <thread>

#include "driver.cuh"

namespace fb {
namespace {

template <class F>
void host_parallel(int64_t n, F&& f) {
    const int t = int(std::max<int64_t>(1, std::min<int64_t>(n, std::max(1u, std::thread::hardware_concurrency()))));
    std::vector<std::thread> pool;
    for (int w = 0; w < t; ++w)
        pool.emplace_back([&, w] {
            for (int64_t i = n * w / t; i < n * (w + 1) / t; ++i) f(i);
        });
    for (auto& th : pool) th.join();
}

}  // namespace

void shard_cuts(int64_t rows, int64_t cols, const int64_t* row_ptr, const int64_t* col_idx, int col_shard,
                int world, int64_t* cuts) {
    require(world >= 1, "shard: world must be >= 1");
    if (!col_shard) {
        // weights w[i] = row_ptr[i] + i (nnz + rows before row i); cut r is the
        // first i with w[i] >= total * r / world
        const double total = double(row_ptr[rows] + rows);
        cuts[0] = 0;
        for (int r = 1; r < world; ++r) {
            const double t = total * r / world;
            int64_t lo = 0, hi = rows + 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) / 2;
                if (double(row_ptr[mid] + mid) < t) lo = mid + 1;
                else hi = mid;
            }
            cuts[r] = lo;
        }
        cuts[world] = rows;
        return;
    }
    // column weights nnz(c) + 1; pref[c] = sum of weights of columns < c
    const int64_t nnz = row_ptr[rows];
    const int nt = int(std::max(1u, std::min(64u, std::thread::hardware_concurrency())));
    std::vector<std::vector<int64_t>> part(size_t(nt), std::vector<int64_t>(size_t(cols), 0));
    host_parallel(nt, [&](int64_t t) {
        std::vector<int64_t>& h = part[size_t(t)];
        for (int64_t p = nnz * t / nt; p < nnz * (t + 1) / nt; ++p) ++h[size_t(col_idx[p])];
    });
    std::vector<double> pref(size_t(cols) + 1, 0.0);
    for (int64_t c = 0; c < cols; ++c) {
        int64_t cnt = 0;
        for (int t = 0; t < nt; ++t) cnt += part[size_t(t)][size_t(c)];
        pref[size_t(c) + 1] = pref[size_t(c)] + double(cnt) + 1.0;
    }
    cuts[0] = 0;
    for (int r = 1; r < world; ++r)
        cuts[r] = int64_t(std::lower_bound(pref.begin(), pref.end(), pref[size_t(cols)] * r / world) - pref.begin());
    cuts[world] = cols;
}

void shard_extract_cols(int64_t rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                        int64_t c0, int64_t c1, std::vector<int64_t>& lrp, std::vector<int64_t>& lci,
                        std::vector<double>& lva) {
    // each row's entries with c0 <= col < c1 are one contiguous run (ids are
    // strictly increasing within a row)
    std::vector<int64_t> b(static_cast<size_t>(rows)), e(static_cast<size_t>(rows));
    host_parallel((rows + 4095) / 4096, [&](int64_t blk) {
        for (int64_t i = blk * 4096; i < std::min(rows, blk * 4096 + 4096); ++i) {
            const int64_t* s = col_idx + row_ptr[i];
            const int64_t* t = col_idx + row_ptr[i + 1];
            b[size_t(i)] = int64_t(std::lower_bound(s, t, c0) - col_idx);
            e[size_t(i)] = int64_t(std::lower_bound(s, t, c1) - col_idx);
        }
    });
    lrp.assign(size_t(rows) + 1, 0);
    for (int64_t i = 0; i < rows; ++i) lrp[size_t(i) + 1] = lrp[size_t(i)] + (e[size_t(i)] - b[size_t(i)]);
    lci.resize(size_t(lrp[size_t(rows)]));
    lva.resize(size_t(lrp[size_t(rows)]));
    host_parallel((rows + 4095) / 4096, [&](int64_t blk) {
        for (int64_t i = blk * 4096; i < std::min(rows, blk * 4096 + 4096); ++i) {
            int64_t o = lrp[size_t(i)];
            for (int64_t p = b[size_t(i)]; p < e[size_t(i)]; ++p, ++o) {
                lci[size_t(o)] = col_idx[p] - c0;
                lva[size_t(o)] = values[p];
            }
        }
    });
}

}  // namespace fb
