// Device CSR at load time: upload + validation (sparse_matrix.hpp:125-142),
// transposed CSR (sparse_matrix.hpp:242-267, moved from a test helper to the
// load step so A^T*Y is a gather, never an atomic scatter), and the
// load-balanced SpMM work lists of both.
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "internal.cuh"

namespace fb {
namespace {

constexpr unsigned long long kNoError = ~0ull;

// Row-level check of validate() (:131): row_ptr non-decreasing. Records the
// first offending row (atomicMin keeps it deterministic).
__global__ void k_check_rowptr(const int64_t* __restrict__ rp, int64_t m,
                               unsigned long long* __restrict__ bad_row) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x)
        if (rp[i] > rp[i + 1]) atomicMin(bad_row, (unsigned long long)i);
}

// Marks the first nonzero of each (valid) row with its row id; an inclusive
// max-scan then yields the row id of every nonzero.
__global__ void k_mark_rows(const int64_t* __restrict__ rp, int64_t m_valid,
                            int32_t* __restrict__ mark) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m_valid;
         i += int64_t(gridDim.x) * blockDim.x)
        if (rp[i + 1] > rp[i]) mark[rp[i]] = int32_t(i);
}

// Per-nonzero checks of validate() (:132-138) fused with the int64 -> int32
// narrowing of the column ids. Key = (row << 33) | (2*offset + kind) so the
// minimum is the first failure in the reference's scan order.
__global__ void k_check_cols(const int64_t* __restrict__ rp, const int32_t* __restrict__ rowid,
                             const int64_t* __restrict__ col64, int64_t nnz_valid, int64_t ncols,
                             int32_t* __restrict__ col32, unsigned long long* __restrict__ err) {
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < nnz_valid;
         p += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = col64[p];
        const int64_t r = rowid[p];
        const int64_t off = p - rp[r];
        if (c < 0 || c >= ncols) {
            atomicMin(err, ((unsigned long long)r << 33) | (unsigned long long)(2 * off + 1));
            col32[p] = 0;
            continue;
        }
        col32[p] = int32_t(c);
        if (off > 0 && !(col64[p - 1] < c))
            atomicMin(err, ((unsigned long long)r << 33) | (unsigned long long)(2 * off + 2));
    }
}

// sort payload of nonzero i: (row id << 32) | i
__global__ void k_pack_rows(const int32_t* __restrict__ rowid, int64_t n, uint64_t* __restrict__ pay) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        pay[i] = (uint64_t(uint32_t(rowid[i])) << 32) | uint64_t(uint32_t(i));
}

// sorted payload -> A^T's column ids (the row ids) and the permutation
__global__ void k_unpack_rows(const uint64_t* __restrict__ pay, int64_t n, int32_t* __restrict__ tcol,
                              int32_t* __restrict__ perm) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n;
         k += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t v = pay[k];
        tcol[k] = int32_t(v >> 32);
        perm[k] = int32_t(uint32_t(v));
    }
}

// Transposed entries from the stable column sort: entry k of A^T is original
// nonzero perm[k]; its column id in A^T is the original row id, its value the
// original value. Random gathers: eight independent loads in flight per
// thread (one per 32-byte sector), so the kernel is not bound by a single
// load's latency.
template <class T>
__global__ void __launch_bounds__(256)
k_gather_perm(const int32_t* __restrict__ perm, const T* __restrict__ src, int64_t n, T* __restrict__ dst) {
    constexpr int U = 8;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * U;
    for (int64_t k0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * U; k0 < n; k0 += stride) {
        if (k0 + U <= n) {
            const int4 a = __ldcs(reinterpret_cast<const int4*>(perm + k0));
            const int4 b = __ldcs(reinterpret_cast<const int4*>(perm + k0 + 4));
            const int idx[U] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            T v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldg(src + idx[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) __stcs(dst + k0 + u, v[u]);
        } else {
            for (int64_t k = k0; k < n; ++k) dst[k] = src[perm[k]];
        }
    }
}

// t_rowptr[c] = lower_bound(sorted_keys, c), c in [0, n].
__global__ void k_rowptr_from_sorted(const int32_t* __restrict__ keys, int64_t nnz, int64_t n,
                                     int64_t* __restrict__ trp) {
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c <= n;
         c += int64_t(gridDim.x) * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < c) lo = mid + 1; else hi = mid;
        }
        trp[c] = lo;
    }
}

// ---- work lists --------------------------------------------------------------
// Row r is "long" if it has more than `ch` nonzeros: it is cut into chunks of
// ch nonzeros (one item each) whose partial sums are combined in order.
// Short rows are grouped: row r starts a group unless its predecessor is a
// short row in the same bin, bin(r) = (row_ptr[r] + r) / ch (weight of a row
// = nnz + 1 for its output write), so a group carries <= ~ch of weight.
__device__ __forceinline__ bool is_long(const int64_t* rp, int64_t r, int64_t ch, const uint8_t* skip) {
    return !(skip && skip[r]) && rp[r + 1] - rp[r] > ch;
}
__device__ __forceinline__ bool is_start(const int64_t* rp, int64_t r, int64_t ch, const uint8_t* skip) {
    if (is_long(rp, r, ch, skip)) return false;
    if (r == 0) return true;
    if (is_long(rp, r - 1, ch, skip)) return true;
    return (rp[r] + r) / ch != (rp[r - 1] + r - 1) / ch;
}

__global__ void k_item_counts(const int64_t* __restrict__ rp, int64_t m, int64_t ch,
                              int32_t* __restrict__ n_items, int32_t* __restrict__ n_slots,
                              int32_t* __restrict__ n_comb, const uint8_t* __restrict__ skip) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m;
         r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t nz = rp[r + 1] - rp[r];
        if (is_long(rp, r, ch, skip)) {
            const int32_t k = int32_t((nz + ch - 1) / ch);
            n_items[r] = k; n_slots[r] = k; n_comb[r] = 1;
        } else {
            n_items[r] = is_start(rp, r, ch, skip) ? 1 : 0; n_slots[r] = 0; n_comb[r] = 0;
        }
    }
}

// chunk cuts of an item list (ItemList::cut_*): for k = 1..kCuts-1 the row r
// of item k nitems / kCuts and the item / combine offsets of that row
// chunk cuts at rows k m / kCuts: a function of the row count alone, so every
// rank of a sharded run (same output rows, its own items) cuts its reduced
// output identically. The first item of chunk k is the first item starting
// at or after its row (o_items counts the items of the rows before it); an
// item straddling the cut (a group of short rows) finishes in chunk k - 1.
__global__ void k_item_cuts(int64_t m, const int32_t* __restrict__ o_items, const int32_t* __restrict__ o_comb,
                            int64_t* __restrict__ out) {
    const int k = threadIdx.x;
    if (k < 1 || k >= kCuts) return;
    const int64_t r = int64_t(k) * m / kCuts;
    out[3 * k] = r;
    out[3 * k + 1] = o_items[r];
    out[3 * k + 2] = o_comb[r];
}

__global__ void k_item_write(const int64_t* __restrict__ rp, int64_t m, int64_t ch,
                             const int32_t* __restrict__ o_items, const int32_t* __restrict__ o_slots,
                             const int32_t* __restrict__ o_comb, WorkItem* __restrict__ items,
                             Combine* __restrict__ comb, const uint8_t* __restrict__ skip) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m;
         r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p0 = rp[r], nz = rp[r + 1] - p0;
        if (is_long(rp, r, ch, skip)) {
            const int32_t k = int32_t((nz + ch - 1) / ch);
            const int32_t s0 = o_slots[r];
            for (int32_t t = 0; t < k; ++t) {
                WorkItem w;
                w.p0 = p0 + int64_t(t) * ch;
                w.p1 = min(p0 + int64_t(t + 1) * ch, p0 + nz);
                w.r0 = int32_t(r);
                w.r1 = -(s0 + t) - 1;
                items[o_items[r] + t] = w;
            }
            Combine cb;
            cb.row = int32_t(r); cb.s0 = s0; cb.s1 = s0 + k; cb.pad = 0;
            comb[o_comb[r]] = cb;
        } else if (is_start(rp, r, ch, skip)) {
            int64_t e = r + 1;
            while (e < m && !is_long(rp, e, ch, skip) && !is_start(rp, e, ch, skip)) ++e;
            WorkItem w;
            w.p0 = 0; w.p1 = 0; w.r0 = int32_t(r); w.r1 = int32_t(e);
            items[o_items[r]] = w;
        }
    }
}

// n elements of d into the context's mapped host words (read_scalar)
template <class T>
__global__ void k_put(const T* __restrict__ src, int n, T* __restrict__ dst) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

uint64_t* mapped_slots(Ctx& c, int n) {
    constexpr int kSlots = 64;
    if (n > kSlots) throw CudaError("mapped_slots: too many words");
    if (!c.mapped.h) {
        void* h = nullptr;
        FB_CUDA(cudaHostAlloc(&h, sizeof(uint64_t) * kSlots, cudaHostAllocMapped));
        c.mapped.h = static_cast<uint64_t*>(h);
        void* d = nullptr;
        FB_CUDA(cudaHostGetDevicePointer(&d, h, 0));
        c.mapped.d = static_cast<uint64_t*>(d);
    }
    return c.mapped.h;
}

int grid_for(const Ctx& c, int64_t n, int threads = 256) {
    const int64_t want = (n + threads - 1) / threads;
    const int64_t cap = int64_t(c.num_sms) * 32;
    return int(std::max<int64_t>(1, std::min(want, cap)));
}

template <class T>
T read_scalar(Ctx& c, const T* d) {
    static_assert(sizeof(T) <= sizeof(uint64_t), "scalar read-back");
    static const bool dbg = std::getenv("FRPCA_DEBUG_E2E") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    uint64_t* slot = mapped_slots(c, 1);
    k_put<T><<<1, 32, 0, c.stream>>>(d, 1, reinterpret_cast<T*>(c.mapped.d));
    FB_LAUNCH_CHECK();
    const auto t1 = std::chrono::steady_clock::now();
    FB_CUDA(cudaStreamSynchronize(c.stream));
    if (dbg) {
        const auto t2 = std::chrono::steady_clock::now();
        const double a = std::chrono::duration<double, std::milli>(t1 - t0).count();
        const double b = std::chrono::duration<double, std::milli>(t2 - t1).count();
        if (a + b > 5.0) std::fprintf(stderr, "[e2e] read_scalar: launch %.2f ms, sync %.2f ms\n", a, b);
    }
    T h;
    std::memcpy(&h, slot, sizeof(T));
    return h;
}

}  // namespace

// item weight: nonzeros + rows (the chunk of a long row, or a group of short rows)
__global__ void k_item_weights(const int64_t* __restrict__ rp, const WorkItem* __restrict__ items, int64_t n,
                               int64_t* __restrict__ w, int32_t* __restrict__ idx) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const WorkItem it = items[i];
        w[i] = it.r1 >= 0 ? (rp[it.r1] - rp[it.r0]) + (it.r1 - it.r0) : (it.p1 - it.p0) + 1;
        idx[i] = int32_t(i);
    }
}

__global__ void k_item_gather(const WorkItem* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                              WorkItem* __restrict__ dst) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = src[idx[i]];
}

// Within each chunk of the list (ItemList::cut_item), the heaviest items
// first: warps take items from a global counter, so the last ones handed out
// are the lightest and the launch's tail is short. Which warp runs an item
// does not enter any sum (results bitwise unchanged). FRPCA_ITEM_ORDER=0 keeps
// row order.
void order_items_heaviest_first(Ctx& c, const DCsr& A, ItemList& L) {
    const char* e = std::getenv("FRPCA_ITEM_ORDER");
    if ((e && e[0] == '0') || L.nitems < 2) return;
    cudaStream_t s = c.stream;
    const int64_t n = L.nitems;
    DBuf<int64_t> w(size_t(n), s), w2(size_t(n), s);
    DBuf<int32_t> idx(size_t(n), s), idx2(size_t(n), s);
    k_item_weights<<<grid_for(c, n), 256, 0, s>>>(A.rowptr.get(), L.items.get(), n, w.get(), idx.get());
    FB_LAUNCH_CHECK();
    std::vector<int32_t> hoff(L.cut_item.begin(), L.cut_item.end());
    DBuf<int32_t> doff(hoff.size(), s);
    FB_CUDA(cudaMemcpyAsync(doff.get(), hoff.data(), sizeof(int32_t) * hoff.size(), cudaMemcpyHostToDevice, s));
    const int nseg = int(hoff.size()) - 1;
    size_t tb = 0;
    FB_CUDA(cub::DeviceSegmentedSort::StableSortPairsDescending(nullptr, tb, w.get(), w2.get(), idx.get(), idx2.get(),
                                                                n, nseg, doff.get(), doff.get() + 1, s));
    DBuf<unsigned char> tmp(tb, s);
    FB_CUDA(cub::DeviceSegmentedSort::StableSortPairsDescending(tmp.get(), tb, w.get(), w2.get(), idx.get(),
                                                                idx2.get(), n, nseg, doff.get(), doff.get() + 1, s));
    DBuf<WorkItem> out(size_t(n), s);
    k_item_gather<<<grid_for(c, n), 256, 0, s>>>(L.items.get(), idx2.get(), n, out.get());
    FB_LAUNCH_CHECK();
    L.items = std::move(out);
    FB_CUDA(cudaStreamSynchronize(s));  // (hoff is host memory read by the copy)
}

void build_items(Ctx& c, const DCsr& A, const uint8_t* skip, ItemList& L, int64_t ch) {
    const int64_t m = A.rows;
    L.nitems = L.ncomb = L.nslots = 0;
    L.chunk = ch;
    if (m == 0) return;
    DBuf<int32_t> cnt(3 * (m + 1), c.stream), off(3 * (m + 1), c.stream);
    int32_t *ni = cnt.get(), *ns = ni + (m + 1), *nc = ns + (m + 1);
    int32_t *oi = off.get(), *os = oi + (m + 1), *oc = os + (m + 1);
    FB_CUDA(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), c.stream));
    k_item_counts<<<grid_for(c, m), 256, 0, c.stream>>>(A.rowptr.get(), m, ch, ni, ns, nc, skip);
    FB_LAUNCH_CHECK();
    size_t tb = 0;
    FB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, ni, oi, m + 1, c.stream));
    DBuf<unsigned char> tmp(tb, c.stream);
    FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, ni, oi, m + 1, c.stream));
    FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, ns, os, m + 1, c.stream));
    FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, nc, oc, m + 1, c.stream));
    L.nitems = read_scalar(c, oi + m);
    L.nslots = read_scalar(c, os + m);
    L.ncomb = read_scalar(c, oc + m);
    L.items.alloc(size_t(L.nitems), c.stream);
    L.comb.alloc(size_t(std::max<int64_t>(L.ncomb, 1)), c.stream);
    k_item_write<<<grid_for(c, m), 256, 0, c.stream>>>(A.rowptr.get(), m, ch, oi, os, oc, L.items.get(),
                                                        L.comb.get(), skip);
    FB_LAUNCH_CHECK();
    // chunk cuts (k_item_cuts); one small gather, one read
    L.cut_row.assign(1, 0);
    L.cut_item.assign(1, 0);
    L.cut_comb.assign(1, 0);
    {
        DBuf<int64_t> cv(3 * kCuts, c.stream);
        k_item_cuts<<<1, 32, 0, c.stream>>>(m, oi, oc, cv.get());
        FB_LAUNCH_CHECK();
        uint64_t* slots = mapped_slots(c, 3 * kCuts);
        k_put<int64_t><<<1, 32, 0, c.stream>>>(cv.get(), 3 * kCuts, reinterpret_cast<int64_t*>(c.mapped.d));
        FB_LAUNCH_CHECK();
        FB_CUDA(cudaStreamSynchronize(c.stream));
        int64_t h[3 * kCuts];
        std::memcpy(h, slots, sizeof(h));
        for (int k = 1; k < kCuts; ++k)
            if (h[3 * k] > L.cut_row.back()) {  // (rows only: the same cuts on every rank)
                L.cut_row.push_back(h[3 * k]);
                L.cut_item.push_back(h[3 * k + 1]);
                L.cut_comb.push_back(h[3 * k + 2]);
            }
    }
    L.cut_row.push_back(m);
    L.cut_item.push_back(L.nitems);
    L.cut_comb.push_back(L.ncomb);
    order_items_heaviest_first(c, A, L);
}

namespace {

// chunk size of the work lists: ~32 items per resident warp, clamped. With
// the heaviest items handed out first, finer items shorten the launch tails:
// per run C3 199.4 (16) -> 194.1 (32) -> 193.3 ms (64), C2 70.4 -> 69.7 ->
// 70.2, C4 306.4 (16) / 307.6 (48), C1 flat (profiles/r2_ab_item_size.json)
int64_t default_chunk(const Ctx& c, const DCsr& A) {
    const char* e = std::getenv("FRPCA_CHUNK_ITEMS");  // items per warp (A/B knob)
    const int64_t per = e && *e ? std::max(1, std::atoi(e)) : 32;
    const int64_t target = int64_t(c.num_sms) * 24 * per;
    const int64_t ch = (A.nnz + A.rows + target - 1) / target;
    return std::max<int64_t>(256, std::min<int64_t>(16384, ch));
}

__global__ void k_col_counts(const int64_t* __restrict__ trp, int64_t n, int32_t* __restrict__ cnt,
                             int32_t* __restrict__ ids) {
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n;
         c += int64_t(gridDim.x) * blockDim.x) {
        cnt[c] = int32_t(trp[c + 1] - trp[c]);
        ids[c] = int32_t(c);
    }
}

__global__ void k_rank_all(const int32_t* __restrict__ ids, int64_t n, int32_t* __restrict__ rank_of) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x)
        rank_of[ids[r]] = int32_t(r);
}

// Re-encode A's column ids for an A*X launch mode (DCsr::enc_*): ids of the
// sx_h most popular columns become kColHot | rank (their X rows are staged in
// shared memory by the sliced kernel), the next ones up to hint_h carry the
// sign bit (L2 evict_last hint), the rest are plain. The original id of any
// encoding is recovered through rank_ids.
__global__ void k_encode_cols(int32_t* __restrict__ col, int64_t nnz, const int32_t* __restrict__ rank_of,
                              const int32_t* __restrict__ rank_ids, int64_t hint_h, int64_t sx_h) {
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < nnz;
         p += int64_t(gridDim.x) * blockDim.x) {
        const int32_t e = col[p];
        const int32_t cc = (e & kColHot) ? rank_ids[e & kRankMask] : (e & kColMask);
        const int32_t r = rank_of[cc];
        col[p] = r < sx_h ? int32_t(kColHot | r) : (r < hint_h ? int32_t(uint32_t(cc) | 0x80000000u) : cc);
    }
}

// Popularity rank of every column of A (counts = row lengths of T), kept for
// the L2 hints of A*X.
void build_ranks(Ctx& c, int64_t n, const DCsr& T, DBuf<int32_t>& rank_of, DBuf<int32_t>& rank_ids) {
    if (n == 0 || T.nnz == 0) return;
    cudaStream_t s = c.stream;
    DBuf<int32_t> cnt(size_t(n), s), ids(size_t(n), s), cnt_s(size_t(n), s), ids_s(size_t(n), s);
    k_col_counts<<<grid_for(c, n), 256, 0, s>>>(T.rowptr.get(), n, cnt.get(), ids.get());
    FB_LAUNCH_CHECK();
    size_t tb = 0;
    FB_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, cnt.get(), cnt_s.get(), ids.get(),
                                                      ids_s.get(), n, 0, 32, s));
    DBuf<unsigned char> tmp(tb, s);
    FB_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.get(), tb, cnt.get(), cnt_s.get(), ids.get(),
                                                      ids_s.get(), n, 0, 32, s));
    rank_of.alloc(size_t(n), s);
    k_rank_all<<<grid_for(c, n), 256, 0, s>>>(ids_s.get(), n, rank_of.get());
    FB_LAUNCH_CHECK();
    rank_ids = std::move(ids_s);
}

// Structure of A^T (stable radix sort by column keeps ascending rows, the
// order spmm_transpose accumulates in, sparse_matrix.hpp:229-237): T.col,
// T.rowptr and the sort permutation (entry k of A^T is nonzero perm[k] of A),
// whose gather of the values comes last (they may still be crossing PCIe).
void transpose_structure(Ctx& c, const DCsr& A, DCsr& T, const int32_t* rowid, DBuf<int32_t>& perm_out) {
    cudaStream_t s = c.stream;
    const int64_t nnz = A.nnz, cols = A.cols;
    if (!nnz) {
        FB_CUDA(cudaMemsetAsync(T.rowptr.get(), 0, T.rowptr.bytes(), s));
        return;
    }
    // the sort carries (row id << 32 | nonzero index): A^T's column ids come
    // out of the sort directly, no random gather of the row ids
    std::unique_ptr<Prof> pt(new Prof(c, "upload_t_sort", 0, 0));
    DBuf<int32_t> keys_out(size_t(nnz), s);
    DBuf<uint64_t> pay_in(size_t(nnz), s), pay_out(size_t(nnz), s);
    k_pack_rows<<<grid_for(c, nnz), 256, 0, s>>>(rowid, nnz, pay_in.get());
    FB_LAUNCH_CHECK();
    int end_bit = 1;
    while (end_bit < 31 && (int64_t(1) << end_bit) <= cols) ++end_bit;
    size_t tb = 0;
    FB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, A.col.get(), keys_out.get(), pay_in.get(),
                                            pay_out.get(), nnz, 0, end_bit, s));
    DBuf<unsigned char> tmp(tb, s);
    FB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, A.col.get(), keys_out.get(), pay_in.get(),
                                            pay_out.get(), nnz, 0, end_bit, s));
    pay_in.release();
    pt.reset(new Prof(c, "upload_t_unpack", 0, 0));
    perm_out.alloc(size_t(nnz), s);
    k_unpack_rows<<<grid_for(c, nnz), 256, 0, s>>>(pay_out.get(), nnz, T.col.get(), perm_out.get());
    FB_LAUNCH_CHECK();
    k_rowptr_from_sorted<<<grid_for(c, cols + 1), 256, 0, s>>>(keys_out.get(), nnz, cols, T.rowptr.get());
    FB_LAUNCH_CHECK();
}

// The builder of a pipelined upload: its own stream, driven from the
// builder thread (PendingValues::builder)
Ctx& builder_ctx(Ctx& c) {
    if (!c.tside) {
        auto b = std::make_unique<Ctx>();
        b->device = c.device;
        b->num_sms = c.num_sms;
        // default (lowest) priority: the run's own kernels (the first A*X, the
        // LU of an even-q frpca) go first and the builder fills the gaps
        // (C4 e2e: the LU took 15.5 instead of 2.9 ms behind top-priority
        // builder kernels); FRPCA_BUILDER_PRIO=hi for the A/B
        int lo = 0, hi = 0;
        FB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const char* e = std::getenv("FRPCA_BUILDER_PRIO");
        FB_CUDA(cudaStreamCreateWithPriority(&b->stream, cudaStreamNonBlocking, (e && e[0] == 'h') ? hi : lo));
        c.tside = std::move(b);
    }
    return *c.tside;
}

const char* kValidateMsg[3] = {
    "csr: row_ptr must be non-decreasing",
    "csr: column index out of range",
    "csr: column indices must be strictly increasing within a row",
};

}  // namespace

// pipelined (frpca_run_csr): the values cross PCIe in kValChunks chunks on the
// copy stream and the call returns without waiting for them; A.pend / M.At.pend
// (PendingValues) tell the first product what to wait for.
constexpr int kValChunks = 8;

void PendingValues::join() {
    if (joined) return;
    joined = true;
    static const bool dbg = std::getenv("FRPCA_DEBUG_E2E") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    if (builder.joinable()) builder.join();
    if (dbg)
        std::fprintf(stderr, "[e2e] builder join waited %.2f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    if (a && rank_of.n) {
        a->rank_of = std::move(rank_of);
        a->rank_ids = std::move(rank_ids);
        a->hint_h = a->sx_h = 0;
    }
    if (err) std::rethrow_exception(err);
}

void consume_pending(Ctx& c, DCsr& A) {
    if (!A.pend) return;
    std::shared_ptr<PendingValues> pv = std::move(A.pend);
    pv->join();  // (the builder has recorded `all` once it is joined)
    if (!pv->ev.empty()) FB_CUDA(cudaStreamWaitEvent(c.stream, pv->ev.back(), 0));
    if (pv->all) FB_CUDA(cudaStreamWaitEvent(c.stream, pv->all, 0));
}

void dcsr_upload_build(Ctx& c, DMat& M, int64_t rows, int64_t cols, int64_t nnz,
                       const int64_t* h_rp, const int64_t* h_col, const double* h_val, int64_t width_hint,
                       bool pipelined) {
    // O(1) checks of validate() (sparse_matrix.hpp:126-130), same messages.
    require(rows >= 0 && cols >= 0, "csr: negative dimension");
    require(nnz >= 0, "csr: col_idx/values length mismatch");
    require(h_rp != nullptr, "csr: row_ptr length must be rows + 1");
    require(h_rp[0] == 0, "csr: row_ptr[0] must be 0");
    require(h_rp[rows] == nnz, "csr: row_ptr[rows] must equal nnz");
    require(rows < (int64_t(1) << 31) && cols < (int64_t(1) << 31) && nnz < (int64_t(1) << 31),
            "frpca_b200: rows, cols and nnz must each be < 2^31 per device");
    cudaStream_t s = c.stream;
    DCsr& A = M.A;
    A.rows = rows; A.cols = cols; A.nnz = nnz;
    A.rowptr.alloc(size_t(rows + 1), s);
    A.col.alloc(size_t(nnz), s);
    A.val.alloc(size_t(nnz), s);
    DBuf<int64_t> col64(size_t(nnz), s);
    std::unique_ptr<Prof> ph(new Prof(c, "upload_h2d", 8.0 * (rows + 1) + 16.0 * nnz, 0));
    FB_CUDA(cudaMemcpyAsync(A.rowptr.get(), h_rp, sizeof(int64_t) * (rows + 1),
                            cudaMemcpyHostToDevice, s));
    // the values are first needed by the transpose's gather: they cross PCIe
    // on the copy stream while the ids are validated and sorted
    cudaEvent_t ev_ids = nullptr, ev_val = nullptr;
    std::shared_ptr<PendingValues> pv;
    if (nnz) {
        FB_CUDA(cudaMemcpyAsync(col64.get(), h_col, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
        if (!c.copy) FB_CUDA(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
        FB_CUDA(cudaEventCreateWithFlags(&ev_ids, cudaEventDisableTiming));
        FB_CUDA(cudaEventCreateWithFlags(&ev_val, cudaEventDisableTiming));
        FB_CUDA(cudaEventRecord(ev_ids, s));
        FB_CUDA(cudaStreamWaitEvent(c.copy, ev_ids, 0));
        if (pipelined) {
            pv = std::make_shared<PendingValues>();
            const int64_t V = (nnz + kValChunks - 1) / kValChunks;
            for (int64_t v0 = 0; v0 < nnz; v0 += V) {
                const int64_t v1 = std::min(nnz, v0 + V);
                FB_CUDA(cudaMemcpyAsync(A.val.get() + v0, h_val + v0, sizeof(double) * (v1 - v0),
                                        cudaMemcpyHostToDevice, c.copy));
                cudaEvent_t e;
                FB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                pv->ev.push_back(e);
                FB_CUDA(cudaEventRecord(e, c.copy));
            }
        } else {
            FB_CUDA(cudaMemcpyAsync(A.val.get(), h_val, sizeof(double) * nnz, cudaMemcpyHostToDevice, c.copy));
        }
        FB_CUDA(cudaEventRecord(ev_val, c.copy));
    }
    struct EvGuard {
        cudaEvent_t& a;
        cudaEvent_t& b;
        cudaStream_t cs;
        ~EvGuard() {
            if (b) cudaStreamSynchronize(cs);  // an early throw must not leave the copy in flight
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } evg{ev_ids, ev_val, c.copy};
    ph.reset(new Prof(c, "upload_validate", 0, 0));
    std::unique_ptr<Prof> pv0(new Prof(c, "upload_v_rowptr", 0, 0));
    DBuf<unsigned long long> err(2, s);
    FB_CUDA(cudaMemsetAsync(err.get(), 0xff, err.bytes(), s));
    if (rows) {
        k_check_rowptr<<<grid_for(c, rows), 256, 0, s>>>(A.rowptr.get(), rows, err.get());
        FB_LAUNCH_CHECK();
    }
    const unsigned long long bad_row = read_scalar(c, err.get());
    const int64_t m_valid = bad_row == kNoError ? rows : int64_t(bad_row);
    int64_t nnz_valid = nnz;
    if (m_valid < rows) {
        int64_t tmp;
        FB_CUDA(cudaMemcpy(&tmp, A.rowptr.get() + m_valid, sizeof(int64_t), cudaMemcpyDeviceToHost));
        nnz_valid = std::min<int64_t>(tmp, nnz);
    }
    // row id of every nonzero (mark + inclusive max-scan)
    pv0.reset(new Prof(c, "upload_v_rowid", 0, 0));
    DBuf<int32_t> rowid(size_t(nnz), s);
    if (nnz) {
        DBuf<int32_t> mark(size_t(nnz), s);
        FB_CUDA(cudaMemsetAsync(mark.get(), 0, mark.bytes(), s));
        if (m_valid) {
            k_mark_rows<<<grid_for(c, m_valid), 256, 0, s>>>(A.rowptr.get(), m_valid, mark.get());
            FB_LAUNCH_CHECK();
        }
        size_t tb = 0;
        FB_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, mark.get(), rowid.get(), cub::Max(),
                                               nnz, s));
        DBuf<unsigned char> tmp(tb, s);
        FB_CUDA(cub::DeviceScan::InclusiveScan(tmp.get(), tb, mark.get(), rowid.get(), cub::Max(),
                                               nnz, s));
        pv0.reset(new Prof(c, "upload_v_cols", 0, 0));
        if (nnz_valid > 0) {
            k_check_cols<<<grid_for(c, nnz_valid), 256, 0, s>>>(
                A.rowptr.get(), rowid.get(), col64.get(), nnz_valid, cols, A.col.get(), err.get() + 1);
            FB_LAUNCH_CHECK();
        }
    }
    const unsigned long long key = read_scalar(c, err.get() + 1);
    pv0.reset();
    if (key != kNoError) {
        const int kind = (key & 1ull) ? 1 : 2;
        throw InvalidArgument(kValidateMsg[kind]);
    }
    if (m_valid < rows) throw InvalidArgument(kValidateMsg[0]);
    col64.release();
    DCsr& T = M.At;
    T.rows = cols; T.cols = rows; T.nnz = nnz;
    T.rowptr.alloc(size_t(cols + 1), s);
    T.col.alloc(size_t(nnz), s);
    T.val.alloc(size_t(nnz), s);
    if (nnz && pv) {
        // Pipelined: A^T's structure (the radix sort) and A's work list now,
        // while the values cross PCIe; the first A*X then starts on the value
        // chunks as they land. The column ranks, A^T's work list and panel
        // plan and the gather of A^T's values are built beside it by the
        // builder thread on its own stream, joined by the first A^T*Y
        // (consume_pending). (With the sort on the builder, its kernels
        // waited for the persistent A*X blocks of each chunk to drain: sort
        // 10 -> 32 ms, first A*X done at 169 instead of ~125 ms at C3.)
        ph.reset(new Prof(c, "upload_transpose", 0, 0));
        transpose_structure(c, A, T, rowid.get(), pv->perm);
        rowid.release();
        ph.reset(new Prof(c, "upload_items", 0, 0));
        build_items(c, A, nullptr, A.L, default_chunk(c, A));
        const int64_t V = (nnz + kValChunks - 1) / kValChunks;
        for (size_t k = 0; k + 1 < A.L.cut_row.size(); ++k) {
            const int64_t e = h_rp[A.L.cut_row[k + 1]];
            pv->need.push_back(int(e > 0 ? (e - 1) / V : 0));
        }
        ph.reset();
        Ctx& b = builder_ctx(c);
        b.prof = c.prof;  // (its brackets join the call's timeline, FRPCA_DEBUG_TIMELINE)
        b.tl_mark = b.pending.size();
        cudaEvent_t ev_ready;
        FB_CUDA(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
        FB_CUDA(cudaEventRecord(ev_ready, s));
        FB_CUDA(cudaEventCreateWithFlags(&pv->all, cudaEventDisableTiming));
        pv->a = &A;
        PendingValues* P = pv.get();
        const cudaEvent_t last = pv->ev.back();
        P->builder = std::thread([&b, &A, &T, P, ev_ready, last, width_hint] {
            try {
                FB_CUDA(cudaSetDevice(b.device));
                FB_CUDA(cudaStreamWaitEvent(b.stream, ev_ready, 0));
                cudaEventDestroy(ev_ready);
                build_ranks(b, A.cols, T, P->rank_of, P->rank_ids);
                build_items(b, T, nullptr, T.L, default_chunk(b, T));
                if (width_hint > 0) {
                    int64_t pr = 0, cap = 0;
                    if (panel_rows_for(T, width_hint, pr, cap)) ensure_panels(b, T, pr, cap);
                }
                FB_CUDA(cudaStreamWaitEvent(b.stream, last, 0));
                k_gather_perm<double><<<grid_for(b, (A.nnz + 7) / 8), 256, 0, b.stream>>>(P->perm.get(), A.val.get(),
                                                                                        A.nnz, T.val.get());
                P->perm.release();
                FB_LAUNCH_CHECK();
            } catch (...) {
                P->err = std::current_exception();
            }
            cudaEventRecord(P->all, b.stream);
        });
        A.pend = pv;
        T.pend = pv;
        FB_CUDA(cudaEventDestroy(ev_val));  // (the recorded work stays queued; the guard must not wait for it)
        ev_val = nullptr;
        return;
    }
    ph.reset(new Prof(c, "upload_transpose", 0, 0));
    DBuf<int32_t> perm_out;
    transpose_structure(c, A, T, rowid.get(), perm_out);
    rowid.release();
    ph.reset(new Prof(c, "upload_items", 0, 0));
    build_ranks(c, A.cols, T, A.rank_of, A.rank_ids);
    A.hint_h = A.sx_h = 0;
    build_items(c, A, nullptr, A.L, default_chunk(c, A));
    build_items(c, T, nullptr, T.L, default_chunk(c, T));
    if (width_hint > 0) {  // the panel plan of the A^T*Y the caller is about to run
        int64_t pr = 0, cap = 0;
        if (panel_rows_for(T, width_hint, pr, cap)) ensure_panels(c, T, pr, cap);
    }
    if (nnz) {
        ph.reset(new Prof(c, "upload_values", 0, 0));
        FB_CUDA(cudaStreamWaitEvent(s, ev_val, 0));
        k_gather_perm<double><<<grid_for(c, (nnz + 7) / 8), 256, 0, s>>>(perm_out.get(), A.val.get(), nnz, T.val.get());
        FB_LAUNCH_CHECK();
    }
    perm_out.release();
    ph.reset();
    FB_CUDA(cudaStreamSynchronize(s));
}

// ---- panelled A^T*Y plan (see PanelPlan in internal.cuh) ---------------------

namespace {

__global__ void k_hot_flags(const int64_t* __restrict__ rp, int64_t n, int64_t thot,
                            uint8_t* __restrict__ skip, int32_t* __restrict__ flag) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
         r += int64_t(gridDim.x) * blockDim.x) {
        const bool h = rp[r + 1] - rp[r] >= thot;
        skip[r] = h;
        flag[r] = h;
    }
}

__global__ void k_hot_list(const int32_t* __restrict__ flag, const int32_t* __restrict__ pos, int64_t n,
                           int32_t* __restrict__ hot) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
         r += int64_t(gridDim.x) * blockDim.x)
        if (flag[r]) hot[pos[r]] = int32_t(r);
}

// first position q in [lo, hi) with col[q] >= key (col ascending within the row)
__device__ __forceinline__ int64_t lower_bound(const int32_t* __restrict__ col, int64_t lo, int64_t hi,
                                               int64_t key) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (col[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// One thread per (panel b, hot row h): the entries of h in panel b are
// [q_b, q_(b+1)) with q_b = lower_bound(row h, b * pr) (T's entries ascend
// within a row), cut into chunks of pch entries. WRITE = false: the chunk
// count k(b, h), stored panel-major (item positions) and row-major (slot
// numbering: a row's partials in panel order). WRITE = true: the k items at
// their panel-major positions with their row-major slots. Balanced over
// (panel, row) pairs: the longest hot row (5.3M entries at C3) no longer
// serialises on one thread.
template <bool WRITE>
__global__ void k_panel_cells(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const int32_t* __restrict__ hot, int64_t nhot, int64_t npan, int64_t pr, int64_t pch,
                              int32_t* __restrict__ cnt_pm, int32_t* __restrict__ cnt_rm,
                              const int32_t* __restrict__ itempos, const int32_t* __restrict__ slotpos,
                              WorkItem* __restrict__ items) {
    const int64_t total = npan * nhot;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = t / nhot, h = t - b * nhot;  // consecutive threads: consecutive rows
        const int32_t r = hot[h];
        const int64_t p0 = rp[r], p1 = rp[r + 1];
        const int64_t q0 = lower_bound(col, p0, p1, b * pr);
        const int64_t q1 = lower_bound(col, q0, p1, (b + 1) * pr);
        const int32_t k = int32_t((q1 - q0 + pch - 1) / pch);
        if (!WRITE) {
            cnt_pm[t] = k;
            cnt_rm[h * npan + b] = k;
            continue;
        }
        const int32_t o = itempos[t], sl = slotpos[h * npan + b];
        for (int32_t u = 0; u < k; ++u) {
            WorkItem w;
            w.p0 = q0 + int64_t(u) * pch;
            w.p1 = min(q1, q0 + int64_t(u + 1) * pch);
            w.r0 = r;
            w.r1 = -(sl + u) - 1;
            items[o + u] = w;
        }
    }
}

// combine entry of hot row h: its slots [slotpos(h, 0), slotpos(h + 1, 0))
__global__ void k_panel_comb(const int32_t* __restrict__ hot, int64_t nhot, int64_t npan,
                             const int32_t* __restrict__ slotpos, Combine* __restrict__ comb) {
    for (int64_t h = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; h < nhot;
         h += int64_t(gridDim.x) * blockDim.x) {
        Combine cb;
        cb.row = hot[h];
        cb.s0 = slotpos[h * npan];
        cb.s1 = slotpos[(h + 1) * npan];
        cb.pad = 0;
        comb[h] = cb;
    }
}

}  // namespace

// Builds (or reuses) the panel plan of T for panels of `pr` rows of the
// gathered operand. Rows with >= thot entries (3 per panel on average: below
// that a per-panel partial costs more than the HBM gathers it saves) are hot;
// thot is doubled until the partials fit `slot_cap` rows.
void ensure_panels(Ctx& c, DCsr& T, int64_t pr, int64_t slot_cap) {
    PanelPlan& P = T.pan;
    if (P.pr == pr) return;
    Prof prof(c, "panel_plan", 0, 0);
    P = PanelPlan{};
    if (T.rows == 0 || T.nnz == 0 || pr <= 0) return;
    cudaStream_t s = c.stream;
    const int64_t n = T.rows;
    const int64_t npan = (T.cols + pr - 1) / pr;
    // chunks short enough that the slowest in-flight chunk does not let the
    // work front run many panels ahead (the window must stay L2-resident)
    const char* ec = std::getenv("FRPCA_PANEL_CHUNK");
    const int64_t pch = std::max<int64_t>(16, ec ? std::atoll(ec) : 256);
    DBuf<int32_t> flag(size_t(n) + 1, s), pos(size_t(n) + 1, s);
    P.skip.alloc(size_t(n), s);
    int64_t thot = 3 * npan, nhot = 0, nitems = 0;
    DBuf<int32_t> hot, cnt_pm, cnt_rm, itempos, slotpos;
    for (;;) {
        FB_CUDA(cudaMemsetAsync(flag.get(), 0, flag.bytes(), s));
        k_hot_flags<<<grid_for(c, n), 256, 0, s>>>(T.rowptr.get(), n, thot, P.skip.get(), flag.get());
        FB_LAUNCH_CHECK();
        size_t tb = 0;
        FB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.get(), pos.get(), n + 1, s));
        DBuf<unsigned char> tmp(tb, s);
        FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, flag.get(), pos.get(), n + 1, s));
        nhot = read_scalar(c, pos.get() + n);
        if (nhot == 0) {
            P = PanelPlan{};
            P.pr = pr;  // cached: nothing is hot at this panel size
            return;
        }
        if (double(npan) * double(nhot) >= double(1 << 30)) { thot *= 2; continue; }
        hot.alloc(size_t(nhot), s);
        k_hot_list<<<grid_for(c, n), 256, 0, s>>>(flag.get(), pos.get(), n, hot.get());
        FB_LAUNCH_CHECK();
        // the +1 entries stay 0: the scans below then end on the totals
        cnt_pm.alloc(size_t(npan * nhot) + 1, s);
        cnt_rm.alloc(size_t(npan * nhot) + 1, s);
        FB_CUDA(cudaMemsetAsync(cnt_pm.get() + npan * nhot, 0, sizeof(int32_t), s));
        FB_CUDA(cudaMemsetAsync(cnt_rm.get() + npan * nhot, 0, sizeof(int32_t), s));
        k_panel_cells<false><<<grid_for(c, npan * nhot), 256, 0, s>>>(T.rowptr.get(), T.col.get(), hot.get(), nhot,
                                                                      npan, pr, pch, cnt_pm.get(), cnt_rm.get(),
                                                                      nullptr, nullptr, nullptr);
        FB_LAUNCH_CHECK();
        // 64-bit total first: the int32 scans below need it < 2^31
        DBuf<int64_t> tot(1, s);
        size_t tb2 = 0;
        FB_CUDA(cub::DeviceReduce::Sum(nullptr, tb2, cnt_pm.get(), tot.get(), npan * nhot, s));
        DBuf<unsigned char> tmp2(tb2, s);
        FB_CUDA(cub::DeviceReduce::Sum(tmp2.get(), tb2, cnt_pm.get(), tot.get(), npan * nhot, s));
        nitems = read_scalar(c, tot.get());
        if (nitems <= slot_cap && nitems < (int64_t(1) << 30)) break;
        thot *= 2;
    }
    itempos.alloc(size_t(npan * nhot) + 1, s);
    slotpos.alloc(size_t(npan * nhot) + 1, s);
    size_t tb = 0;
    FB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt_pm.get(), itempos.get(), npan * nhot + 1, s));
    DBuf<unsigned char> tmp(tb, s);
    FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt_pm.get(), itempos.get(), npan * nhot + 1, s));
    FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt_rm.get(), slotpos.get(), npan * nhot + 1, s));
    P.hot.items.alloc(size_t(nitems), s);
    P.hot.comb.alloc(size_t(nhot), s);
    k_panel_cells<true><<<grid_for(c, npan * nhot), 256, 0, s>>>(T.rowptr.get(), T.col.get(), hot.get(), nhot, npan,
                                                                 pr, pch, nullptr, nullptr, itempos.get(),
                                                                 slotpos.get(), P.hot.items.get());
    FB_LAUNCH_CHECK();
    k_panel_comb<<<grid_for(c, nhot), 256, 0, s>>>(hot.get(), nhot, npan, slotpos.get(), P.hot.comb.get());
    FB_LAUNCH_CHECK();
    P.hot.nitems = P.hot.nslots = nitems;
    P.hot.ncomb = nhot;
    P.hot.chunk = pch;
    build_items(c, T, P.skip.get(), P.cold, T.L.chunk);
    P.counter.alloc(1, s);
    P.npanels = npan;
    P.thot = thot;
    P.nhot = nhot;
    P.pr = pr;
    FB_CUDA(cudaStreamSynchronize(s));
    if (std::getenv("FRPCA_DEBUG_PANELS"))
        std::fprintf(stderr, "panels: rows %lld pr %lld npanels %lld thot %lld nhot %lld hot_items %lld cold_items %lld "
                     "cold_slots %lld\n", (long long)T.rows, (long long)pr, (long long)npan, (long long)thot,
                     (long long)nhot, (long long)nitems, (long long)P.cold.nitems, (long long)P.cold.nslots);
}

// ---- from_triplets on the device (sparse_matrix.hpp:62-95) -----
// Keys row*cols+col, stable radix sort (duplicates keep input order), each run
// of equal keys summed sequentially, exact-zero sums dropped, row pointers by
// counting. The reference sorts with std::sort (not stable), so for three or
// more duplicates of one coordinate its summation order can differ (rounding
// level); with at most two the sums are identical (a + b == b + a).

namespace {

__global__ void k_trip_check(const int64_t* __restrict__ r, const int64_t* __restrict__ c, int64_t n, int64_t rows,
                             int64_t cols, unsigned long long* __restrict__ keys, int* __restrict__ bad) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t ri = r[i], ci = c[i];
        if (ri < 0 || ri >= rows || ci < 0 || ci >= cols) {
            atomicOr(bad, 1);
            keys[i] = 0;
        } else {
            keys[i] = (unsigned long long)ri * (unsigned long long)cols + (unsigned long long)ci;
        }
    }
}

__global__ void k_run_heads(const unsigned long long* __restrict__ k, int64_t n, int64_t* __restrict__ head) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        head[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// run starting at i (a head): sequential sum; keep[s] = (sum != 0)
__global__ void k_run_sums(const unsigned long long* __restrict__ k, const double* __restrict__ v, int64_t n,
                           const int64_t* __restrict__ head, const int64_t* __restrict__ seg,
                           unsigned long long* __restrict__ skey, double* __restrict__ ssum,
                           int64_t* __restrict__ keep) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        if (!head[i]) continue;
        const unsigned long long key = k[i];
        double sum = 0.0;
        for (int64_t t = i; t < n && k[t] == key; ++t) sum += v[t];
        const int64_t s = seg[i];
        skey[s] = key;
        ssum[s] = sum;
        keep[s] = sum != 0.0 ? 1 : 0;
    }
}

__global__ void k_trip_emit(const unsigned long long* __restrict__ skey, const double* __restrict__ ssum,
                            const int64_t* __restrict__ keep, const int64_t* __restrict__ pos, int64_t nseg,
                            int64_t cols, int64_t* __restrict__ col, double* __restrict__ val,
                            int64_t* __restrict__ rowcnt) {
    for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < nseg; s += int64_t(gridDim.x) * blockDim.x) {
        if (!keep[s]) continue;
        const int64_t o = pos[s];
        const int64_t row = int64_t(skey[s] / (unsigned long long)cols);
        col[o] = int64_t(skey[s] % (unsigned long long)cols);
        val[o] = ssum[s];
        atomicAdd(reinterpret_cast<unsigned long long*>(rowcnt + row + 1), 1ull);
    }
}

template <class T>
void exclusive_scan(Ctx& c, const T* in, T* out, int64_t n) {
    size_t tb = 0;
    FB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, c.stream));
    DBuf<unsigned char> tmp(tb, c.stream);
    FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, in, out, n, c.stream));
}

}  // namespace

void csr_from_triplets_device(Ctx& c, int64_t rows, int64_t cols, int64_t n, const int64_t* r, const int64_t* ci,
                              const double* v, int64_t* nnz, int64_t* row_ptr, int64_t* col_idx, double* values) {
    cudaStream_t s = c.stream;
    if (n == 0) {
        std::memset(row_ptr, 0, sizeof(int64_t) * size_t(rows + 1));
        *nnz = 0;
        return;
    }
    DBuf<int64_t> dr(size_t(n), s), dc(size_t(n), s);
    DBuf<double> dv(size_t(n), s), dv2(size_t(n), s);
    DBuf<unsigned long long> key(size_t(n), s), key2(size_t(n), s);
    DBuf<int> bad(1, s);
    FB_CUDA(cudaMemcpyAsync(dr.get(), r, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    FB_CUDA(cudaMemcpyAsync(dc.get(), ci, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    FB_CUDA(cudaMemcpyAsync(dv.get(), v, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    FB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    k_trip_check<<<grid_for(c, n), 256, 0, s>>>(dr.get(), dc.get(), n, rows, cols, key.get(), bad.get());
    FB_LAUNCH_CHECK();
    if (read_scalar(c, bad.get())) throw InvalidArgument("from_triplets: entry out of bounds");
    dr.release();
    dc.release();
    int end_bit = 1;
    const unsigned long long kmax = (unsigned long long)std::max<int64_t>(rows, 1) * (unsigned long long)cols;
    while (end_bit < 64 && (1ull << end_bit) < kmax) ++end_bit;
    {
        size_t tb = 0;
        FB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.get(), key2.get(), dv.get(), dv2.get(), n, 0,
                                                end_bit, s));
        DBuf<unsigned char> tmp(tb, s);
        FB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, key.get(), key2.get(), dv.get(), dv2.get(), n, 0,
                                                end_bit, s));
    }
    DBuf<int64_t> head(size_t(n) + 1, s), seg(size_t(n) + 1, s);
    FB_CUDA(cudaMemsetAsync(head.get(), 0, head.bytes(), s));
    k_run_heads<<<grid_for(c, n), 256, 0, s>>>(key2.get(), n, head.get());
    FB_LAUNCH_CHECK();
    exclusive_scan(c, head.get(), seg.get(), n + 1);
    const int64_t nseg = read_scalar(c, seg.get() + n);
    DBuf<unsigned long long> skey(size_t(nseg), s);
    DBuf<double> ssum(size_t(nseg), s);
    DBuf<int64_t> keep(size_t(nseg) + 1, s), pos(size_t(nseg) + 1, s);
    FB_CUDA(cudaMemsetAsync(keep.get(), 0, keep.bytes(), s));
    k_run_sums<<<grid_for(c, n), 256, 0, s>>>(key2.get(), dv2.get(), n, head.get(), seg.get(), skey.get(), ssum.get(),
                                              keep.get());
    FB_LAUNCH_CHECK();
    exclusive_scan(c, keep.get(), pos.get(), nseg + 1);
    const int64_t total = read_scalar(c, pos.get() + nseg);
    DBuf<int64_t> ocol(size_t(std::max<int64_t>(total, 1)), s), cnt(size_t(rows) + 1, s), rp(size_t(rows) + 1, s);
    DBuf<double> oval(size_t(std::max<int64_t>(total, 1)), s);
    FB_CUDA(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));
    k_trip_emit<<<grid_for(c, nseg), 256, 0, s>>>(skey.get(), ssum.get(), keep.get(), pos.get(), nseg, cols,
                                                  ocol.get(), oval.get(), cnt.get());
    FB_LAUNCH_CHECK();
    // cnt[r + 1] = entries of row r -> inclusive prefix = row_ptr
    {
        size_t tb = 0;
        FB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt.get(), rp.get(), rows + 1, s));
        DBuf<unsigned char> tmp(tb, s);
        FB_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb, cnt.get(), rp.get(), rows + 1, s));
    }
    FB_CUDA(cudaMemcpyAsync(row_ptr, rp.get(), sizeof(int64_t) * (rows + 1), cudaMemcpyDeviceToHost, s));
    if (total) {
        FB_CUDA(cudaMemcpyAsync(col_idx, ocol.get(), sizeof(int64_t) * total, cudaMemcpyDeviceToHost, s));
        FB_CUDA(cudaMemcpyAsync(values, oval.get(), sizeof(double) * total, cudaMemcpyDeviceToHost, s));
    }
    FB_CUDA(cudaStreamSynchronize(s));
    *nnz = total;
}

void ensure_encoding(Ctx& c, DCsr& A, int64_t hint_h, int64_t sx_h) {
    if (!A.rank_of.n) return;
    hint_h = std::min(hint_h, A.cols);
    sx_h = std::min(sx_h, A.cols);
    if (hint_h == A.hint_h && sx_h == A.sx_h) return;
    k_encode_cols<<<grid_for(c, A.nnz), 256, 0, c.stream>>>(A.col.get(), A.nnz, A.rank_of.get(), A.rank_ids.get(),
                                                             hint_h, sx_h);
    FB_LAUNCH_CHECK();
    A.hint_h = hint_h;
    A.sx_h = sx_h;
}

void ensure_hint(Ctx& c, DCsr& A, int64_t w) {
    // budget of L2-kept X rows
    const char* e = std::getenv("FRPCA_HINT_MB");
    const double mb = e && *e ? std::atof(e) : 64.0;
    const double budget = mb * 1048576.0;
    int64_t H = 0;
    // (at C1, X = 2.5x the budget, the hints cost 2%: only well beyond it)
    if (budget > 0 && 8.0 * double(A.cols) * double(w) > 4.0 * budget)
        H = std::min<int64_t>(A.cols, std::max<int64_t>(1, int64_t(budget / (8.0 * double(w)))));
    ensure_encoding(c, A, H, 0);
}

void download_csr(Ctx& c, const DCsr& A, int64_t* rp, int64_t* ci, double* v) {
    std::vector<int32_t> tmp(static_cast<size_t>(A.nnz));
    FB_CUDA(cudaMemcpyAsync(rp, A.rowptr.get(), sizeof(int64_t) * (A.rows + 1),
                            cudaMemcpyDeviceToHost, c.stream));
    if (A.nnz) {
        FB_CUDA(cudaMemcpyAsync(tmp.data(), A.col.get(), sizeof(int32_t) * A.nnz,
                                cudaMemcpyDeviceToHost, c.stream));
        FB_CUDA(cudaMemcpyAsync(v, A.val.get(), sizeof(double) * A.nnz, cudaMemcpyDeviceToHost,
                                c.stream));
    }
    FB_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<int32_t> ids;
    if (A.sx_h > 0) {
        ids.resize(size_t(A.sx_h));
        FB_CUDA(cudaMemcpy(ids.data(), A.rank_ids.get(), sizeof(int32_t) * ids.size(), cudaMemcpyDeviceToHost));
    }
    for (int64_t i = 0; i < A.nnz; ++i) {
        const int32_t e = tmp[size_t(i)];
        ci[i] = (e & kColHot) ? ids[size_t(e & kRankMask)] : (e & kColMask);
    }
}

int64_t read_i64(Ctx& c, const int64_t* d) { return read_scalar(c, d); }

}  // namespace fb
