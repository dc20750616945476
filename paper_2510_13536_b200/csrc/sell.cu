// sell.cu -- CsrMatrix (sparse.py:36-87, int64 or int32 indices, FP64 values)
// -> device SELL-32 layout (common.cuh: SellMatrix).
//
// The reference keeps CSR and walks rows with one scalar thread.  On B200 the
// SpMV is HBM-bound, so the layout is chosen for coalescing and bytes: slices
// of 32 rows (one warp), entries column-major inside a slice, padding marked
// by a sentinel column (no row-length array), and int16 column deltas when
// the matrix is banded enough.  Row order of entries is preserved, so the
// per-row left-to-right accumulation (and hence every bit of the result) is
// unchanged.
#include <algorithm>
#include <climits>
#include <unordered_map>
#include <vector>
#include <cub/cub.cuh>
#include "common.cuh"
#include "mwcg_internal.h"
#include "ops.cuh"
#include "../../include/mwcg_cuda.h"

namespace mwcg {

// slice sizes (32 * max row length in the slice) and the int16 feasibility
// flag (any |col - row| >= 2^15 -> int32 columns)
template <typename I>
__global__ void sell_scan_kernel(const I *__restrict__ rp, const I *__restrict__ ci, int64_t n_rows,
                                 int64_t n_pad, int64_t row_base, int64_t *__restrict__ slice_sz,
                                 unsigned int *__restrict__ too_wide) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int len = 0;
    bool wide = false;
    if (r < n_rows) {
        const int64_t lo = rp[r], hi = rp[r + 1];
        len = (int)(hi - lo);
        const int64_t g = row_base + r;
        for (int64_t k = lo; k < hi; k++) {
            const int64_t d = (int64_t)ci[k] - g;
            wide |= (d < -32767 || d > 32767);
        }
    }
    int m = len;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0 && r < n_pad) slice_sz[r >> 5] = (int64_t)m * SLICE;
    if (__any_sync(0xffffffffu, wide) && (threadIdx.x & 31) == 0) atomicOr(too_wide, 1u);
}

__global__ void fill16_kernel(int16_t *__restrict__ p, int64_t n, int16_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

template <typename I, typename C>
__global__ void sell_fill_kernel(const I *__restrict__ rp, const I *__restrict__ ci,
                                 const double *__restrict__ va, int64_t n_rows, int64_t row_base,
                                 const int64_t *__restrict__ slice_ptr, const int32_t *__restrict__ pos_of,
                                 C *__restrict__ cols, double *__restrict__ vals) {
    // one warp per row: coalesced reads of the CSR row, strided SELL writes
    // (at the row's storage position: its own, or its SELL-sigma slot)
    int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (gw >= n_rows) return;
    int64_t r = gw;
    const int64_t pos = pos_of ? (int64_t)pos_of[r] : r;
    int64_t base = slice_ptr[pos >> 5] + (pos & 31);
    int64_t lo = rp[r], hi = rp[r + 1];
    for (int64_t k = lo + lane; k < hi; k += 32) {
        int64_t kk = k - lo;
        if (sizeof(C) == 2) cols[base + kk * SLICE] = (C)((int64_t)ci[k] - (row_base + r));
        else cols[base + kk * SLICE] = (C)ci[k];
        vals[base + kk * SLICE] = va[k];
    }
}

// ---------------------------------------------------------------------------
// SELL-sigma (sigma = one 1024-row tile): the rows of each tile are ranked by
// (length descending, row ascending) and stored in that order, so a slice
// holds rows of similar length and pads less (C5: 35 % -> 1.5 %).  Rows never
// leave their tile, so the tile partials of the fused dots are unchanged.
template <typename I>
__global__ void __launch_bounds__(1024) sigma_rank_kernel(const I *__restrict__ rp, int64_t n_rows,
                                                          uint16_t *__restrict__ perm,
                                                          int32_t *__restrict__ pos_of) {
    __shared__ int lens[1024];
    const int64_t t0 = (int64_t)blockIdx.x * 1024;
    const int i = threadIdx.x;
    const int64_t r = t0 + i;
    const int len = r < n_rows ? (int)(rp[r + 1] - rp[r]) : -1;  // past the end: last
    lens[i] = len;
    __syncthreads();
    int rank = 0;
    for (int j = 0; j < 1024; j++) {
        const int lj = lens[j];
        rank += (lj > len) || (lj == len && j < i);
    }
    perm[t0 + rank] = (uint16_t)i;
    if (r < n_rows) pos_of[r] = (int32_t)(t0 + rank);
}

template <typename I>
__global__ void sigma_slice_kernel(const I *__restrict__ rp, int64_t n_rows, const uint16_t *__restrict__ perm,
                                   int64_t n_pad, int64_t *__restrict__ slice_sz) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int len = 0;
    if (pos < n_pad) {
        const int64_t r = (pos & ~(int64_t)1023) + perm[pos];
        if (r < n_rows) len = (int)(rp[r + 1] - rp[r]);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, off));
    if ((threadIdx.x & 31) == 0 && pos < n_pad) slice_sz[pos >> 5] = (int64_t)len * SLICE;
}

// ---------------------------------------------------------------------------
// Slice-shared offsets (common.cuh): one warp per slice walks its 32 rows'
// CSR entries in lock-step by ascending column offset (warp min over the
// lanes' heads); every distinct offset becomes one slot with the ballot of
// the lanes that have it.  Pass 1 counts slots (capped: a slice needing more
// than cap = Lmax + DIA_SLACK slots marks the matrix as not DIA-friendly);
// pass 2 writes the slot words and the values.
// ---------------------------------------------------------------------------
constexpr int DIA_SLACK = 2;

template <typename I, bool FILL>
__global__ void dia_walk_kernel(const I *__restrict__ rp, const I *__restrict__ ci, const double *__restrict__ va,
                                int64_t n_rows, int64_t n_slices, int64_t row_base, int64_t *__restrict__ slice_sz,
                                const int64_t *__restrict__ slice_ptr, uint64_t *__restrict__ om,
                                double *__restrict__ vals, unsigned int *__restrict__ reject) {
    const int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (sl >= n_slices) return;
    const int64_t r = sl * SLICE + lane;
    int64_t head = 0, hi = 0;
    if (r < n_rows) {
        head = rp[r];
        hi = rp[r + 1];
    }
    int len = (int)(hi - head);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, off));
    const int cap = len + DIA_SLACK;
    const int64_t g = row_base + r;
    const int64_t s0 = FILL ? slice_ptr[sl] : 0;
    int k = 0;
    for (;;) {
        const int cur = head < hi ? (int)((int64_t)ci[head] - g) : INT_MAX;
        const int m = __reduce_min_sync(0xffffffffu, cur);
        if (m == INT_MAX) break;
        const bool present = cur == m;
        const unsigned int mask = __ballot_sync(0xffffffffu, present);
        if (!FILL && k == cap) {  // more distinct offsets than the slice is worth
            if (lane == 0) atomicOr(reject, 1u);
            break;
        }
        if (FILL) {
            if (lane == 0) om[(s0 >> 5) + k] = ((uint64_t)mask << 32) | (uint64_t)(uint32_t)m;
            vals[s0 + (int64_t)k * SLICE + lane] = present ? va[head] : 0.0;
        }
        if (present) head++;
        k++;
    }
    if (!FILL && lane == 0) slice_sz[sl] = (int64_t)k * SLICE;
}

// Slot-word patterns: stencil and band slices repeat a handful of (offset,
// mask) sequences (interior / boundary combinations), so the slot words are
// deduplicated into a pattern table small enough to stay in L1, and each
// slice's descriptor packs its value offset with its pattern base:
//   desc[j] = (slice_start / 32) | (pattern_base << 36),
// desc[n_slices] = total / 32.  A row's gathers then wait on one L2 load
// (desc) and one L1 hit (the pattern word) instead of two L2 loads.
static int dia_patterns(SellMatrixOwned *M, int64_t *slice_ptr, int64_t n_words, cudaStream_t st) {
    SellMatrix &A = M->view;
    const int64_t ns = A.n_slices;
    std::vector<int64_t> sp(ns + 1);
    std::vector<uint64_t> om(n_words);
    MWCG_CUDA(cudaMemcpyAsync(sp.data(), slice_ptr, sizeof(int64_t) * (ns + 1), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaMemcpyAsync(om.data(), M->om, sizeof(uint64_t) * n_words, cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    std::vector<uint64_t> pat;
    std::vector<uint64_t> desc(ns + 1);
    std::unordered_multimap<uint64_t, std::pair<int64_t, int64_t>> seen;  // hash -> (pattern base, length)
    for (int64_t j = 0; j < ns; j++) {
        const int64_t b = sp[j] >> 5, len = (sp[j + 1] - sp[j]) >> 5;
        uint64_t hsh = 1469598103934665603ull ^ (uint64_t)len;
        for (int64_t k = 0; k < len; k++) hsh = (hsh ^ om[b + k]) * 1099511628211ull;
        int64_t base = -1;
        auto rng = seen.equal_range(hsh);
        for (auto it = rng.first; it != rng.second && base < 0; ++it)
            if (it->second.second == len &&
                std::equal(om.begin() + b, om.begin() + b + len, pat.begin() + it->second.first))
                base = it->second.first;
        if (base < 0) {
            base = (int64_t)pat.size();
            pat.insert(pat.end(), om.begin() + b, om.begin() + b + len);
            pat.insert(pat.end(), DIA_PAD, 0ull);  // empty slots: chunks may read past the end
            seen.emplace(hsh, std::make_pair(base, len));
        }
        if (base >= (1ll << 28)) {
            set_error("slice-shared offsets: pattern table too large");
            return MWCG_ERR_VALUE;
        }
        desc[j] = (uint64_t)(sp[j] >> 5) | ((uint64_t)base << 36);
    }
    desc[ns] = (uint64_t)(sp[ns] >> 5);
    if (pat.empty()) pat.assign(DIA_PAD, 0ull);
    pool_free(M->om, st);
    M->om = nullptr;
    MWCG_CUDA(pool_alloc((void **)&M->om, sizeof(uint64_t) * pat.size(), st));
    MWCG_CUDA(cudaMemcpyAsync(M->om, pat.data(), sizeof(uint64_t) * pat.size(), cudaMemcpyHostToDevice, st));
    desc.resize(ns + 1 + DESC_PAD, desc[ns]);
    MWCG_CUDA(cudaMemcpyAsync(slice_ptr, desc.data(), sizeof(uint64_t) * desc.size(), cudaMemcpyHostToDevice, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    M->n_patterns_words = (int64_t)pat.size();
    M->pat_host = std::move(pat);
    desc.resize(ns + 1);
    M->desc_host = std::move(desc);
    return 0;
}

// Try the slice-shared-offset layout: returns 1 (built), 0 (not worth it:
// more than DIA_SLACK extra slots in some slice, or > 6 % more slots than the
// padded SELL layout, or offsets beyond int32), or an error code < 0 / > 1.
template <typename I>
static int build_dia(SellMatrixOwned *M, const I *rp, const I *ci, const double *va, int64_t sell_total,
                     bool force, cudaStream_t st) {
    SellMatrix &A = M->view;
    if (A.n_slices == 0) return 0;  // no rows: the (empty) SELL layout
    int64_t *slice_sz = nullptr, *slice_ptr = nullptr;
    unsigned int *flag = nullptr;
    MWCG_CUDA(pool_alloc((void **)&slice_sz, sizeof(int64_t) * (A.n_slices + 1), st));
    MWCG_CUDA(pool_alloc((void **)&flag, sizeof(unsigned int), st));
    MWCG_CUDA(cudaMemsetAsync(slice_sz, 0, sizeof(int64_t) * (A.n_slices + 1), st));
    MWCG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned int), st));
    const unsigned blocks = (unsigned)((A.n_slices * 32 + 255) / 256);
    dia_walk_kernel<I, false><<<blocks, 256, 0, st>>>(rp, ci, va, A.n_rows, A.n_slices, A.row_base, slice_sz,
                                                      nullptr, nullptr, nullptr, flag);
    MWCG_CHECK_LAUNCH();
    MWCG_CUDA(pool_alloc((void **)&slice_ptr, sizeof(int64_t) * (A.n_slices + 1 + DESC_PAD), st));
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, slice_sz, slice_ptr, A.n_slices + 1, st);
    void *tmp = nullptr;
    MWCG_CUDA(pool_alloc(&tmp, tmp_bytes, st));
    MWCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, slice_sz, slice_ptr, A.n_slices + 1, st));
    int64_t total = 0;
    unsigned int reject = 0;
    MWCG_CUDA(cudaMemcpyAsync(&total, slice_ptr + A.n_slices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaMemcpyAsync(&reject, flag, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    pool_free(tmp, st);
    pool_free(slice_sz, st);
    pool_free(flag, st);
    if (!force && (reject || total * 100 > sell_total * 106)) {
        pool_free(slice_ptr, st);
        return 0;
    }
    if (reject) {
        pool_free(slice_ptr, st);
        set_error("slice-shared offsets: a slice needs more than Lmax + %d slots", DIA_SLACK);
        return MWCG_ERR_VALUE;
    }
    const size_t ne = (size_t)(total > 0 ? total : 32);
    MWCG_CUDA(pool_alloc((void **)&M->om, sizeof(uint64_t) * (ne / 32), st));
    // DIA_PAD slots of slack: a chunk of the last slice reads past its end
    MWCG_CUDA(pool_alloc((void **)&M->vals, sizeof(double) * (ne + DIA_PAD * SLICE), st));
    MWCG_CUDA(cudaMemsetAsync(M->vals + ne, 0, sizeof(double) * DIA_PAD * SLICE, st));
    dia_walk_kernel<I, true><<<blocks, 256, 0, st>>>(rp, ci, va, A.n_rows, A.n_slices, A.row_base, nullptr,
                                                     slice_ptr, M->om, M->vals, nullptr);
    MWCG_CHECK_LAUNCH();
    int rc = dia_patterns(M, slice_ptr, (int64_t)(ne / 32), st);
    if (rc) return rc;
    M->slice_ptr = slice_ptr;
    A.total = total;
    A.dia = 1;
    A.col16 = 0;
    A.slice_ptr = slice_ptr;
    A.cols = nullptr;
    A.vals = M->vals;
    A.om = M->om;
    MWCG_CUDA(cudaStreamSynchronize(st));
    return 1;
}

template <typename I>
static int build_sell(SellMatrixOwned *M, const I *rp, const I *ci, const double *va, int col_format,
                      int sigma, cudaStream_t st) {
    SellMatrix &A = M->view;
    int64_t n_pad = A.n_slices * SLICE;
    int64_t *slice_sz = nullptr;
    unsigned int *flag = nullptr;
    MWCG_CUDA(pool_alloc((void **)&M->slice_ptr, sizeof(int64_t) * (A.n_slices + 1), st));
    MWCG_CUDA(pool_alloc((void **)&slice_sz, sizeof(int64_t) * (A.n_slices + 1), st));
    MWCG_CUDA(pool_alloc((void **)&flag, sizeof(unsigned int), st));
    MWCG_CUDA(cudaMemsetAsync(slice_sz, 0, sizeof(int64_t) * (A.n_slices + 1), st));
    MWCG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned int), st));
    if (n_pad > 0) {
        int threads = 256;
        int64_t blocks = (n_pad + threads - 1) / threads;
        sell_scan_kernel<I><<<(unsigned)blocks, threads, 0, st>>>(rp, ci, A.n_rows, n_pad, A.row_base, slice_sz,
                                                                  flag);
        MWCG_CHECK_LAUNCH();
    }
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, slice_sz, M->slice_ptr, A.n_slices + 1, st);
    void *tmp = nullptr;
    MWCG_CUDA(pool_alloc(&tmp, tmp_bytes, st));
    MWCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, slice_sz, M->slice_ptr, A.n_slices + 1, st));
    int64_t total = 0;
    unsigned int wide = 0;
    MWCG_CUDA(cudaMemcpyAsync(&total, M->slice_ptr + A.n_slices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaMemcpyAsync(&wide, flag, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    pool_free(tmp, st);
    pool_free(slice_sz, st);
    pool_free(flag, st);
    A.total = total;
    if (col_format == 2 || col_format < 0) {  // slice-shared offsets when they pay
        const int64_t *sell_ptr = M->slice_ptr;
        M->slice_ptr = nullptr;
        int rc = build_dia<I>(M, rp, ci, va, total, col_format == 2, st);
        if (rc == 1) {
            pool_free((void *)sell_ptr, st);
            return 0;
        }
        M->slice_ptr = (int64_t *)sell_ptr;
        A.total = total;
        if (rc != 0) return rc;
    }
    if (col_format == 1 && wide) {
        set_error("column offsets do not fit int16 deltas");
        return MWCG_ERR_VALUE;
    }
    A.col16 = (col_format == 1 || (col_format < 0 && !wide)) ? 1 : 0;
    int32_t *pos_of = nullptr;
    if (sigma >= 0 && A.n_rows > 0) {
        // SELL-sigma candidate: rank rows inside their tile, re-size the slices
        const int64_t ntl = (A.n_rows + 1023) / 1024;
        int64_t *sz2 = nullptr, *ptr2 = nullptr;
        MWCG_CUDA(pool_alloc((void **)&M->perm, sizeof(uint16_t) * (size_t)ntl * 1024, st));
        MWCG_CUDA(pool_alloc((void **)&pos_of, sizeof(int32_t) * (size_t)A.n_rows, st));
        MWCG_CUDA(pool_alloc((void **)&sz2, sizeof(int64_t) * (A.n_slices + 1), st));
        MWCG_CUDA(pool_alloc((void **)&ptr2, sizeof(int64_t) * (A.n_slices + 1), st));
        MWCG_CUDA(cudaMemsetAsync(sz2, 0, sizeof(int64_t) * (A.n_slices + 1), st));
        sigma_rank_kernel<I><<<(unsigned)ntl, 1024, 0, st>>>(rp, A.n_rows, M->perm, pos_of);
        sigma_slice_kernel<I><<<(unsigned)((n_pad + 255) / 256), 256, 0, st>>>(rp, A.n_rows, M->perm, n_pad, sz2);
        MWCG_CHECK_LAUNCH();
        size_t tb2 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb2, sz2, ptr2, A.n_slices + 1, st);
        void *tmp2 = nullptr;
        MWCG_CUDA(pool_alloc(&tmp2, tb2, st));
        MWCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, tb2, sz2, ptr2, A.n_slices + 1, st));
        int64_t total2 = 0;
        MWCG_CUDA(cudaMemcpyAsync(&total2, ptr2 + A.n_slices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        MWCG_CUDA(cudaStreamSynchronize(st));
        pool_free(tmp2, st);
        pool_free(sz2, st);
        if (sigma > 0 || total2 * 100 <= total * 95) {
            pool_free(M->slice_ptr, st);
            M->slice_ptr = ptr2;
            total = total2;
            A.total = total;
            A.perm = M->perm;
        } else {
            pool_free(ptr2, st);
            pool_free(pos_of, st);
            pool_free(M->perm, st);
            pos_of = nullptr;
            M->perm = nullptr;
        }
    }
    const size_t ne = (size_t)(total > 0 ? total : 1);
    MWCG_CUDA(pool_alloc((void **)&M->cols, ne * (A.col16 ? 2 : 4), st));
    MWCG_CUDA(pool_alloc((void **)&M->vals, sizeof(double) * ne, st));
    // padding: sentinel column, value 0
    if (A.col16) {
        fill16_kernel<<<148 * 8, 256, 0, st>>>((int16_t *)M->cols, (int64_t)ne, COL16_SENT);
        MWCG_CHECK_LAUNCH();
    } else {
        MWCG_CUDA(cudaMemsetAsync(M->cols, 0xFF, ne * 4, st));  // -1
    }
    MWCG_CUDA(cudaMemsetAsync(M->vals, 0, sizeof(double) * ne, st));
    if (A.n_rows > 0) {
        int threads = 256;
        int64_t blocks = (A.n_rows * 32 + threads - 1) / threads;
        if (A.col16)
            sell_fill_kernel<I, int16_t><<<(unsigned)blocks, threads, 0, st>>>(
                rp, ci, va, A.n_rows, A.row_base, M->slice_ptr, pos_of, (int16_t *)M->cols, M->vals);
        else
            sell_fill_kernel<I, int32_t><<<(unsigned)blocks, threads, 0, st>>>(
                rp, ci, va, A.n_rows, A.row_base, M->slice_ptr, pos_of, (int32_t *)M->cols, M->vals);
        MWCG_CHECK_LAUNCH();
    }
    pool_free(pos_of, st);
    A.slice_ptr = M->slice_ptr;
    A.cols = M->cols;
    A.vals = M->vals;
    MWCG_CUDA(cudaStreamSynchronize(st));
    return 0;
}

int sell_create(SellMatrixOwned **out, int64_t n_rows, int64_t n_cols, int64_t nnz,
                const void *row_ptr, const void *col_idx, const double *values, int index_bytes,
                int64_t row_base, int col_format, cudaStream_t st) {
    if (n_rows < 0 || n_cols < 0 || nnz < 0 || row_base < 0) {
        set_error("negative dimensions");
        return MWCG_ERR_VALUE;
    }
    if (n_cols > INT32_MAX || n_rows > INT32_MAX) {
        set_error("dimensions above 2^31-1 are not supported by the int32 SELL layout");
        return MWCG_ERR_VALUE;
    }
    if (index_bytes != 4 && index_bytes != 8) {
        set_error("index_bytes must be 4 or 8");
        return MWCG_ERR_VALUE;
    }
    // flags (include/mwcg_cuda.h): sigma -1 off / 0 auto / 1 forced
    int sigma = 0;
    if (col_format >= 0) {
        sigma = (col_format & MWCG_SELL_SIGMA) ? 1 : ((col_format & MWCG_SELL_NO_SIGMA) ? -1 : 0);
        col_format &= 15;
        if (col_format == 15) col_format = -1;
    }
    auto *M = new SellMatrixOwned();
    M->view.n_rows = n_rows;
    M->view.n_cols = n_cols;
    M->view.nnz = nnz;
    M->view.n_slices = (n_rows + SLICE - 1) / SLICE;
    M->view.row_base = row_base;
    int rc = (index_bytes == 8)
                 ? build_sell<int64_t>(M, (const int64_t *)row_ptr, (const int64_t *)col_idx, values,
                                       col_format, sigma, st)
                 : build_sell<int32_t>(M, (const int32_t *)row_ptr, (const int32_t *)col_idx, values,
                                       col_format, sigma, st);
    if (rc != 0) {
        sell_destroy(M);
        return rc;
    }
    *out = M;
    return 0;
}

void sell_destroy(SellMatrixOwned *M) {
    if (!M) return;
    pool_free(M->slice_ptr, 0);
    pool_free(M->cols, 0);
    pool_free(M->vals, 0);
    pool_free(M->om, 0);
    pool_free(M->perm, 0);
    delete M;
}

}  // namespace mwcg
