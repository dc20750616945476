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
#include <cstdlib>
#include <cstring>
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
// than cap = Lmax + DIA_SLACK slots, or more than DIA_MAX_SLOTS, marks the
// matrix as not DIA-friendly) and decides whether the slice is value-uniform
// (every slot: all present lanes hold the same value bits); pass 2 writes the
// slot records (offset word + uniform value) and, for the other slices, the
// per-lane values.
// ---------------------------------------------------------------------------
constexpr int DIA_SLACK = 2;
constexpr int DIA_UNIFORM_BIT = 1 << 8;  // slice_info: slots | uniform << 8 | full << 9
constexpr int DIA_FULL_BIT = 1 << 9;     // every slot present in all 32 rows

template <typename I, bool FILL>
__global__ void dia_walk_kernel(const I *__restrict__ rp, const I *__restrict__ ci, const double *__restrict__ va,
                                int64_t n_rows, int64_t n_slices, int64_t row_base, int allow_uniform,
                                int64_t *__restrict__ val_sz, int64_t *__restrict__ rec_sz,
                                int32_t *__restrict__ slice_info, const int64_t *__restrict__ val_ptr,
                                const int64_t *__restrict__ rec_ptr, ulonglong2 *__restrict__ rec,
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
    const int cap = min(len + DIA_SLACK, DIA_MAX_SLOTS);
    const int64_t g = row_base + r;
    bool uniform = FILL ? (slice_info[sl] & DIA_UNIFORM_BIT) != 0 : allow_uniform != 0;
    bool full = true;
    const int64_t v0 = FILL ? val_ptr[sl] : 0;
    const int64_t r0 = FILL ? rec_ptr[sl] : 0;
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
        const unsigned long long bits = present ? (unsigned long long)__double_as_longlong(va[head]) : 0ull;
        // value bits of the first present lane
        const unsigned long long first = __shfl_sync(0xffffffffu, bits, __ffs((int)mask) - 1);
        if (!FILL) uniform = uniform && __all_sync(0xffffffffu, !present || bits == first);
        full = full && mask == 0xffffffffu;
        if (FILL) {
            if (lane == 0)
                rec[r0 + k] = make_ulonglong2(((unsigned long long)mask << 32) | (unsigned long long)(uint32_t)m,
                                              uniform ? first : 0ull);
            if (!uniform) vals[v0 + (int64_t)k * SLICE + lane] = __longlong_as_double((long long)bits);
        }
        if (present) head++;
        k++;
    }
    if (!FILL && lane == 0) {
        val_sz[sl] = uniform ? 0 : (int64_t)k * SLICE;
        rec_sz[sl] = k;
        slice_info[sl] = k | (uniform ? DIA_UNIFORM_BIT : 0) | (full && k > 0 ? DIA_FULL_BIT : 0);
    }
}

// Slot-record patterns: stencil and band slices repeat a handful of (offset,
// mask[, value]) sequences (interior / boundary combinations), so the slot
// records are deduplicated into a pattern table small enough to stay in L1,
// and each slice gets a two-word descriptor
//   { value_start / 32 | slots << 40 | uniform << 48,  pattern base }.
// A row's gathers then wait on one L2 load (the descriptor) and one L1 hit
// (the pattern record) instead of two L2 loads.
static int dia_patterns(SellMatrixOwned *M, const int64_t *val_ptr, const int64_t *rec_ptr,
                        const int32_t *slice_info, const ulonglong2 *rec, int64_t n_rec, cudaStream_t st) {
    SellMatrix &A = M->view;
    const int64_t ns = A.n_slices;
    std::vector<int64_t> vp(ns + 1), rp(ns + 1);
    std::vector<int32_t> info(ns);
    std::vector<ulonglong2> rc((size_t)n_rec);
    MWCG_CUDA(cudaMemcpyAsync(vp.data(), val_ptr, sizeof(int64_t) * (ns + 1), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaMemcpyAsync(rp.data(), rec_ptr, sizeof(int64_t) * (ns + 1), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaMemcpyAsync(info.data(), slice_info, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, st));
    if (n_rec > 0)
        MWCG_CUDA(cudaMemcpyAsync(rc.data(), rec, sizeof(ulonglong2) * (size_t)n_rec, cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    std::vector<ulonglong2> pat;
    std::vector<uint64_t> desc(2 * (size_t)(ns + DESC_PAD));
    std::unordered_multimap<uint64_t, std::pair<int64_t, int64_t>> seen;  // hash -> (pattern base, length)
    auto same = [](const ulonglong2 &a, const ulonglong2 &b) { return a.x == b.x && a.y == b.y; };
    // consecutive slices of a stencil repeat a handful of patterns: the last
    // few distinct ones are tried first (one memcmp each), the hash map only
    // on a miss -- the loop is ~10 ns per slice instead of a hash + lookup
    constexpr int RECENT = 4;
    int64_t recent_base[RECENT], recent_len[RECENT];
    int n_recent = 0, next_recent = 0;
    for (int64_t j = 0; j < ns; j++) {
        const int64_t b = rp[j], len = rp[j + 1] - rp[j];
        int64_t base = -1;
        for (int r = 0; r < n_recent && base < 0; r++)
            if (recent_len[r] == len &&
                (len == 0 || std::memcmp(&rc[b], &pat[recent_base[r]], sizeof(ulonglong2) * (size_t)len) == 0))
                base = recent_base[r];
        if (base < 0) {
            uint64_t hsh = 1469598103934665603ull ^ (uint64_t)len;
            for (int64_t k = 0; k < len; k++) {
                hsh = (hsh ^ rc[b + k].x) * 1099511628211ull;
                hsh = (hsh ^ rc[b + k].y) * 1099511628211ull;
            }
            auto rng = seen.equal_range(hsh);
            for (auto it = rng.first; it != rng.second && base < 0; ++it)
                if (it->second.second == len &&
                    std::equal(rc.begin() + b, rc.begin() + b + len, pat.begin() + it->second.first, same))
                    base = it->second.first;
            if (base < 0) {
                base = (int64_t)pat.size();
                pat.insert(pat.end(), rc.begin() + b, rc.begin() + b + len);
                pat.insert(pat.end(), DIA_PAD, make_ulonglong2(0ull, 0ull));  // empty slots: chunks may read past the end
                seen.emplace(hsh, std::make_pair(base, len));
            }
            recent_base[next_recent] = base;
            recent_len[next_recent] = len;
            next_recent = (next_recent + 1) % RECENT;
            n_recent = std::min(n_recent + 1, RECENT);
        }
        const uint64_t uni = (info[j] & DIA_UNIFORM_BIT) ? 1ull : 0ull;
        const uint64_t ful = (info[j] & DIA_FULL_BIT) ? 1ull : 0ull;
        desc[2 * j] = (uint64_t)(vp[j] >> 5) | ((uint64_t)len << DIA_LBITS) | (uni << (DIA_LBITS + 8)) |
                      (ful << (DIA_LBITS + 9));
        desc[2 * j + 1] = (uint64_t)base;
    }
    if (pat.empty()) pat.assign(DIA_PAD, make_ulonglong2(0ull, 0ull));
    // descriptors past the last slice: empty slices (L = 0) on the empty pattern
    for (int64_t j = ns; j < ns + DESC_PAD; j++) {
        desc[2 * j] = (uint64_t)(vp[ns] >> 5);
        desc[2 * j + 1] = (uint64_t)(pat.size() - DIA_PAD);
    }
    MWCG_CUDA(pool_alloc((void **)&M->pat, sizeof(ulonglong2) * pat.size(), st));
    MWCG_CUDA(cudaMemcpyAsync(M->pat, pat.data(), sizeof(ulonglong2) * pat.size(), cudaMemcpyHostToDevice, st));
    MWCG_CUDA(pool_alloc((void **)&M->slice_ptr, sizeof(uint64_t) * desc.size(), st));
    MWCG_CUDA(cudaMemcpyAsync(M->slice_ptr, desc.data(), sizeof(uint64_t) * desc.size(), cudaMemcpyHostToDevice, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    M->n_patterns_words = (int64_t)pat.size();
    return 0;
}

// Try the slice-shared-offset layout: returns 1 (built), 0 (not worth it:
// more than DIA_SLACK extra slots in some slice, or > 6 % more slots than the
// padded SELL layout, or offsets beyond int32), or an error code < 0 / > 1.
template <typename I>
static int build_dia(SellMatrixOwned *M, const I *rp, const I *ci, const double *va, int64_t sell_total,
                     bool force, bool allow_uniform, cudaStream_t st) {
    SellMatrix &A = M->view;
    if (A.n_slices == 0) return 0;  // no rows: the (empty) SELL layout
    const int64_t ns = A.n_slices;
    int64_t *sz = nullptr, *ptr = nullptr;  // [0, ns]: value entries, [ns+1, 2ns+1]: records
    int32_t *info = nullptr;
    unsigned int *flag = nullptr;
    MWCG_CUDA(pool_alloc((void **)&sz, sizeof(int64_t) * 2 * (ns + 1), st));
    MWCG_CUDA(pool_alloc((void **)&ptr, sizeof(int64_t) * 2 * (ns + 1), st));
    MWCG_CUDA(pool_alloc((void **)&info, sizeof(int32_t) * ns, st));
    MWCG_CUDA(pool_alloc((void **)&flag, sizeof(unsigned int), st));
    MWCG_CUDA(cudaMemsetAsync(sz, 0, sizeof(int64_t) * 2 * (ns + 1), st));
    MWCG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned int), st));
    const unsigned blocks = (unsigned)((ns * 32 + 255) / 256);
    dia_walk_kernel<I, false><<<blocks, 256, 0, st>>>(rp, ci, va, A.n_rows, ns, A.row_base, allow_uniform ? 1 : 0, sz,
                                                      sz + ns + 1, info, nullptr, nullptr, nullptr, nullptr, flag);
    MWCG_CHECK_LAUNCH();
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sz, ptr, ns + 1, st);
    void *tmp = nullptr;
    MWCG_CUDA(pool_alloc(&tmp, tmp_bytes, st));
    MWCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sz, ptr, ns + 1, st));
    MWCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sz + ns + 1, ptr + ns + 1, ns + 1, st));
    int64_t stored = 0, n_rec = 0;
    unsigned int reject = 0;
    MWCG_CUDA(cudaMemcpyAsync(&stored, ptr + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaMemcpyAsync(&n_rec, ptr + 2 * ns + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaMemcpyAsync(&reject, flag, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    pool_free(tmp, st);
    pool_free(sz, st);
    pool_free(flag, st);
    const int64_t total = n_rec * SLICE;
    auto drop = [&]() {
        pool_free(ptr, st);
        pool_free(info, st);
    };
    if (!force && (reject || total * 100 > sell_total * 106)) {
        drop();
        return 0;
    }
    if (reject) {
        drop();
        set_error("slice-shared offsets: a slice needs more than Lmax + %d (or %d) slots", DIA_SLACK,
                  DIA_MAX_SLOTS);
        return MWCG_ERR_VALUE;
    }
    if ((uint64_t)(stored >> 5) > DIA_START_MASK) {
        drop();
        set_error("slice-shared offsets: too many stored values");
        return MWCG_ERR_VALUE;
    }
    ulonglong2 *rec = nullptr;
    MWCG_CUDA(pool_alloc((void **)&rec, sizeof(ulonglong2) * (size_t)(n_rec > 0 ? n_rec : 1), st));
    // DIA_PAD slots of slack: a chunk of the last slice reads past its end
    MWCG_CUDA(pool_alloc((void **)&M->vals, sizeof(double) * ((size_t)stored + DIA_PAD * SLICE), st));
    MWCG_CUDA(cudaMemsetAsync(M->vals + stored, 0, sizeof(double) * DIA_PAD * SLICE, st));
    dia_walk_kernel<I, true><<<blocks, 256, 0, st>>>(rp, ci, va, A.n_rows, ns, A.row_base, 0, nullptr, nullptr, info,
                                                     ptr, ptr + ns + 1, rec, M->vals, nullptr);
    MWCG_CHECK_LAUNCH();
    int rc = dia_patterns(M, ptr, ptr + ns + 1, info, rec, n_rec, st);
    pool_free(rec, st);
    drop();
    if (rc) return rc;
    A.total = total;
    A.stored = stored;
    A.dia = 1;
    A.col16 = 0;
    A.slice_ptr = M->slice_ptr;
    A.cols = nullptr;
    A.vals = M->vals;
    A.pat = M->pat;
    A.pat_len = M->n_patterns_words;
    MWCG_CUDA(cudaStreamSynchronize(st));
    return 1;
}

template <typename I>
static int build_sell(SellMatrixOwned *M, const I *rp, const I *ci, const double *va, int col_format,
                      int sigma, bool uniform, cudaStream_t st) {
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
        int rc = build_dia<I>(M, rp, ci, va, total, col_format == 2, uniform, st);
        if (rc == 1) {
            pool_free((void *)sell_ptr, st);
            return 0;
        }
        pool_free(M->slice_ptr, st);  // a descriptor table of a rejected attempt
        pool_free(M->vals, st);
        pool_free(M->pat, st);
        M->vals = nullptr;
        M->pat = nullptr;
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
    A.stored = total;
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
    bool uniform = true;
    if (const char *e = getenv("MWCG_DIA_UNIFORM")) uniform = atoi(e) != 0;  // A/B switch (tools/)
    if (col_format >= 0) {
        sigma = (col_format & MWCG_SELL_SIGMA) ? 1 : ((col_format & MWCG_SELL_NO_SIGMA) ? -1 : 0);
        if (col_format & MWCG_DIA_STREAM_VALUES) uniform = false;
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
                                       col_format, sigma, uniform, st)
                 : build_sell<int32_t>(M, (const int32_t *)row_ptr, (const int32_t *)col_idx, values,
                                       col_format, sigma, uniform, st);
    if (rc != 0) {
        sell_destroy(M);
        return rc;
    }
    *out = M;
    return 0;
}

// ---------------------------------------------------------------------------
// Column blocks (irregular matrices whose gathered vector does not fit the
// L2: BASELINE config 5).  The columns are cut into ranges of `cols_per_block`
// and each range becomes its own SELL matrix holding, for every row, the run
// of the row's entries that falls in the range (CSR rows are sorted by
// column, so the run is contiguous and the runs of successive blocks ARE the
// row's entries in order).  K1 walks the blocks one after the other with the
// row's running sum carried in q: the additions and their left-to-right
// order are those of the unblocked walk -- every bit of q is the same -- but
// the gathers of one pass touch only cols_per_block records of p, which stay
// in L2.
// ---------------------------------------------------------------------------
template <typename I>
__global__ void colblock_count_kernel(const I *__restrict__ rp, const I *__restrict__ ci, int64_t n_rows,
                                      int64_t c0, int64_t c1, int64_t *__restrict__ lo_out,
                                      int64_t *__restrict__ cnt) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rows) return;
    const int64_t b = rp[r], e = rp[r + 1];
    auto lower = [&](int64_t key) {  // first k in [b, e) with ci[k] >= key
        int64_t lo = b, hi = e;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)ci[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    const int64_t k0 = lower(c0), k1 = lower(c1);
    lo_out[r] = k0;
    cnt[r] = k1 - k0;
}

template <typename I>
__global__ void colblock_fill_kernel(const I *__restrict__ ci, const double *__restrict__ va, int64_t n_rows,
                                     const int64_t *__restrict__ lo_in, const int64_t *__restrict__ rp_b,
                                     int32_t *__restrict__ rp32, int32_t *__restrict__ ci_b,
                                     double *__restrict__ va_b) {
    // one warp per row
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r > n_rows) return;
    if (r == n_rows) {
        if (lane == 0) rp32[r] = (int32_t)rp_b[r];
        return;
    }
    const int64_t src = lo_in[r], dst = rp_b[r], len = rp_b[r + 1] - dst;
    if (lane == 0) rp32[r] = (int32_t)dst;
    for (int64_t k = lane; k < len; k += 32) {
        ci_b[dst + k] = (int32_t)ci[src + k];
        va_b[dst + k] = va[src + k];
    }
}

// entries whose column lies at least `width` away from their row: the gathers
// that leave the row's L2-resident neighbourhood (what column blocks are for)
template <typename I>
__global__ void far_entries_kernel(const I *__restrict__ rp, const I *__restrict__ ci, int64_t n_rows,
                                   int64_t row_base, int64_t width, unsigned long long *__restrict__ far) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= n_rows) return;
    unsigned int c = 0;
    for (int64_t k = rp[r] + lane; k < rp[r + 1]; k += 32) {
        const int64_t d = (int64_t)ci[k] - (row_base + r);
        c += (d >= width || d <= -width);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0 && c) atomicAdd(far, (unsigned long long)c);
}

template <typename I>
static int far_fraction(double *out, const SellMatrix &A, const I *rp, const I *ci, int64_t width,
                        cudaStream_t st) {
    unsigned long long *d = nullptr, h = 0;
    MWCG_CUDA(pool_alloc((void **)&d, sizeof(unsigned long long), st));
    MWCG_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
    far_entries_kernel<I><<<(unsigned)((A.n_rows * 32 + 255) / 256), 256, 0, st>>>(rp, ci, A.n_rows, A.row_base,
                                                                                  width, d);
    MWCG_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    pool_free(d, st);
    *out = A.nnz > 0 ? (double)h / (double)A.nnz : 0.0;
    return 0;
}

template <typename I>
static int build_colblocks(std::vector<SellMatrixOwned *> &out, const SellMatrix &full, const I *rp, const I *ci,
                           const double *va, int64_t cols_per_block, cudaStream_t st) {
    const int64_t n = full.n_rows;
    const int64_t nb = (full.n_cols + cols_per_block - 1) / cols_per_block;
    int64_t *lo = nullptr, *cnt = nullptr, *rpb = nullptr;
    int32_t *rp32 = nullptr;
    MWCG_CUDA(pool_alloc((void **)&lo, sizeof(int64_t) * (n + 1), st));
    MWCG_CUDA(pool_alloc((void **)&cnt, sizeof(int64_t) * (n + 1), st));
    MWCG_CUDA(pool_alloc((void **)&rpb, sizeof(int64_t) * (n + 1), st));
    MWCG_CUDA(pool_alloc((void **)&rp32, sizeof(int32_t) * (n + 1), st));
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, rpb, n + 1, st);
    void *tmp = nullptr;
    MWCG_CUDA(pool_alloc(&tmp, tmp_bytes, st));
    int rc = 0;
    for (int64_t b = 0; b < nb && rc == 0; b++) {
        const int64_t c0 = b * cols_per_block, c1 = std::min(full.n_cols, c0 + cols_per_block);
        MWCG_CUDA(cudaMemsetAsync(cnt + n, 0, sizeof(int64_t), st));
        colblock_count_kernel<I><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rp, ci, n, c0, c1, lo, cnt);
        MWCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, rpb, n + 1, st));
        int64_t nnz_b = 0;
        MWCG_CUDA(cudaMemcpyAsync(&nnz_b, rpb + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        MWCG_CUDA(cudaStreamSynchronize(st));
        if (nnz_b > INT32_MAX) {
            set_error("column block with more than 2^31-1 entries");
            rc = MWCG_ERR_VALUE;
            break;
        }
        int32_t *ci_b = nullptr;
        double *va_b = nullptr;
        MWCG_CUDA(pool_alloc((void **)&ci_b, sizeof(int32_t) * (size_t)std::max<int64_t>(nnz_b, 1), st));
        MWCG_CUDA(pool_alloc((void **)&va_b, sizeof(double) * (size_t)std::max<int64_t>(nnz_b, 1), st));
        colblock_fill_kernel<I><<<(unsigned)(((n + 1) * 32 + 255) / 256), 256, 0, st>>>(ci, va, n, lo, rpb, rp32, ci_b,
                                                                                      va_b);
        SellMatrixOwned *Mb = nullptr;
        // int32 columns, SELL-sigma when it pays (block rows are short and ragged)
        rc = sell_create(&Mb, n, full.n_cols, nnz_b, rp32, ci_b, va_b, 4, full.row_base, 0, st);
        pool_free(ci_b, st);
        pool_free(va_b, st);
        if (rc == 0) {
            Mb->col0 = c0;
            Mb->col1 = c1;
            out.push_back(Mb);
        }
    }
    MWCG_CUDA(cudaStreamSynchronize(st));
    pool_free(tmp, st);
    pool_free(lo, st);
    pool_free(cnt, st);
    pool_free(rpb, st);
    pool_free(rp32, st);
    if (rc) {
        for (auto *b : out) sell_destroy(b);
        out.clear();
    }
    return rc;
}

int sell_colblocks(std::vector<SellMatrixOwned *> &out, const SellMatrixOwned *M, const void *row_ptr,
                   const void *col_idx, const double *values, int index_bytes, int64_t cols_per_block,
                   bool automatic, cudaStream_t st) {
    out.clear();
    const SellMatrix &A = M->view;
    if (cols_per_block <= 0 || A.dia || A.col16 || A.n_rows == 0 || A.n_cols <= cols_per_block) return 0;
    if (automatic) {
        // the automatic choice also asks that the far gathers matter: a matrix
        // whose columns stay near the diagonal (irregular but local) gains
        // nothing from the passes and would pay their per-row overhead
        double far = 0.0;
        const int rc = index_bytes == 8
                           ? far_fraction<int64_t>(&far, A, (const int64_t *)row_ptr, (const int64_t *)col_idx,
                                                   cols_per_block, st)
                           : far_fraction<int32_t>(&far, A, (const int32_t *)row_ptr, (const int32_t *)col_idx,
                                                   cols_per_block, st);
        if (rc) return rc;
        if (far < 0.10) return 0;
    }
    return index_bytes == 8
               ? build_colblocks<int64_t>(out, A, (const int64_t *)row_ptr, (const int64_t *)col_idx, values,
                                          cols_per_block, st)
               : build_colblocks<int32_t>(out, A, (const int32_t *)row_ptr, (const int32_t *)col_idx, values,
                                          cols_per_block, st);
}

void sell_destroy(SellMatrixOwned *M) {
    if (!M) return;
    pool_free(M->slice_ptr, 0);
    pool_free(M->cols, 0);
    pool_free(M->vals, 0);
    pool_free(M->pat, 0);
    pool_free(M->perm, 0);
    delete M;
}

}  // namespace mwcg
