// ops.cuh -- per-row / per-element device bodies shared by the operator-level
// kernels (ops.cu) and the fused CG kernels (cg.cu).
#pragma once
#include <type_traits>
#include "common.cuh"

namespace mwcg {

// The matrix is streamed once per iteration: its loads carry an evict-first
// L2 policy (ld.global.cs) so they do not push the multi-word vectors, which
// the next kernel re-reads, out of the 126 MB L2.
__device__ __forceinline__ int ld_stream(const int32_t *p) { return __ldcs(p); }
__device__ __forceinline__ int16_t ld_stream(const int16_t *p) { return __ldcs((const short *)p); }
__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }

// One SpMV row: y_r = sum_k add(acc, dxmul(a_rk, x_{c_rk})), acc from +0,
// strictly left to right (spmv_<mode>: _fast.py:284-290, 329-339, 383-393,
// 443-455, 501-513; kernels.py:175-180).
//
// The slice's padded length L (warp-uniform, from slice_ptr) bounds the
// walk; a lane skips entries holding the sentinel column (its row is
// shorter), so no per-row length is loaded.  Columns are decoded from int16
// deltas or int32 (A.col16: a grid-uniform branch).  Chunks of U entries: the
// U column/value loads issue back to back (indices clamped, unconditional),
// then the U gathers of x, then the dependent arithmetic chain -- two memory
// round trips per chunk (a 7-point row is one chunk).
template <typename CT>
struct ColCodec;
template <>
struct ColCodec<int16_t> {  // int16 delta to the (global) row
    static constexpr int16_t SENT = COL16_SENT;
    static __device__ __forceinline__ int col(int grow, int16_t d) { return grow + d; }
};
template <>
struct ColCodec<int32_t> {  // absolute int32 column
    static constexpr int32_t SENT = COL32_SENT;
    static __device__ __forceinline__ int col(int, int32_t d) { return d; }
};

// The two slice words a row's walk starts from (slice_ptr[s], slice_ptr[s+1]:
// entry offsets, or dia descriptors).  Loading them is the first link of
// the row's dependency chain, so callers that walk several rows load the
// next row's words ahead (cg_spmv_pq).  Rows past the last slice clamp to
// it (their results are discarded).
struct SliceWords {
    int64_t w0, w1;
};
__device__ __forceinline__ SliceWords slice_words(const SellMatrix &A, int64_t row) {
    const int64_t sl = min(row >> 5, A.n_slices - 1);
    return SliceWords{__ldg(A.slice_ptr + sl), __ldg(A.slice_ptr + sl + 1)};
}

// Slice-shared-offset walk: the U slot words (warp-uniform broadcast loads
// from the L1-resident pattern table) and the U values issue together; each
// gather's address depends only on its slot word, so the gathers overlap the
// value stream.  Every pattern in the table is followed by DIA_PAD zero words
// and the value array by DIA_PAD slots, so a chunk reads past the slice's
// last slot without clamping: those slots have an empty lane mask.  A lane
// without an entry in a slot gathers its own row (always in bounds) and
// skips the arithmetic.
constexpr int DIA_PAD = 8;  // >= the largest U

template <int M, int U, bool XAOS>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row_dia(const SellMatrix &A,
                                                               const double *__restrict__ x, int64_t ldx,
                                                               int64_t row, SliceWords sw) {
    static_assert(U <= DIA_PAD, "pattern padding must cover a chunk");
    using Ar = mw::Arith<M>;
    constexpr int W = Ar::W;
    // slice descriptor: (start / 32) | (pattern base << 36)  (sell.cu: dia_patterns)
    constexpr uint64_t LO = (1ull << 36) - 1;
    const uint64_t d0 = (uint64_t)sw.w0, d1 = (uint64_t)sw.w1;
    const int64_t s0 = (int64_t)(d0 & LO) << 5;
    const int L = (int)((d1 & LO) - (d0 & LO));
    const int lane = (int)(row & 31);
    const int grow = (int)(A.row_base + row);
    const uint64_t *__restrict__ op = A.om + (d0 >> 36);
    const double *__restrict__ vp = A.vals + s0 + lane;
    mw::V<W> s = mw::zero<W>();
    for (int k0 = 0; k0 < L; k0 += U, op += U, vp += U * SLICE) {
        uint64_t om[U];
        double a[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            om[u] = __ldg(op + u);
            a[u] = ld_stream(vp + u * SLICE);
        }
        bool ok[U];
        mw::V<W> xv[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            ok[u] = (uint32_t)(om[u] >> 32) & (1u << lane);
            const int c = grow + (ok[u] ? (int)(uint32_t)om[u] : 0);
            xv[u] = XAOS ? mw::load_aos_ro<W>(x, c) : mw::load_ro<W>(x, ldx, c);
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            if (ok[u]) s = Ar::add(s, Ar::dxmul(a[u], xv[u]));
    }
    return s;
}

template <int M, int U, typename CT, bool XAOS = false>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row_sell(const SellMatrix &A,
                                                                const double *__restrict__ x, int64_t ldx,
                                                                int64_t row, SliceWords sw) {
    using Ar = mw::Arith<M>;
    constexpr int W = Ar::W;
    // `row` is the storage position (slice row); columns decode against the
    // natural row (SELL-sigma: sell_row)
    const int64_t s0 = sw.w0;
    const int L = (int)((sw.w1 - s0) >> 5);
    const int64_t off = s0 + (row & 31);
    const int grow = (int)(A.row_base + (std::is_same<CT, int16_t>::value ? sell_row(A, row) : row));
    const CT *__restrict__ cp = (const CT *)A.cols + off;
    const double *__restrict__ vp = A.vals + off;
    mw::V<W> s = mw::zero<W>();
    for (int k0 = 0; k0 < L; k0 += U) {
        int c[U];
        bool ok[U];
        double a[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t kk = min(k0 + u, L - 1);
            const CT d = ld_stream(cp + kk * SLICE);
            a[u] = ld_stream(vp + kk * SLICE);
            ok[u] = (k0 + u < L) && (d != ColCodec<CT>::SENT);
            c[u] = ok[u] ? ColCodec<CT>::col(grow, d) : 0;
        }
        mw::V<W> xv[U];
#pragma unroll
        for (int u = 0; u < U; u++)
            xv[u] = XAOS ? mw::load_aos_ro<W>(x, c[u]) : mw::load_ro<W>(x, ldx, c[u]);
#pragma unroll
        for (int u = 0; u < U; u++)
            if (ok[u]) s = Ar::add(s, Ar::dxmul(a[u], xv[u]));
    }
    return s;
}

// one row of y = A x in the matrix's layout
template <int M, int U, typename CT, bool XAOS = false>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row(const SellMatrix &A,
                                                           const double *__restrict__ x, int64_t ldx,
                                                           int64_t row, SliceWords sw) {
    if constexpr (std::is_same<CT, DiaTag>::value) return spmv_row_dia<M, U, XAOS>(A, x, ldx, row, sw);
    else return spmv_row_sell<M, U, CT, XAOS>(A, x, ldx, row, sw);
}
template <int M, int U, typename CT, bool XAOS = false>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row(const SellMatrix &A,
                                                           const double *__restrict__ x, int64_t ldx,
                                                           int64_t row) {
    return spmv_row<M, U, CT, XAOS>(A, x, ldx, row, slice_words(A, row));
}

// dispatch helper: F(CT) with the matrix's format tag / column type
#define MWCG_COLS(A, F) ((A).dia ? F(DiaTag) : ((A).col16 ? F(int16_t) : F(int32_t)))

}  // namespace mwcg
