// ops.cuh -- per-row / per-element device bodies shared by the operator-level
// kernels (ops.cu) and the fused CG kernels (cg.cu).
#pragma once
#include "common.cuh"

namespace mwcg {

// One SpMV row: y_r = sum_k add(acc, dxmul(a_rk, x_{c_rk})), acc from +0,
// strictly left to right (spmv_<mode>: _fast.py:284-290, 329-339, 383-393,
// 443-455, 501-513; kernels.py:175-180).
//
// Memory-level parallelism: a row is fetched in chunks of U entries.  The
// U column/value loads of a chunk are UNCONDITIONAL (indices clamped to the
// row's last entry, a cache hit) so they issue back to back, then the U
// gathers of x, then the dependent arithmetic chain -- two memory round trips
// per chunk (a 7-point row is one chunk).  Only the arithmetic is predicated.
template <int U>
struct RowFetch {
    int c[U];
    double a[U];
};

// The matrix is streamed once per iteration: its loads carry an evict-first
// L2 policy (ld.global.cs) so they do not push the multi-word vectors, which
// the next kernel re-reads, out of the 126 MB L2.
__device__ __forceinline__ int ld_stream(const int32_t *p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }

// Row descriptor: entry count and the address of entry 0 (SELL-32).
__device__ __forceinline__ void row_desc(const SellMatrix &A, int64_t row, int &len, int64_t &off) {
    len = ld_stream(A.row_len + row);
    off = __ldg(A.slice_ptr + (row >> 5)) + (row & 31);
}

template <int U>
__device__ __forceinline__ void fetch_chunk(const SellMatrix &A, int64_t off, int len, int k0,
                                            RowFetch<U> &f) {
    const int last = len - 1;
    if (last < 0) return;
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int kk = min(k0 + u, last);
        f.c[u] = ld_stream(A.cols + off + (int64_t)kk * SLICE);
        f.a[u] = ld_stream(A.vals + off + (int64_t)kk * SLICE);
    }
}

template <int M, int U>
__device__ __forceinline__ void consume_chunk(const RowFetch<U> &f, int len, int k0,
                                              const double *__restrict__ x, int64_t ldx,
                                              mw::V<mw::Arith<M>::W> &s) {
    using Ar = mw::Arith<M>;
    constexpr int W = Ar::W;
    if (len <= k0) return;
    mw::V<W> xv[U];
#pragma unroll
    for (int u = 0; u < U; u++) xv[u] = mw::load_ro<W>(x, ldx, f.c[u]);
#pragma unroll
    for (int u = 0; u < U; u++)
        if (k0 + u < len) s = Ar::add(s, Ar::dxmul(f.a[u], xv[u]));
}

template <int M, int U = 8>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row(const SellMatrix &A,
                                                           const double *__restrict__ x, int64_t ldx,
                                                           int64_t row) {
    constexpr int W = mw::Arith<M>::W;
    int len;
    int64_t off;
    row_desc(A, row, len, off);
    RowFetch<U> f;
    mw::V<W> s = mw::zero<W>();
    for (int k0 = 0; k0 < len; k0 += U) {
        fetch_chunk<U>(A, off, len, k0, f);
        consume_chunk<M, U>(f, len, k0, x, ldx, s);
    }
    return s;
}

}  // namespace mwcg
