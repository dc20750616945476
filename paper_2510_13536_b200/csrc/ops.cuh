// ops.cuh -- per-row / per-element device bodies shared by the operator-level
// kernels (ops.cu) and the fused CG kernels (cg.cu).
#pragma once
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
template <int M, int U = 8>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row(const SellMatrix &A,
                                                           const double *__restrict__ x, int64_t ldx,
                                                           int64_t row) {
    using Ar = mw::Arith<M>;
    constexpr int W = Ar::W;
    const int64_t sl = row >> 5;
    const int64_t s0 = __ldg(A.slice_ptr + sl);
    const int L = (int)((__ldg(A.slice_ptr + sl + 1) - s0) >> 5);
    const int64_t off = s0 + (row & 31);
    const int64_t grow = A.row_base + row;
    const double *__restrict__ vp = A.vals + off;
    mw::V<W> s = mw::zero<W>();
    for (int k0 = 0; k0 < L; k0 += U) {
        int64_t c[U];
        bool ok[U];
        double a[U];
        if (A.col16) {
            const int16_t *__restrict__ cp = (const int16_t *)A.cols + off;
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int kk = min(k0 + u, L - 1);
                const int16_t d = ld_stream(cp + (int64_t)kk * SLICE);
                ok[u] = (k0 + u < L) && (d != COL16_SENT);
                c[u] = ok[u] ? grow + d : 0;
            }
        } else {
            const int32_t *__restrict__ cp = (const int32_t *)A.cols + off;
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int kk = min(k0 + u, L - 1);
                const int32_t d = ld_stream(cp + (int64_t)kk * SLICE);
                ok[u] = (k0 + u < L) && (d != COL32_SENT);
                c[u] = ok[u] ? d : 0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) a[u] = ld_stream(vp + (int64_t)min(k0 + u, L - 1) * SLICE);
        mw::V<W> xv[U];
#pragma unroll
        for (int u = 0; u < U; u++) xv[u] = mw::load_ro<W>(x, ldx, c[u]);
#pragma unroll
        for (int u = 0; u < U; u++)
            if (ok[u]) s = Ar::add(s, Ar::dxmul(a[u], xv[u]));
    }
    return s;
}

}  // namespace mwcg
