// ops.cuh -- per-row / per-element device bodies shared by the operator-level
// kernels (ops.cu) and the fused CG kernels (cg.cu).
#pragma once
#include "common.cuh"

namespace mwcg {

// One SpMV row: y_r = sum_k add(acc, dxmul(a_rk, x_{c_rk})), acc from +0,
// strictly left to right (spmv_<mode>: _fast.py:284-290, 329-339, 383-393,
// 443-455, 501-513; kernels.py:175-180).  Column/value loads for a chunk of
// U entries are issued before the dependent arithmetic chain.
template <int M>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row(const SellMatrix &A,
                                                           const double *__restrict__ x, int64_t ldx,
                                                           int64_t row) {
    using Ar = mw::Arith<M>;
    constexpr int W = Ar::W;
    constexpr int U = 4;
    const int len = __ldg(A.row_len + row);
    const int64_t off = __ldg(A.slice_ptr + (row >> 5)) + (row & 31);
    const int32_t *__restrict__ cp = A.cols + off;
    const double *__restrict__ vp = A.vals + off;
    mw::V<W> s = mw::zero<W>();
    int k = 0;
    for (; k + U <= len; k += U) {
        int c[U];
        double a[U];
        mw::V<W> xv[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            c[u] = __ldg(cp + (int64_t)(k + u) * SLICE);
            a[u] = __ldg(vp + (int64_t)(k + u) * SLICE);
        }
#pragma unroll
        for (int u = 0; u < U; u++) xv[u] = mw::load_ro<W>(x, ldx, c[u]);
#pragma unroll
        for (int u = 0; u < U; u++) s = Ar::add(s, Ar::dxmul(a[u], xv[u]));
    }
    for (; k < len; k++) {
        int c = __ldg(cp + (int64_t)k * SLICE);
        double a = __ldg(vp + (int64_t)k * SLICE);
        s = Ar::add(s, Ar::dxmul(a, mw::load_ro<W>(x, ldx, c)));
    }
    return s;
}

}  // namespace mwcg
