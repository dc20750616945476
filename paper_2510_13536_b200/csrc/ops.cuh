// ops.cuh -- per-row / per-element device bodies shared by the operator-level
// kernels (ops.cu) and the fused CG kernels (cg.cu).
#pragma once
#include <type_traits>
#include "common.cuh"

namespace mwcg {

// The matrix is streamed once per iteration.  Its loads (a) do not allocate
// in L1 -- the L1 is kept for the gathered vector, whose near-diagonal records
// are re-read by neighbouring rows -- and (b) carry an evict-first L2 policy,
// so they do not push the multi-word vectors, which the next kernel re-reads,
// out of the 126 MB L2.  (MWCG_STREAM_EF: the plain ld.global.cs form.)
#ifdef MWCG_STREAM_EF
__device__ __forceinline__ int ld_stream(const int32_t *p) { return __ldcs(p); }
__device__ __forceinline__ int16_t ld_stream(const int16_t *p) { return __ldcs((const short *)p); }
__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }
#else
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ int ld_stream(const int32_t *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(evict_first_policy()));
    return v;
}
__device__ __forceinline__ int16_t ld_stream(const int16_t *p) {
    short v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s16 %0, [%1], %2;"
                 : "=h"(v) : "l"(p), "l"(evict_first_policy()));
    return v;
}
__device__ __forceinline__ double ld_stream(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(evict_first_policy()));
    return v;
}
#endif
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

// The two slice words a row's walk starts from: slice_ptr[s], slice_ptr[s+1]
// (entry offsets, SELL layouts) or the slice's descriptor pair (dia layout,
// one 16-B load).  Loading them is the first link of the row's dependency
// chain, so callers that walk several rows load the next row's words ahead
// (cg_spmv_pq).  Rows past the last slice clamp to it (their results are
// discarded).
struct SliceWords {
    int64_t w0, w1;
};
template <typename CT>
__device__ __forceinline__ SliceWords slice_words(const SellMatrix &A, int64_t row) {
    const int sl = min((int)(row >> 5), (int)A.n_slices - 1);  // rows < 2^31
    if constexpr (std::is_same<CT, DiaTag>::value) {
        const longlong2 d = __ldg(reinterpret_cast<const longlong2 *>(A.slice_ptr) + sl);
        return SliceWords{d.x, d.y};
    } else {
        return SliceWords{__ldg(A.slice_ptr + sl), __ldg(A.slice_ptr + sl + 1)};
    }
}

// Slice-shared-offset walk: the U slot records (warp-uniform broadcast loads
// from the L1-resident pattern table) and the U values issue together; each
// gather's address depends only on its slot word, so the gathers overlap the
// value stream.  Every pattern in the table is followed by DIA_PAD zero
// records and the value array by DIA_PAD slots, so a chunk reads past the
// slice's last slot without clamping: those slots have an empty lane mask.  A
// lane without an entry in a slot gathers its own row (always in bounds) and
// skips the arithmetic.  A slice whose slots are value-uniform (descriptor
// flag) takes its values from the records and streams nothing.
constexpr int DIA_PAD = 8;  // >= the largest U
constexpr int DIA_LBITS = 40;                       // descriptor word 0: start/32 | L << 40 | uniform << 48
constexpr uint64_t DIA_START_MASK = (1ull << DIA_LBITS) - 1;
constexpr int DIA_MAX_SLOTS = 255;

// base + off * SCALE bytes as ONE wide multiply-add (IMAD.WIDE); written in
// PTX because the compiler otherwise sign-extends the offset and adds the
// halves separately (three instructions per gather).
template <int SCALE>
__device__ __forceinline__ const double *wide_offset(const double *base, int off) {
    const double *r;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"(off), "n"(SCALE), "l"(base));
    return r;
}

// Gather of x at (row + off): the row's own record address xg (computed once
// per row) plus a 32-bit offset.
template <int W, bool XAOS>
__device__ __forceinline__ mw::V<W> dia_gather(const double *__restrict__ xg, int64_t ldx, int off) {
    mw::V<W> r;
    if (XAOS) {
        const double *__restrict__ e = wide_offset<8 * W>(xg, off);
        if (W == 2) {
            const double2 t = __ldg(reinterpret_cast<const double2 *>(e));
            r.w[0] = t.x;
            r.w[W - 1] = t.y;
        } else {
#pragma unroll
            for (int k = 0; k < W; k++) r.w[k] = __ldg(e + k);
        }
    } else {
        const double *__restrict__ e = wide_offset<8>(xg, off);
#pragma unroll
        for (int k = 0; k < W; k++) r.w[k] = __ldg(e + k * ldx);
    }
    return r;
}

// s = ok ? t : s, word by word (a lane without an entry in the slot keeps its sum)
template <int W>
__device__ __forceinline__ mw::V<W> keep_if(bool ok, mw::V<W> t, mw::V<W> s) {
#pragma unroll
    for (int k = 0; k < W; k++) s.w[k] = ok ? t.w[k] : s.w[k];
    return s;
}

// One chunk of N slots of a slice-shared-offset row.  The N records (and,
// for a streamed slice, the N values) are loaded first, then the N gathers
// issue, then the arithmetic runs -- branch-free: a lane without an entry in
// a slot gathers its own row (always in bounds), multiplies, and keeps its
// old sum by a select.  (With a branch on the lane predicate the compiler
// sinks each slot's loads into its branch: one memory round trip per entry.)
// FULL: every slot of the slice is present in all 32 rows (interior stencil /
// band slices): no lane predicate, no offset select, no keep-select.
template <int M, int N, bool XAOS, bool UNIFORM, bool FULL = false>
__device__ __forceinline__ void dia_chunk(mw::V<mw::Arith<M>::W> &s, const ulonglong2 *__restrict__ op,
                                          const double *__restrict__ vp, const double *__restrict__ xg,
                                          int64_t ldx, uint32_t lbit, const SellMatrix &A, int64_t grow) {
    using Ar = mw::Arith<M>;
    constexpr int W = Ar::W;
    double a[N];
    bool ok[N];
    mw::V<W> xv[N];
#pragma unroll
    for (int u = 0; u < N; u++) {
        uint64_t om;
        MWCG_ASSERT(op + u >= A.pat && op + u < A.pat + A.pat_len);
        MWCG_ASSERT(UNIFORM || (vp + u * SLICE >= A.vals && vp + u * SLICE < A.vals + A.stored + DIA_PAD * SLICE));
        if (UNIFORM) {
            const ulonglong2 rec = __ldg(op + u);
            om = rec.x;
            a[u] = __longlong_as_double((long long)rec.y);
        } else {
            om = __ldg(&op[u].x);
            a[u] = ld_stream(vp + u * SLICE);
        }
        ok[u] = FULL || ((uint32_t)(om >> 32) & lbit) != 0;
        MWCG_ASSERT(!FULL || (uint32_t)(om >> 32) == 0xffffffffu);
        MWCG_ASSERT(!ok[u] || (grow + (int)(uint32_t)om >= 0 && grow + (int)(uint32_t)om < A.n_cols));
        xv[u] = dia_gather<W, XAOS>(xg, ldx, ok[u] ? (int)(uint32_t)om : 0);
    }
    // streamed TW/QTW rows keep the lane branch (C4 QTW K1: 78 us against
    // 87 us branch-free; every other case is as fast or faster branch-free)
    constexpr bool BRANCHY = !UNIFORM && W == 3 && !FULL;
#pragma unroll
    for (int u = 0; u < N; u++) {
        if (FULL) {
            s = Ar::add(s, Ar::dxmul(a[u], xv[u]));
        } else if (BRANCHY) {
            if (ok[u]) s = Ar::add(s, Ar::dxmul(a[u], xv[u]));
        } else {
            s = keep_if<W>(ok[u], Ar::add(s, Ar::dxmul(a[u], xv[u])), s);
        }
    }
}

// the slots of a row: full chunks of U, then one exact chunk for the rest
template <int M, int U, bool XAOS, bool UNIFORM, bool FULL = false>
__device__ __forceinline__ void dia_walk(mw::V<mw::Arith<M>::W> &s, int L, const ulonglong2 *__restrict__ op,
                                         const double *__restrict__ vp, const double *__restrict__ xg,
                                         int64_t ldx, uint32_t lbit, const SellMatrix &A, int64_t grow) {
    int k0 = 0;
    for (; k0 + U <= L; k0 += U, op += U, vp += U * SLICE) dia_chunk<M, U, XAOS, UNIFORM, FULL>(s, op, vp, xg, ldx, lbit, A, grow);
    const int rem = L - k0;
    if (U > 1 && rem == 1) dia_chunk<M, 1, XAOS, UNIFORM, FULL>(s, op, vp, xg, ldx, lbit, A, grow);
    if (U > 2 && rem == 2) dia_chunk<M, 2, XAOS, UNIFORM, FULL>(s, op, vp, xg, ldx, lbit, A, grow);
    if (U > 3 && rem == 3) dia_chunk<M, 3, XAOS, UNIFORM, FULL>(s, op, vp, xg, ldx, lbit, A, grow);
    if (U > 4 && rem >= 4) {  // U up to 8: 4 + (rem - 4)
        dia_chunk<M, 4, XAOS, UNIFORM, FULL>(s, op, vp, xg, ldx, lbit, A, grow);
        op += 4;
        vp += 4 * SLICE;
        if (rem == 5) dia_chunk<M, 1, XAOS, UNIFORM, FULL>(s, op, vp, xg, ldx, lbit, A, grow);
        if (rem == 6) dia_chunk<M, 2, XAOS, UNIFORM, FULL>(s, op, vp, xg, ldx, lbit, A, grow);
        if (rem == 7) dia_chunk<M, 3, XAOS, UNIFORM, FULL>(s, op, vp, xg, ldx, lbit, A, grow);
    }
}

// Two rows of one thread walked TOGETHER (rows pos and pos + NT of a tile) when
// both sit in value-uniform slices with the SAME pattern (interior stencil
// rows): the slot records are loaded once, each slot's two gathers issue
// together and the two multi-word sums advance as independent dependency
// chains.  A dependent FP64 operation issues every ~20 cycles, so one chain per
// warp with 8 warps per scheduler leaves the FP64 pipe at ~45 %; two chains per
// thread double the arithmetic in flight without more warps.  Each row's own
// additions and their order are unchanged.
template <int M, int N, bool XAOS>
__device__ __forceinline__ void dia_chunk_pair(mw::V<mw::Arith<M>::W> &sa, mw::V<mw::Arith<M>::W> &sb,
                                               const ulonglong2 *__restrict__ op,
                                               const double *__restrict__ xga, const double *__restrict__ xgb,
                                               int64_t ldx, uint32_t lbit) {
    using Ar = mw::Arith<M>;
    constexpr int W = Ar::W;
    double a[N];
    bool ok[N];
    mw::V<W> xa[N], xb[N];
#pragma unroll
    for (int u = 0; u < N; u++) {
        const ulonglong2 rec = __ldg(op + u);
        a[u] = __longlong_as_double((long long)rec.y);
        ok[u] = ((uint32_t)(rec.x >> 32) & lbit) != 0;
        const int off = ok[u] ? (int)(uint32_t)rec.x : 0;
        xa[u] = dia_gather<W, XAOS>(xga, ldx, off);
        xb[u] = dia_gather<W, XAOS>(xgb, ldx, off);
    }
#pragma unroll
    for (int u = 0; u < N; u++) {
        sa = keep_if<W>(ok[u], Ar::add(sa, Ar::dxmul(a[u], xa[u])), sa);
        sb = keep_if<W>(ok[u], Ar::add(sb, Ar::dxmul(a[u], xb[u])), sb);
    }
}

// true (and both sums computed) when the pair could be walked together;
// false: the caller walks the rows one by one
template <int M, int UP, bool XAOS>
__device__ __forceinline__ bool spmv_pair_dia(const SellMatrix &A, const double *__restrict__ x, int64_t ldx,
                                              int64_t rowa, int64_t rowb, SliceWords swa, SliceWords swb,
                                              mw::V<mw::Arith<M>::W> &sa, mw::V<mw::Arith<M>::W> &sb) {
    constexpr int W = mw::Arith<M>::W;
    const uint32_t fa = (uint32_t)((uint64_t)swa.w0 >> DIA_LBITS), fb = (uint32_t)((uint64_t)swb.w0 >> DIA_LBITS);
    // same pattern base, both uniform (then the slot counts agree too)
    if (swa.w1 != swb.w1 || ((fa & fb) & 0x100u) == 0 || ((fa ^ fb) & 0xffu) != 0) return false;
    const int L = (int)(fa & 0xffu);
    const uint32_t lbit = 1u << ((int)rowa & 31);
    const double *__restrict__ xga = x + (A.row_base + rowa) * (XAOS ? W : 1);
    const double *__restrict__ xgb = x + (A.row_base + rowb) * (XAOS ? W : 1);
    const ulonglong2 *__restrict__ op = A.pat + swa.w1;
    sa = mw::zero<W>();
    sb = mw::zero<W>();
    int k0 = 0;
    for (; k0 + UP <= L; k0 += UP, op += UP) dia_chunk_pair<M, UP, XAOS>(sa, sb, op, xga, xgb, ldx, lbit);
    const int rem = L - k0;
    if (UP > 1 && rem == 1) dia_chunk_pair<M, 1, XAOS>(sa, sb, op, xga, xgb, ldx, lbit);
    if (UP > 2 && rem == 2) dia_chunk_pair<M, 2, XAOS>(sa, sb, op, xga, xgb, ldx, lbit);
    if (UP > 3 && rem == 3) dia_chunk_pair<M, 3, XAOS>(sa, sb, op, xga, xgb, ldx, lbit);
    return true;
}

template <int M, int U, bool XAOS, int UU = U>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row_dia(const SellMatrix &A,
                                                               const double *__restrict__ x, int64_t ldx,
                                                               int64_t row, SliceWords sw) {
    static_assert(U <= 8 && UU <= 8, "chunk tails cover U <= 8");
    using Ar = mw::Arith<M>;
    constexpr int W = Ar::W;
    const uint64_t d0 = (uint64_t)sw.w0;
    const int L = (int)((uint32_t)(d0 >> DIA_LBITS) & 0xffu);
    const bool uniform = ((uint32_t)(d0 >> DIA_LBITS) & 0x100u) != 0;
    MWCG_ASSERT(A.row_base + row < A.n_cols && sw.w1 >= 0 && sw.w1 + L <= A.pat_len);
    const uint32_t lbit = 1u << ((int)row & 31);
    // the row's own element: every gather is this address + a slot offset
    const double *__restrict__ xg = x + (A.row_base + row) * (XAOS ? W : 1);
    const ulonglong2 *__restrict__ op = A.pat + sw.w1;
    mw::V<W> s = mw::zero<W>();
    // the predicate-free walk of full slices pays for FP64 only (C4 57.5 -> 51.1
    // us/it); the multi-word modes lose more to the extra code than the selects
    // cost (TW +12 %, QTW +5-9 %, DW/QDW +-2 %: profiles/r3d_full_slices_sweep.json)
    const bool full = W == 1 && ((uint32_t)(d0 >> DIA_LBITS) & 0x200u) != 0;
    if (uniform) {
        if (full) dia_walk<M, UU, XAOS, true, true>(s, L, op, nullptr, xg, ldx, lbit, A, A.row_base + row);
        else dia_walk<M, UU, XAOS, true>(s, L, op, nullptr, xg, ldx, lbit, A, A.row_base + row);
    } else {
        const double *__restrict__ vp = A.vals + (((int64_t)(d0 & DIA_START_MASK) << 5) + ((int)row & 31));
        if (full) dia_walk<M, U, XAOS, false, true>(s, L, op, vp, xg, ldx, lbit, A, A.row_base + row);
        else dia_walk<M, U, XAOS, false>(s, L, op, vp, xg, ldx, lbit, A, A.row_base + row);
    }
    return s;
}

// `sum0`: the sum the walk starts from (+0, or the row's running sum when the
// matrix is one column block of a larger one: sell.cu, column blocks)
template <int M, int U, typename CT, bool XAOS = false>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row_sell(const SellMatrix &A,
                                                                const double *__restrict__ x, int64_t ldx,
                                                                int64_t row, SliceWords sw,
                                                                mw::V<mw::Arith<M>::W> sum0) {
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
    mw::V<W> s = sum0;
    for (int k0 = 0; k0 < L; k0 += U) {
        int c[U];
        bool ok[U];
        double a[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t kk = min(k0 + u, L - 1);
            MWCG_ASSERT(off + kk * SLICE >= 0 && off + kk * SLICE < A.total);
            const CT d = ld_stream(cp + kk * SLICE);
            a[u] = ld_stream(vp + kk * SLICE);
            ok[u] = (k0 + u < L) && (d != ColCodec<CT>::SENT);
            c[u] = ok[u] ? ColCodec<CT>::col(grow, d) : 0;
            MWCG_ASSERT(c[u] >= 0 && c[u] < A.n_cols);
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
template <int M, int U, typename CT, bool XAOS = false, int UU = U>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row(const SellMatrix &A,
                                                           const double *__restrict__ x, int64_t ldx,
                                                           int64_t row, SliceWords sw) {
    if constexpr (std::is_same<CT, DiaTag>::value) return spmv_row_dia<M, U, XAOS, UU>(A, x, ldx, row, sw);
    else return spmv_row_sell<M, U, CT, XAOS>(A, x, ldx, row, sw, mw::zero<mw::Arith<M>::W>());
}
template <int M, int U, typename CT, bool XAOS = false>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> spmv_row(const SellMatrix &A,
                                                           const double *__restrict__ x, int64_t ldx,
                                                           int64_t row) {
    return spmv_row<M, U, CT, XAOS>(A, x, ldx, row, slice_words<CT>(A, row));
}

// dispatch helper: F(CT) with the matrix's format tag / column type
#define MWCG_COLS(A, F) ((A).dia ? F(DiaTag) : ((A).col16 ? F(int16_t) : F(int32_t)))

}  // namespace mwcg
