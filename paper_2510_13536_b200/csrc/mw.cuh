// mw.cuh -- multi-word FP64 arithmetic for sm_100a (device, register-resident).
//
// Bit-exact restatement of the reference scalar algorithms:
//   EFTs                      _fast.py:41-60        (eft.py:78-122)
//   DW / QDW add, mul, mixed  _fast.py:63-126       (multiword.py:101-168)
//   TW / QTW add, mul, mixed  _fast.py:129-277      (multiword.py:175-323)
//   division                  multiword.py:360-409
//
// REQUIRED compile flags: -fmad=false (no contraction: the reference kernels
// are unfused and TwoProd's p=a*b must not fuse into a later add), no
// --use_fast_math (IEEE div/sqrt).  Fused operations are explicit __fma_rn.
//
// The TW operations are branchy in the reference (3+3 magnitude merge, VecSum,
// VSEB with data-dependent early exit).  Here they are unrolled register code
// with selects: no local-memory arrays, identical results including the
// tie rule (ties take the FIRST operand, _fast.py:186).
#pragma once
#include <cstdint>

namespace mw {

enum Mode : int { FP64 = 0, DW = 1, QDW = 2, TW = 3, QTW = 4 };

__host__ __device__ constexpr int words_of(int m) { return m == FP64 ? 1 : (m <= QDW ? 2 : 3); }

template <int W>
struct V {
    double w[W];
};

#define MWI __device__ __forceinline__

// --------------------------------------------------------------- EFTs
MWI void two_sum(double a, double b, double &x, double &y) {
    double s = __dadd_rn(a, b);
    double z = __dsub_rn(s, a);
    y = __dadd_rn(__dsub_rn(a, __dsub_rn(s, z)), __dsub_rn(b, z));
    x = s;
}
MWI void quick_two_sum(double a, double b, double &x, double &y) {
    double s = __dadd_rn(a, b);
    y = __dadd_rn(__dsub_rn(a, s), b);
    x = s;
}
MWI void two_prod(double a, double b, double &x, double &y) {
    double p = __dmul_rn(a, b);
    y = __fma_rn(a, b, -p);
    x = p;
}

// magnitude compare |a| >= |b| (IEEE: false if either is NaN)
MWI bool mag_ge(double a, double b) { return fabs(a) >= fabs(b); }

// ------------------------------------------------------------ DW / QDW
MWI V<2> dw_add(V<2> a, V<2> b) {
    double s, e;
    two_sum(a.w[0], b.w[0], s, e);
    e = __dadd_rn(__dadd_rn(e, a.w[1]), b.w[1]);
    V<2> r;
    quick_two_sum(s, e, r.w[0], r.w[1]);
    return r;
}
MWI V<2> qdw_add(V<2> a, V<2> b) {
    double s, e;
    two_sum(a.w[0], b.w[0], s, e);
    e = __dadd_rn(__dadd_rn(e, a.w[1]), b.w[1]);
    return V<2>{{s, e}};
}
MWI V<2> dw_mul(V<2> a, V<2> b) {
    double p, e;
    two_prod(a.w[0], b.w[0], p, e);
    e = __fma_rn(a.w[0], b.w[1], e);
    e = __fma_rn(a.w[1], b.w[0], e);
    V<2> r;
    quick_two_sum(p, e, r.w[0], r.w[1]);
    return r;
}
MWI V<2> qdw_mul(V<2> a, V<2> b) {
    double p, e;
    two_prod(a.w[0], b.w[0], p, e);
    e = __fma_rn(a.w[0], b.w[1], e);
    e = __fma_rn(a.w[1], b.w[0], e);
    return V<2>{{p, e}};
}
MWI V<2> dxdw_mul(double a, V<2> b) {
    double p, e;
    two_prod(a, b.w[0], p, e);
    e = __fma_rn(a, b.w[1], e);
    V<2> r;
    quick_two_sum(p, e, r.w[0], r.w[1]);
    return r;
}
MWI V<2> dxqdw_mul(double a, V<2> b) {
    double p, e;
    two_prod(a, b.w[0], p, e);
    e = __fma_rn(a, b.w[1], e);
    return V<2>{{p, e}};
}
MWI V<2> dxdw_add(double a, V<2> b) {
    double s, e;
    two_sum(a, b.w[0], s, e);
    e = __dadd_rn(e, b.w[1]);
    V<2> r;
    quick_two_sum(s, e, r.w[0], r.w[1]);
    return r;
}
MWI V<2> dxqdw_add(double a, V<2> b) {
    double s, e;
    two_sum(a, b.w[0], s, e);
    e = __dadd_rn(e, b.w[1]);
    return V<2>{{s, e}};
}
// _norm_dw: _fast.py:121-126
MWI V<2> norm_dw(V<2> a) {
    V<2> r;
    if (mag_ge(a.w[0], a.w[1])) quick_two_sum(a.w[0], a.w[1], r.w[0], r.w[1]);
    else two_sum(a.w[0], a.w[1], r.w[0], r.w[1]);
    return r;
}

// ------------------------------------------------------------ TW / QTW
// VSEB_m over an error-free chain e[0..N-1] (_fast.py:136-163,
// multiword.py:187-203): emit the rounded partial sum whenever the running
// error is non-zero; stop after m words.  Branch-free: every step is
// computed, the emission slot is selected with predicates (cnt <= i is known
// at compile time per step), and steps after the m-th emission are masked.
//
// When e is a VecSum chain (every call site here), step 0 is two_sum(e0, e1)
// with e1 the exact error of the rounding that produced e0, so
// fl(e0 + e1) = e0 and the error is e1 for finite e0; for non-finite e0, e1 is
// NaN and both forms give NaN.  Step 0 therefore costs one DADD
// (CHAIN = true).
template <int N, int M, bool CHAIN = true>
MWI V<3> vseb_general(const double (&e)[N]) {
    double r0 = 0.0, r1 = 0.0, r2 = 0.0;
    int cnt = 0;
    bool done = false;
    double eps = e[0];
#pragma unroll
    for (int i = 0; i < N - 1; i++) {
        double rj, en;
        if (CHAIN && i == 0) {
            rj = __dadd_rn(eps, e[1]);
            en = e[1];
        } else {
            two_sum(eps, e[i + 1], rj, en);
        }
        const bool nz = en != 0.0;
        const bool emit = nz && !done;
        r0 = (emit && cnt == 0) ? rj : r0;
        if (i >= 1) r1 = (emit && cnt == 1) ? rj : r1;
        if (i >= 2 && M == 3) r2 = (emit && cnt == 2) ? rj : r2;
        if (i >= M - 1) done = done || (emit && cnt == M - 1);
        cnt += emit ? 1 : 0;
        eps = nz ? en : rj;
    }
    if (!done) {
        r0 = (cnt == 0) ? eps : r0;
        r1 = (cnt == 1) ? eps : r1;
        if (M == 3) r2 = (cnt == 2) ? eps : r2;
    }
    return V<3>{{r0, r1, r2}};
}

template <int N, int M, bool CHAIN = true>
MWI V<3> vseb(const double (&e)[N]) {
    return vseb_general<N, M, CHAIN>(e);
}

// _vec_sum: multiword.py:175-184 (bottom-up chained TwoSum)
template <int N>
MWI void vec_sum(const double (&z)[N], double (&e)[N]) {
    double s = z[N - 1];
#pragma unroll
    for (int k = N - 2; k >= 0; k--) {
        double err;
        two_sum(z[k], s, s, err);
        e[k + 1] = err;
    }
    e[0] = s;
}

// _vecsum3: _fast.py:129-133 (top-down; the QTW normalization)
MWI V<3> vecsum3(V<3> a) {
    V<3> r;
    double c1;
    two_sum(a.w[0], a.w[1], r.w[0], c1);
    two_sum(c1, a.w[2], r.w[1], r.w[2]);
    return r;
}

// _renorm3: _fast.py:166-175
MWI V<3> renorm3(double c0, double c1, double c2) {
    double z[3] = {c0, c1, c2}, e[3];
    vec_sum<3>(z, e);
    return vseb<3, 3>(e);
}

// _tw_add: _fast.py:178-198.  The reference's two-pointer merge by magnitude
// (ties take the first operand; inputs need not be ordered), written as its
// state machine: after k steps the state (i, j), i+j = k, is one of at most
// four predicates, and each output word is a select among the heads that
// state can see -- no dynamic register indexing.
MWI V<3> tw_add(V<3> a, V<3> b) {
    const double a0 = a.w[0], a1 = a.w[1], a2 = a.w[2];
    const double b0 = b.w[0], b1 = b.w[1], b2 = b.w[2];
    // head comparisons c_ij = |a_i| >= |b_j|
    const bool c00 = mag_ge(a0, b0), c10 = mag_ge(a1, b0), c01 = mag_ge(a0, b1);
    const bool c20 = mag_ge(a2, b0), c11 = mag_ge(a1, b1), c02 = mag_ge(a0, b2);
    const bool c21 = mag_ge(a2, b1), c12 = mag_ge(a1, b2), c22 = mag_ge(a2, b2);
    double z[6];
    // step 0: state (0,0)
    z[0] = c00 ? a0 : b0;
    // step 1: state (1,0) if c00 else (0,1)
    const bool t1 = c00 ? c10 : c01;  // took from a at step 1
    z[1] = c00 ? (c10 ? a1 : b0) : (c01 ? a0 : b1);
    // step 2: states (2,0) (1,1) (0,2)
    const bool s20 = c00 && t1, s02 = !c00 && !t1, s11 = !s20 && !s02;
    const bool t2 = s20 ? c20 : (s11 ? c11 : c02);
    z[2] = s20 ? (c20 ? a2 : b0) : (s11 ? (c11 ? a1 : b1) : (c02 ? a0 : b2));
    // step 3: states (3,0) (2,1) (1,2) (0,3)
    const bool s30 = s20 && t2, s21 = (s20 && !t2) || (s11 && t2);
    const bool s03 = s02 && !t2, s12 = !s30 && !s21 && !s03;
    const bool t3 = s30 ? false : (s21 ? c21 : (s12 ? c12 : true));
    z[3] = s30 ? b0 : (s21 ? (c21 ? a2 : b1) : (s12 ? (c12 ? a1 : b2) : a0));
    // step 4: states (3,1) (2,2) (1,3)
    const bool s31 = s30 || (s21 && t3), s13 = s03 || (s12 && !t3), s22 = !s31 && !s13;
    const bool t4 = s31 ? false : (s22 ? c22 : true);
    z[4] = s31 ? b1 : (s22 ? (c22 ? a2 : b2) : a1);
    // step 5: states (3,2) (2,3)
    const bool s32 = s31 || (s22 && t4);
    z[5] = s32 ? b2 : a2;
    double e[6];
    vec_sum<6>(z, e);
    return vseb<6, 3>(e);
}
// _qtw_add: _fast.py:201-207
MWI V<3> qtw_add(V<3> a, V<3> b) {
    double c0, e1, c1, e2, e3;
    two_sum(a.w[0], b.w[0], c0, e1);
    two_sum(a.w[1], b.w[1], c1, e2);
    two_sum(c1, e1, c1, e3);
    double c2 = __dadd_rn(__dadd_rn(__dadd_rn(a.w[2], b.w[2]), e2), e3);
    return V<3>{{c0, c1, c2}};
}
// _tw_mul: _fast.py:210-218
MWI V<3> tw_mul(V<3> a, V<3> b) {
    double c0, e1, t2, e2, t3, e3, c1, e4, e5;
    two_prod(a.w[0], b.w[0], c0, e1);
    two_prod(a.w[0], b.w[1], t2, e2);
    two_prod(a.w[1], b.w[0], t3, e3);
    two_sum(t2, t3, c1, e4);
    two_sum(c1, e1, c1, e5);
    double c2 = __dadd_rn(
        __fma_rn(a.w[1], b.w[1], __dadd_rn(__fma_rn(a.w[2], b.w[0], e2), __fma_rn(a.w[0], b.w[2], e3))),
        __dadd_rn(e4, e5));
    return renorm3(c0, c1, c2);
}
// _qtw_mul: _fast.py:221-229
MWI V<3> qtw_mul(V<3> a, V<3> b) {
    double c0, e1, t2, e2, t3, e3, c1, e4, e5;
    two_prod(a.w[0], b.w[0], c0, e1);
    two_prod(a.w[0], b.w[1], t2, e2);
    two_prod(a.w[1], b.w[0], t3, e3);
    two_sum(t2, t3, c1, e4);
    two_sum(c1, e1, c1, e5);
    double c2 = __dadd_rn(
        __dadd_rn(__dadd_rn(__fma_rn(a.w[2], b.w[0], e2), __fma_rn(a.w[1], b.w[1], e3)),
                  __fma_rn(a.w[0], b.w[2], e4)),
        e5);
    return V<3>{{c0, c1, c2}};
}
// _dxqtw_mul: _fast.py:232-238
MWI V<3> dxqtw_mul(double a, V<3> b) {
    double c0, e1, c1, e2, e5;
    two_prod(a, b.w[0], c0, e1);
    two_prod(a, b.w[1], c1, e2);
    two_sum(c1, e1, c1, e5);
    return V<3>{{c0, c1, __dadd_rn(__fma_rn(a, b.w[2], e2), e5)}};
}
// _dxtw_mul: _fast.py:241-247
MWI V<3> dxtw_mul(double a, V<3> b) {
    double c0, e1, c1, e2, e5;
    two_prod(a, b.w[0], c0, e1);
    two_prod(a, b.w[1], c1, e2);
    two_sum(c1, e1, c1, e5);
    return renorm3(c0, c1, __dadd_rn(__fma_rn(a, b.w[2], e2), e5));
}
// _dxqtw_add: _fast.py:250-255
MWI V<3> dxqtw_add(double a, V<3> b) {
    double c0, e1, c1, e3;
    two_sum(a, b.w[0], c0, e1);
    two_sum(b.w[1], e1, c1, e3);
    return V<3>{{c0, c1, __dadd_rn(b.w[2], e3)}};
}
// _dxtw_add: _fast.py:258-277.  The single FP64 word is inserted before the
// first b_j it is >= in magnitude (the two-pointer merge with one element).
MWI V<3> dxtw_add(double a, V<3> b) {
    bool g0 = mag_ge(a, b.w[0]);
    bool g1 = mag_ge(a, b.w[1]);
    bool g2 = mag_ge(a, b.w[2]);
    double z[4];
    // position of a: 0 if g0, 1 if g1, 2 if g2, else 3
    z[0] = g0 ? a : b.w[0];
    z[1] = g0 ? b.w[0] : (g1 ? a : b.w[1]);
    z[2] = (g0 || g1) ? b.w[1] : (g2 ? a : b.w[2]);
    z[3] = (g0 || g1 || g2) ? b.w[2] : a;
    double e[4];
    vec_sum<4>(z, e);
    return vseb<4, 3>(e);
}

// ------------------------------------------------------------ division
// Division runs once per dot product, on one thread, in the serial tail of a
// kernel (the scalar step of K1 / K2): what matters there is the size of the
// straight-line code, not its instruction count -- cold instruction fetches of
// a fully inlined tw_div (4 x (dxtw_mul + tw_add) = ~1500 instructions executed
// once) cost more than the arithmetic.  tw_div's loop is therefore kept rolled
// and the TW operations it calls are single out-of-line copies.
#define MWNI static __device__ __noinline__
MWNI V<3> tw_add_ni(V<3> a, V<3> b) { return tw_add(a, b); }
MWNI V<3> dxtw_mul_ni(double a, V<3> b) { return dxtw_mul(a, b); }

// dw_div: multiword.py:370-382 (normalized ops, also used for QDW 408)
MWI V<2> dw_div(V<2> a, V<2> b) {
    V<2> bn = norm_dw(b);
    double bc = __dadd_rn(bn.w[0], bn.w[1]);
    if (bc == 0.0) return V<2>{{__ddiv_rn(__dadd_rn(a.w[0], a.w[1]), bc), 0.0}};
    V<2> r = a;
    double q[3];
#pragma unroll
    for (int i = 0; i < 3; i++) {
        q[i] = __ddiv_rn(r.w[0], bn.w[0]);
        V<2> t = dxdw_mul(q[i], bn);
        r = dw_add(r, V<2>{{-t.w[0], -t.w[1]}});
    }
    double e[3];
    vec_sum<3>(q, e);
    V<3> c = vseb<3, 2>(e);
    return V<2>{{c.w[0], c.w[1]}};
}
// tw_div: multiword.py:385-397, _strict_normalize_tw 400-402.  COMPACT (TW): the
// rolled loop over out-of-line copies; QTW keeps the inlined form (its tail is
// short enough to stay resident: compact costs it 1.5-3 us/it).
template <bool COMPACT>
MWI V<3> tw_div_t(V<3> a, V<3> b) {
    double bz[3] = {b.w[0], b.w[1], b.w[2]}, be[3];
    vec_sum<3>(bz, be);
    V<3> bn = vseb<3, 3>(be);
    double bc = __dadd_rn(__dadd_rn(bn.w[0], bn.w[1]), bn.w[2]);
    if (bc == 0.0)
        return V<3>{{__ddiv_rn(__dadd_rn(__dadd_rn(a.w[0], a.w[1]), a.w[2]), bc), 0.0, 0.0}};
    V<3> r = a;
    double q[4];
    if constexpr (COMPACT) {
#pragma unroll 1
        for (int i = 0; i < 4; i++) {
            q[i] = __ddiv_rn(r.w[0], bn.w[0]);
            V<3> t = dxtw_mul_ni(q[i], bn);
            r = tw_add_ni(r, V<3>{{-t.w[0], -t.w[1], -t.w[2]}});
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            q[i] = __ddiv_rn(r.w[0], bn.w[0]);
            V<3> t = dxtw_mul(q[i], bn);
            r = tw_add(r, V<3>{{-t.w[0], -t.w[1], -t.w[2]}});
        }
    }
    double e[4];
    vec_sum<4>(q, e);
    return vseb<4, 3>(e);
}
MWI V<3> tw_div(V<3> a, V<3> b) { return tw_div_t<false>(a, b); }

// ------------------------------------------------------------ mode traits
template <int M>
struct Arith;

template <>
struct Arith<FP64> {
    static constexpr int W = 1;
    using T = V<1>;
    static MWI T add(T a, T b) { return T{{__dadd_rn(a.w[0], b.w[0])}}; }
    static MWI T mul(T a, T b) { return T{{__dmul_rn(a.w[0], b.w[0])}}; }
    static MWI T dxmul(double a, T b) { return T{{__dmul_rn(a, b.w[0])}}; }
    static MWI T dxadd(double a, T b) { return T{{__dadd_rn(a, b.w[0])}}; }
    static MWI T norm(T a) { return a; }
    static MWI T div(T a, T b) { return T{{__ddiv_rn(a.w[0], b.w[0])}}; }
    static MWI double collapse(T a) { return a.w[0]; }
};
template <>
struct Arith<DW> {
    static constexpr int W = 2;
    using T = V<2>;
    static MWI T add(T a, T b) { return dw_add(a, b); }
    static MWI T mul(T a, T b) { return dw_mul(a, b); }
    static MWI T dxmul(double a, T b) { return dxdw_mul(a, b); }
    static MWI T dxadd(double a, T b) { return dxdw_add(a, b); }
    static MWI T norm(T a) { return a; }
    static MWI T div(T a, T b) { return dw_div(a, b); }
    static MWI double collapse(T a) { return __dadd_rn(a.w[0], a.w[1]); }
};
template <>
struct Arith<QDW> {
    static constexpr int W = 2;
    using T = V<2>;
    static MWI T add(T a, T b) { return qdw_add(a, b); }
    static MWI T mul(T a, T b) { return qdw_mul(a, b); }
    static MWI T dxmul(double a, T b) { return dxqdw_mul(a, b); }
    static MWI T dxadd(double a, T b) { return dxqdw_add(a, b); }
    static MWI T norm(T a) { return norm_dw(a); }
    static MWI T div(T a, T b) { return dw_div(a, b); }
    static MWI double collapse(T a) { return __dadd_rn(a.w[0], a.w[1]); }
};
template <>
struct Arith<TW> {
    static constexpr int W = 3;
    using T = V<3>;
    static MWI T add(T a, T b) { return tw_add(a, b); }
    static MWI T mul(T a, T b) { return tw_mul(a, b); }
    static MWI T dxmul(double a, T b) { return dxtw_mul(a, b); }
    static MWI T dxadd(double a, T b) { return dxtw_add(a, b); }
    static MWI T norm(T a) { return a; }
    static MWI T div(T a, T b) { return tw_div_t<true>(a, b); }
    static MWI double collapse(T a) { return __dadd_rn(__dadd_rn(a.w[0], a.w[1]), a.w[2]); }
};
template <>
struct Arith<QTW> {
    static constexpr int W = 3;
    using T = V<3>;
    static MWI T add(T a, T b) { return qtw_add(a, b); }
    static MWI T mul(T a, T b) { return qtw_mul(a, b); }
    static MWI T dxmul(double a, T b) { return dxqtw_mul(a, b); }
    static MWI T dxadd(double a, T b) { return dxqtw_add(a, b); }
    static MWI T norm(T a) { return vecsum3(a); }
    static MWI T div(T a, T b) { return tw_div(a, b); }
    static MWI double collapse(T a) { return __dadd_rn(__dadd_rn(a.w[0], a.w[1]), a.w[2]); }
};

// One out-of-line copy of a mode's addition, for code that runs once per
// kernel (the last-CTA reduction of the tile partials): see "division" above.
template <int M>
__device__ __noinline__ V<Arith<M>::W> add_cold(V<Arith<M>::W> a, V<Arith<M>::W> b) {
    return Arith<M>::add(a, b);
}

template <int W>
MWI V<W> zero() {
    V<W> r;
#pragma unroll
    for (int k = 0; k < W; k++) r.w[k] = 0.0;
    return r;
}
template <int W>
MWI V<W> neg(V<W> a) {
    V<W> r;
#pragma unroll
    for (int k = 0; k < W; k++) r.w[k] = -a.w[k];
    return r;
}

// SoA word-plane access: word k of element i at v[k*ld + i]
template <int W>
MWI V<W> load(const double *__restrict__ v, int64_t ld, int64_t i) {
    V<W> r;
#pragma unroll
    for (int k = 0; k < W; k++) r.w[k] = v[k * ld + i];
    return r;
}
template <int W>
MWI V<W> load_ro(const double *__restrict__ v, int64_t ld, int64_t i) {
    V<W> r;
#pragma unroll
    for (int k = 0; k < W; k++) r.w[k] = __ldg(v + k * ld + i);
    return r;
}
template <int W>
MWI void store(double *__restrict__ v, int64_t ld, int64_t i, V<W> a) {
#pragma unroll
    for (int k = 0; k < W; k++) v[k * ld + i] = a.w[k];
}
// Interleaved (AoS) records: word k of element i at v[i*W + k].  The solver
// stores the search direction p this way: a gather of p[c] is one 8/16/24-B
// record instead of W loads in W different word planes (sectors).
template <int W>
MWI V<W> load_aos(const double *__restrict__ v, int64_t i) {
    V<W> r;
    if (W == 2) {
        const double2 t = *reinterpret_cast<const double2 *>(v + 2 * i);
        r.w[0] = t.x;
        r.w[W - 1] = t.y;
    } else {
#pragma unroll
        for (int k = 0; k < W; k++) r.w[k] = v[i * W + k];
    }
    return r;
}
template <int W>
MWI V<W> load_aos_ro(const double *__restrict__ v, int64_t i) {
    V<W> r;
    if (W == 2) {
        const double2 t = __ldg(reinterpret_cast<const double2 *>(v + 2 * i));
        r.w[0] = t.x;
        r.w[W - 1] = t.y;
    } else {
#pragma unroll
        for (int k = 0; k < W; k++) r.w[k] = __ldg(v + i * W + k);
    }
    return r;
}
template <int W>
MWI void store_aos(double *__restrict__ v, int64_t i, V<W> a) {
    if (W == 2) {
        *reinterpret_cast<double2 *>(v + 2 * i) = make_double2(a.w[0], a.w[W - 1]);
    } else {
#pragma unroll
        for (int k = 0; k < W; k++) v[i * W + k] = a.w[k];
    }
}

template <int W>
MWI V<W> shfl_down(V<W> a, int off) {
    V<W> r;
#pragma unroll
    for (int k = 0; k < W; k++) r.w[k] = __shfl_down_sync(0xffffffffu, a.w[k], off);
    return r;
}

}  // namespace mw
