/*
 * mwcg_oracle.c -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain-C restatement of the reference package `mwcg` hot path:
 *   EFTs            /root/reference/pkg/src/mwcg/_fast.py:41-60   (eft.py:78-122)
 *   DW/QDW ops      _fast.py:63-126                              (multiword.py:101-168)
 *   TW/QTW ops      _fast.py:129-277                             (multiword.py:175-323)
 *   division        multiword.py:360-409
 *   kernels         _fast.py:284-589, dispatch kernels.py:174-296
 *   norm metrics    kernels.py:299-328
 *   CG loop         cg.py:78-183
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load this library, and only as the checker / the
 * CPU baseline.  The product (paper_2510_13536_b200) never links it.
 *
 * Parity is pinned by tests/golden/ (vectors produced by the real reference,
 * imported in the build container; see tests/golden/make_golden.py).
 *
 * Two reduction shapes are provided for every dot product:
 *   partitions P  : the reference's own shape (kernels.py:158-162,
 *                   _fast.py:342-356): P sequential partitions with bounds
 *                   floor(n*p/P), combined left-to-right.  P=1 is the
 *                   sequential specification.
 *   tile tree     : the canonical GPU shape of this repo (DESIGN.md
 *                   "Reduction order").  Tiles of TB*E elements; thread t of
 *                   a tile accumulates elements tile*T + j*TB + t (j=0..E-1),
 *                   then a 32-lane tree (lane i += lane i+off, off=16..1),
 *                   then a tree over the TB/32 warp results, giving one
 *                   partial per tile; the partials are reduced by the same
 *                   procedure with E' = ceil(ntiles/TB).
 *
 * Build: gcc -O3 -ffp-contract=off -fopenmp -shared -fPIC (see Makefile).
 * -ffp-contract=off is REQUIRED: the reference kernels are unfused
 * (numba does not contract), and TwoProd's x=a*b must not fuse into later
 * additions.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#if defined(__FP_FAST_FMA) && 0
#endif

enum { M_FP64 = 0, M_DW = 1, M_QDW = 2, M_TW = 3, M_QTW = 4 };
enum { NORM_NONE = 0, NORM_AFTER_AXPY = 1, NORM_EVERY_OP = 2 };
enum { REASON_CONVERGED = 1, REASON_MAX_ITERS = 2, REASON_BREAKDOWN = 3 };

static const int WORDS[5] = {1, 2, 2, 3, 3};

typedef struct { double v[3]; } mw;

/* ------------------------------------------------------------------ EFTs */
/* _fast.py:41-60 */
static inline void two_sum(double a, double b, double *x, double *y) {
    double s = a + b;
    double z = s - a;
    *y = (a - (s - z)) + (b - z);
    *x = s;
}
static inline void quick_two_sum(double a, double b, double *x, double *y) {
    double s = a + b;
    *y = (a - s) + b;
    *x = s;
}
static inline void two_prod(double a, double b, double *x, double *y) {
    double p = a * b;
    *y = fma(a, b, -p);
    *x = p;
}

/* ---------------------------------------------------------- DW / QDW ops */
/* _fast.py:63-126 */
static inline mw dw_add(mw a, mw b) {
    double s, e; mw r;
    two_sum(a.v[0], b.v[0], &s, &e);
    e = (e + a.v[1]) + b.v[1];
    quick_two_sum(s, e, &r.v[0], &r.v[1]);
    r.v[2] = 0.0;
    return r;
}
static inline mw qdw_add(mw a, mw b) {
    double s, e; mw r;
    two_sum(a.v[0], b.v[0], &s, &e);
    e = (e + a.v[1]) + b.v[1];
    r.v[0] = s; r.v[1] = e; r.v[2] = 0.0;
    return r;
}
static inline mw dw_mul(mw a, mw b) {
    double p, e; mw r;
    two_prod(a.v[0], b.v[0], &p, &e);
    e = fma(a.v[0], b.v[1], e);
    e = fma(a.v[1], b.v[0], e);
    quick_two_sum(p, e, &r.v[0], &r.v[1]);
    r.v[2] = 0.0;
    return r;
}
static inline mw qdw_mul(mw a, mw b) {
    double p, e; mw r;
    two_prod(a.v[0], b.v[0], &p, &e);
    e = fma(a.v[0], b.v[1], e);
    e = fma(a.v[1], b.v[0], e);
    r.v[0] = p; r.v[1] = e; r.v[2] = 0.0;
    return r;
}
static inline mw dxdw_mul(double a, mw b) {
    double p, e; mw r;
    two_prod(a, b.v[0], &p, &e);
    e = fma(a, b.v[1], e);
    quick_two_sum(p, e, &r.v[0], &r.v[1]);
    r.v[2] = 0.0;
    return r;
}
static inline mw dxqdw_mul(double a, mw b) {
    double p, e; mw r;
    two_prod(a, b.v[0], &p, &e);
    e = fma(a, b.v[1], e);
    r.v[0] = p; r.v[1] = e; r.v[2] = 0.0;
    return r;
}
static inline mw dxdw_add(double a, mw b) {
    double s, e; mw r;
    two_sum(a, b.v[0], &s, &e);
    e = e + b.v[1];
    quick_two_sum(s, e, &r.v[0], &r.v[1]);
    r.v[2] = 0.0;
    return r;
}
static inline mw dxqdw_add(double a, mw b) {
    double s, e; mw r;
    two_sum(a, b.v[0], &s, &e);
    e = e + b.v[1];
    r.v[0] = s; r.v[1] = e; r.v[2] = 0.0;
    return r;
}
static inline mw norm_dw(mw a) {
    mw r; r.v[2] = 0.0;
    if (fabs(a.v[0]) >= fabs(a.v[1])) quick_two_sum(a.v[0], a.v[1], &r.v[0], &r.v[1]);
    else two_sum(a.v[0], a.v[1], &r.v[0], &r.v[1]);
    return r;
}

/* ---------------------------------------------------------- TW / QTW ops */
/* _vseb3: _fast.py:136-163 (multiword.py:187-203 with m=3) */
static inline mw vseb(const double *e, int n, int m) {
    double r[3] = {0.0, 0.0, 0.0};
    int j = 0;
    double eps = e[0];
    for (int i = 0; i < n - 1; i++) {
        double rj, en;
        two_sum(eps, e[i + 1], &rj, &en);
        if (en != 0.0) {
            r[j] = rj;
            if (j == m - 1) { mw o = {{r[0], r[1], r[2]}}; return o; }
            j++;
            eps = en;
        } else {
            eps = rj;
        }
    }
    r[j] = eps;
    mw o = {{r[0], r[1], r[2]}};
    return o;
}
/* _vec_sum: multiword.py:175-184 */
static inline void vec_sum(const double *z, int n, double *e) {
    double s = z[n - 1];
    for (int k = n - 2; k >= 0; k--) {
        double err;
        two_sum(z[k], s, &s, &err);
        e[k + 1] = err;
    }
    e[0] = s;
}
/* _vecsum3: _fast.py:129-133 */
static inline mw vecsum3(mw a) {
    mw r;
    double c1;
    two_sum(a.v[0], a.v[1], &r.v[0], &c1);
    two_sum(c1, a.v[2], &r.v[1], &r.v[2]);
    return r;
}
/* _renorm3: _fast.py:166-175 */
static inline mw renorm3(double c0, double c1, double c2) {
    double z[3] = {c0, c1, c2}, e[3];
    vec_sum(z, 3, e);
    return vseb(e, 3, 3);
}
/* _tw_add: _fast.py:178-198 -- stable merge by |.| (ties: first operand) */
static inline mw tw_add(mw a, mw b) {
    double z[6], e[6];
    int i = 0, j = 0;
    for (int k = 0; k < 6; k++) {
        if (i < 3 && (j >= 3 || fabs(a.v[i]) >= fabs(b.v[j]))) z[k] = a.v[i++];
        else z[k] = b.v[j++];
    }
    vec_sum(z, 6, e);
    return vseb(e, 6, 3);
}
/* _qtw_add: _fast.py:201-207 */
static inline mw qtw_add(mw a, mw b) {
    double c0, e1, c1, e2, e3; mw r;
    two_sum(a.v[0], b.v[0], &c0, &e1);
    two_sum(a.v[1], b.v[1], &c1, &e2);
    two_sum(c1, e1, &c1, &e3);
    r.v[0] = c0; r.v[1] = c1;
    r.v[2] = ((a.v[2] + b.v[2]) + e2) + e3;
    return r;
}
/* _tw_mul: _fast.py:210-218 */
static inline mw tw_mul(mw a, mw b) {
    double c0, e1, t2, e2, t3, e3, c1, e4, e5;
    two_prod(a.v[0], b.v[0], &c0, &e1);
    two_prod(a.v[0], b.v[1], &t2, &e2);
    two_prod(a.v[1], b.v[0], &t3, &e3);
    two_sum(t2, t3, &c1, &e4);
    two_sum(c1, e1, &c1, &e5);
    double c2 = fma(a.v[1], b.v[1], fma(a.v[2], b.v[0], e2) + fma(a.v[0], b.v[2], e3)) + (e4 + e5);
    return renorm3(c0, c1, c2);
}
/* _qtw_mul: _fast.py:221-229 */
static inline mw qtw_mul(mw a, mw b) {
    double c0, e1, t2, e2, t3, e3, c1, e4, e5; mw r;
    two_prod(a.v[0], b.v[0], &c0, &e1);
    two_prod(a.v[0], b.v[1], &t2, &e2);
    two_prod(a.v[1], b.v[0], &t3, &e3);
    two_sum(t2, t3, &c1, &e4);
    two_sum(c1, e1, &c1, &e5);
    r.v[0] = c0; r.v[1] = c1;
    r.v[2] = ((fma(a.v[2], b.v[0], e2) + fma(a.v[1], b.v[1], e3)) + fma(a.v[0], b.v[2], e4)) + e5;
    return r;
}
/* _dxqtw_mul: _fast.py:232-238 */
static inline mw dxqtw_mul(double a, mw b) {
    double c0, e1, c1, e2, e5; mw r;
    two_prod(a, b.v[0], &c0, &e1);
    two_prod(a, b.v[1], &c1, &e2);
    two_sum(c1, e1, &c1, &e5);
    r.v[0] = c0; r.v[1] = c1; r.v[2] = fma(a, b.v[2], e2) + e5;
    return r;
}
/* _dxtw_mul: _fast.py:241-247 */
static inline mw dxtw_mul(double a, mw b) {
    double c0, e1, c1, e2, e5;
    two_prod(a, b.v[0], &c0, &e1);
    two_prod(a, b.v[1], &c1, &e2);
    two_sum(c1, e1, &c1, &e5);
    return renorm3(c0, c1, fma(a, b.v[2], e2) + e5);
}
/* _dxqtw_add: _fast.py:250-255 */
static inline mw dxqtw_add(double a, mw b) {
    double c0, e1, c1, e3; mw r;
    two_sum(a, b.v[0], &c0, &e1);
    two_sum(b.v[1], e1, &c1, &e3);
    r.v[0] = c0; r.v[1] = c1; r.v[2] = b.v[2] + e3;
    return r;
}
/* _dxtw_add: _fast.py:258-277 */
static inline mw dxtw_add(double a, mw b) {
    double z[4], e[4];
    int i = 0, j = 0;
    for (int k = 0; k < 4; k++) {
        if (i < 1 && (j >= 3 || fabs(a) >= fabs(b.v[j]))) { z[k] = a; i++; }
        else z[k] = b.v[j++];
    }
    vec_sum(z, 4, e);
    return vseb(e, 4, 3);
}

/* ------------------------------------------------------ mode dispatch */
static inline mw op_add(int m, mw a, mw b) {
    switch (m) {
    case M_FP64: { mw r = {{a.v[0] + b.v[0], 0.0, 0.0}}; return r; }
    case M_DW: return dw_add(a, b);
    case M_QDW: return qdw_add(a, b);
    case M_TW: return tw_add(a, b);
    default: return qtw_add(a, b);
    }
}
static inline mw op_mul(int m, mw a, mw b) {
    switch (m) {
    case M_FP64: { mw r = {{a.v[0] * b.v[0], 0.0, 0.0}}; return r; }
    case M_DW: return dw_mul(a, b);
    case M_QDW: return qdw_mul(a, b);
    case M_TW: return tw_mul(a, b);
    default: return qtw_mul(a, b);
    }
}
static inline mw op_dxmul(int m, double a, mw b) {
    switch (m) {
    case M_FP64: { mw r = {{a * b.v[0], 0.0, 0.0}}; return r; }
    case M_DW: return dxdw_mul(a, b);
    case M_QDW: return dxqdw_mul(a, b);
    case M_TW: return dxtw_mul(a, b);
    default: return dxqtw_mul(a, b);
    }
}
static inline mw op_dxadd(int m, double a, mw b) {
    switch (m) {
    case M_FP64: { mw r = {{a + b.v[0], 0.0, 0.0}}; return r; }
    case M_DW: return dxdw_add(a, b);
    case M_QDW: return dxqdw_add(a, b);
    case M_TW: return dxtw_add(a, b);
    default: return dxqtw_add(a, b);
    }
}
static inline mw op_norm(int m, mw a) {
    if (m == M_QDW) return norm_dw(a);
    if (m == M_QTW) return vecsum3(a);
    return a;
}
static inline mw op_neg(int m, mw a) {
    mw r = {{-a.v[0], -a.v[1], -a.v[2]}};
    if (WORDS[m] < 3) r.v[2] = 0.0;
    if (WORDS[m] < 2) r.v[1] = 0.0;
    return r;
}
static inline double op_collapse(int m, mw a) {
    /* scalar_to_fp64: kernels.py:139-142, multiword.py:88-94 */
    if (WORDS[m] == 1) return a.v[0];
    if (WORDS[m] == 2) return a.v[0] + a.v[1];
    return (a.v[0] + a.v[1]) + a.v[2];
}

/* _ieee_div: multiword.py:360-367 (C division already has IEEE semantics) */
static inline double ieee_div(double x, double y) { return x / y; }

/* dw_div: multiword.py:370-382 */
static mw dw_div(mw a, mw b) {
    mw bn = norm_dw(b);
    mw out = {{0.0, 0.0, 0.0}};
    if (bn.v[0] + bn.v[1] == 0.0) {
        out.v[0] = ieee_div(a.v[0] + a.v[1], bn.v[0] + bn.v[1]);
        return out;
    }
    mw r = a; r.v[2] = 0.0;
    double q[3], e[3];
    for (int i = 0; i < 3; i++) {
        q[i] = r.v[0] / bn.v[0];
        mw t = dxdw_mul(q[i], bn);
        t.v[0] = -t.v[0]; t.v[1] = -t.v[1];
        r = dw_add(r, t);
    }
    vec_sum(q, 3, e);
    return vseb(e, 3, 2);
}
/* tw_div: multiword.py:385-397 with _strict_normalize_tw 400-402 */
static mw tw_div(mw a, mw b) {
    double e3[3];
    vec_sum(b.v, 3, e3);
    mw bn = vseb(e3, 3, 3);
    mw out = {{0.0, 0.0, 0.0}};
    double bc = (bn.v[0] + bn.v[1]) + bn.v[2];
    if (bc == 0.0) {
        out.v[0] = ieee_div((a.v[0] + a.v[1]) + a.v[2], bc);
        return out;
    }
    mw r = a;
    double q[4], e[4];
    for (int i = 0; i < 4; i++) {
        q[i] = r.v[0] / bn.v[0];
        mw t = dxtw_mul(q[i], bn);
        t.v[0] = -t.v[0]; t.v[1] = -t.v[1]; t.v[2] = -t.v[2];
        r = tw_add(r, t);
    }
    vec_sum(q, 4, e);
    return vseb(e, 4, 3);
}
/* scalar_div: kernels.py:131-136 (qdw/qtw reuse the normalized divisions,
 * multiword.py:408-409) */
static inline mw op_div(int m, mw a, mw b) {
    if (m == M_FP64) { mw r = {{ieee_div(a.v[0], b.v[0]), 0.0, 0.0}}; return r; }
    if (WORDS[m] == 2) return dw_div(a, b);
    return tw_div(a, b);
}

/* ----------------------------------------------------------- vectors */
/* Vectors are SoA word planes: word k of element i at v[k*n + i]. */
static inline mw ld(const double *v, int64_t n, int w, int64_t i) {
    mw r = {{v[i], 0.0, 0.0}};
    if (w > 1) r.v[1] = v[n + i];
    if (w > 2) r.v[2] = v[2 * n + i];
    return r;
}
static inline void st(double *v, int64_t n, int w, int64_t i, mw a) {
    v[i] = a.v[0];
    if (w > 1) v[n + i] = a.v[1];
    if (w > 2) v[2 * n + i] = a.v[2];
}

static int g_threads = 1;

void orc_set_threads(int t) { g_threads = t < 1 ? 1 : t; }
int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Scalar op entry for the unit tests.
 * op: 0 add, 1 mul, 2 dxmul(a[0], b), 3 dxadd(a[0], b), 4 normalize(a),
 *     5 div, 6 neg, 7 two_sum, 8 quick_two_sum, 9 two_prod, 10 collapse */
void orc_scalar_op(int op, int mode, const double *a, const double *b, double *out) {
    mw A = {{a[0], a[1], a[2]}}, B = {{0, 0, 0}}, R = {{0, 0, 0}};
    if (b) { B.v[0] = b[0]; B.v[1] = b[1]; B.v[2] = b[2]; }
    switch (op) {
    case 0: R = op_add(mode, A, B); break;
    case 1: R = op_mul(mode, A, B); break;
    case 2: R = op_dxmul(mode, a[0], B); break;
    case 3: R = op_dxadd(mode, a[0], B); break;
    case 4: R = op_norm(mode, A); break;
    case 5: R = op_div(mode, A, B); break;
    case 6: R = op_neg(mode, A); break;
    case 7: two_sum(a[0], b[0], &R.v[0], &R.v[1]); break;
    case 8: quick_two_sum(a[0], b[0], &R.v[0], &R.v[1]); break;
    case 9: two_prod(a[0], b[0], &R.v[0], &R.v[1]); break;
    case 10: R.v[0] = op_collapse(mode, A); break;
    }
    out[0] = R.v[0]; out[1] = R.v[1]; out[2] = R.v[2];
}

/* spmv_<mode>: _fast.py:284-290, 329-339, 383-393, 443-455, 501-513 */
void orc_spmv(int mode, int64_t n_rows, const int64_t *rp, const int64_t *ci,
              const double *va, const double *x, int64_t nx, double *y) {
    int w = WORDS[mode];
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t i = 0; i < n_rows; i++) {
        mw s = {{0.0, 0.0, 0.0}};
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) {
            mw xv = ld(x, nx, w, ci[k]);
            s = op_add(mode, s, op_dxmul(mode, va[k], xv));
        }
        st(y, n_rows, w, i, s);
    }
}

/* dot_<mode> with partitions: _fast.py:293-304 etc.; bounds kernels.py:158-162 */
void orc_dot_partitions(int mode, int64_t n, const double *x, const double *y,
                        int64_t parts, double *out) {
    int w = WORDS[mode];
    mw *t = (mw *)malloc(sizeof(mw) * (size_t)parts);
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t p = 0; p < parts; p++) {
        /* n*p//P without overflow for the sizes used here */
        int64_t lo = (int64_t)(((__int128)n * p) / parts);
        int64_t hi = (int64_t)(((__int128)n * (p + 1)) / parts);
        mw acc = {{0.0, 0.0, 0.0}};
        for (int64_t i = lo; i < hi; i++)
            acc = op_add(mode, acc, op_mul(mode, ld(x, n, w, i), ld(y, n, w, i)));
        t[p] = acc;
    }
    mw s = t[0];
    for (int64_t p = 1; p < parts; p++) s = op_add(mode, s, t[p]);
    out[0] = s.v[0]; out[1] = s.v[1]; out[2] = s.v[2];
    free(t);
}

/* Canonical tile-tree combine of TB per-thread accumulators (see header). */
static mw tree_combine(int mode, mw *acc, int tb) {
    for (int base = 0; base < tb; base += 32) {
        for (int off = 16; off >= 1; off >>= 1)
            for (int l = 0; l < off; l++)
                acc[base + l] = op_add(mode, acc[base + l], acc[base + l + off]);
    }
    int nw = tb / 32;
    mw ws[64];
    for (int i = 0; i < nw; i++) ws[i] = acc[i * 32];
    for (int off = nw / 2; off >= 1; off >>= 1)
        for (int l = 0; l < off; l++) ws[l] = op_add(mode, ws[l], ws[l + off]);
    return ws[0];
}

/* Term for element i of the tile-tree dot: mul(x_i, y_i). */
static mw tile_tree_dot_impl(int mode, int64_t n, const double *x, const double *y,
                             int tb, int e) {
    int w = WORDS[mode];
    int64_t T = (int64_t)tb * e;
    int64_t ntiles = (n + T - 1) / T;
    if (ntiles == 0) { mw z = {{0, 0, 0}}; return z; }
    mw *part = (mw *)malloc(sizeof(mw) * (size_t)ntiles);
#pragma omp parallel num_threads(g_threads)
    {
        mw *acc = (mw *)malloc(sizeof(mw) * (size_t)tb);
#pragma omp for schedule(static)
        for (int64_t b = 0; b < ntiles; b++) {
            for (int t = 0; t < tb; t++) {
                mw a = {{0.0, 0.0, 0.0}};
                for (int j = 0; j < e; j++) {
                    int64_t i = b * T + (int64_t)j * tb + t;
                    if (i < n) a = op_add(mode, a, op_mul(mode, ld(x, n, w, i), ld(y, n, w, i)));
                }
                acc[t] = a;
            }
            part[b] = tree_combine(mode, acc, tb);
        }
        free(acc);
    }
    /* second pass over the tile partials */
    mw *acc = (mw *)malloc(sizeof(mw) * (size_t)tb);
    for (int t = 0; t < tb; t++) {
        mw a = {{0.0, 0.0, 0.0}};
        for (int64_t idx = t; idx < ntiles; idx += tb) a = op_add(mode, a, part[idx]);
        acc[t] = a;
    }
    mw r = tree_combine(mode, acc, tb);
    free(acc);
    free(part);
    return r;
}

/* Per-tile partials of the canonical tile tree (the first pass of
 * tile_tree_dot_impl) written SoA into out[k*ld + tile_off + b]. */
void orc_tile_partials(int mode, int64_t n, const double *x, int64_t ldx, const double *y,
                       int64_t ldy, int tb, int e, double *out, int64_t ldo, int64_t tile_off) {
    int w = WORDS[mode];
    int64_t T = (int64_t)tb * e;
    int64_t ntiles = (n + T - 1) / T;
    mw *acc = (mw *)malloc(sizeof(mw) * (size_t)tb);
    for (int64_t b = 0; b < ntiles; b++) {
        for (int t = 0; t < tb; t++) {
            mw a = {{0.0, 0.0, 0.0}};
            for (int j = 0; j < e; j++) {
                int64_t i = b * T + (int64_t)j * tb + t;
                if (i < n) a = op_add(mode, a, op_mul(mode, ld(x, ldx, w, i), ld(y, ldy, w, i)));
            }
            acc[t] = a;
        }
        mw r = tree_combine(mode, acc, tb);
        st(out + tile_off, ldo, w, b, r);
    }
    free(acc);
}

void orc_dot_tile(int mode, int64_t n, const double *x, const double *y, int tb, int e,
                  double *out) {
    mw r = tile_tree_dot_impl(mode, n, x, y, tb, e);
    out[0] = r.v[0]; out[1] = r.v[1]; out[2] = r.v[2];
}

/* Reduce pre-computed tile partials (w-word, SoA over ntiles) with the
 * canonical second pass; used to check the device's partial arrays. */
void orc_reduce_partials(int mode, int64_t ntiles, const double *part_soa, int tb, double *out) {
    int w = WORDS[mode];
    mw *acc = (mw *)malloc(sizeof(mw) * (size_t)tb);
    for (int t = 0; t < tb; t++) {
        mw a = {{0.0, 0.0, 0.0}};
        for (int64_t idx = t; idx < ntiles; idx += tb) a = op_add(mode, a, ld(part_soa, ntiles, w, idx));
        acc[t] = a;
    }
    mw r = tree_combine(mode, acc, tb);
    free(acc);
    out[0] = r.v[0]; out[1] = r.v[1]; out[2] = r.v[2];
}

/* axpy_<mode>: y <- add(y, mul(alpha, x)) _fast.py:307-310, 359-363, ... */
void orc_axpy(int mode, int64_t n, const double *alpha, const double *x, double *y) {
    int w = WORDS[mode];
    mw a = {{alpha[0], w > 1 ? alpha[1] : 0.0, w > 2 ? alpha[2] : 0.0}};
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t i = 0; i < n; i++)
        st(y, n, w, i, op_add(mode, ld(y, n, w, i), op_mul(mode, a, ld(x, n, w, i))));
}

/* scal_add_<mode>: p <- add(r, mul(beta, p)) _fast.py:313-316, 366-370, ... */
void orc_scal_add(int mode, int64_t n, const double *beta, double *p, const double *r) {
    int w = WORDS[mode];
    mw b = {{beta[0], w > 1 ? beta[1] : 0.0, w > 2 ? beta[2] : 0.0}};
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t i = 0; i < n; i++)
        st(p, n, w, i, op_add(mode, ld(r, n, w, i), op_mul(mode, b, ld(p, n, w, i))));
}

/* residual_<mode>: r = dxadd(b, -q) _fast.py:319-322, 373-376, ... */
void orc_residual(int mode, int64_t n, const double *bvec, const double *q, double *r) {
    int w = WORDS[mode];
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t i = 0; i < n; i++) {
        mw qi = op_neg(mode, ld(q, n, w, i));
        st(r, n, w, i, op_dxadd(mode, bvec[i], qi));
    }
}

/* normalize_arr_q{dw,tw}: _fast.py:433-436, 555-558 */
void orc_normalize(int mode, int64_t n, double *v) {
    int w = WORDS[mode];
    if (mode != M_QDW && mode != M_QTW) return;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t i = 0; i < n; i++) st(v, n, w, i, op_norm(mode, ld(v, n, w, i)));
}

/* sumsq_collapsed_{1,2,3}: _fast.py:565-589 (sequential, unfused) */
double orc_sumsq(int words, int64_t n, const double *v) {
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double c = v[i];
        if (words == 2) c = v[i] + v[n + i];
        else if (words == 3) c = (v[i] + v[n + i]) + v[2 * n + i];
        s = s + c * c;
    }
    return s;
}

/* ------------------------------------------------------------ metrics */
typedef struct {
    int reduction;   /* 0 = partitions (metrics always use P=1), 1 = tile tree */
    int tb, e;
} red_t;

static double tw_norm_sq(const red_t *rd, int64_t n, const double *v3) {
    /* _tw_norm_sq: kernels.py:299-302 -- dot(v, v) with partitions=1 */
    double out[3];
    if (rd->reduction == 1) orc_dot_tile(M_TW, n, v3, v3, rd->tb, rd->e, out);
    else orc_dot_partitions(M_TW, n, v3, v3, 1, out);
    return (out[0] + out[1]) + out[2];
}

/* norm_metrics_tw: kernels.py:305-328.  x is in `mode` (promoted to TW). */
static void norm_metrics(const red_t *rd, int mode, int64_t n, const int64_t *rp,
                         const int64_t *ci, const double *va, const double *x,
                         const double *x_star, const double *b, double *err,
                         double *true_res, double *ws /* 9n doubles */) {
    int w = WORDS[mode];
    double *xt = ws, *q = ws + 3 * n, *res = ws + 6 * n;
    memset(xt, 0, sizeof(double) * 3 * (size_t)n);
    memcpy(xt, x, sizeof(double) * (size_t)(w * n));  /* promote_tw kernels.py:107-112 */
    orc_spmv(M_TW, n, rp, ci, va, xt, n, q);
    orc_residual(M_TW, n, b, q, res);
    /* bt = from_fp64(b, tw) */
    double *bt = q;  /* q no longer needed */
    memset(bt, 0, sizeof(double) * 3 * (size_t)n);
    memcpy(bt, b, sizeof(double) * (size_t)n);
    double bn = tw_norm_sq(rd, n, bt);
    if (bn == 0.0) bn = 1.0;
    *true_res = sqrt(tw_norm_sq(rd, n, res) / bn);
    if (x_star) {
        orc_residual(M_TW, n, x_star, xt, res);  /* diff = x* - x */
        memset(bt, 0, sizeof(double) * 3 * (size_t)n);
        memcpy(bt, x_star, sizeof(double) * (size_t)n);
        double xs = tw_norm_sq(rd, n, bt);
        if (xs == 0.0) xs = 1.0;
        *err = sqrt(tw_norm_sq(rd, n, res) / xs);
    } else {
        *err = NAN;
    }
}

void orc_norm_metrics_tw(int mode, int reduction, int tb, int e, int64_t n, const int64_t *rp,
                         const int64_t *ci, const double *va, const double *x,
                         const double *x_star, const double *b, double *err_out,
                         double *true_res_out) {
    red_t rd = {reduction, tb, e};
    double *ws = (double *)malloc(sizeof(double) * 9 * (size_t)(n > 0 ? n : 1));
    norm_metrics(&rd, mode, n, rp, ci, va, x, x_star, b, err_out, true_res_out, ws);
    free(ws);
}

/* ------------------------------------------------------------ CG solve */
typedef struct {
    int mode;
    int normalization;
    int reduction;        /* 0 = partitions, 1 = tile tree */
    int tb, e;            /* tile-tree shape */
    int record_history;   /* 0: skip metrics (faster); records still counted */
    double epsilon;
    int64_t max_iterations;
    int64_t history_stride;
    int64_t partitions;
} orc_cfg;

typedef struct {
    int64_t iterations;
    int reason;
    double final_rel;
    int64_t n_hist;
} orc_result;

static void dot_cfg(const orc_cfg *c, int64_t n, const double *x, const double *y, mw *o) {
    double out[3];
    if (c->reduction == 1) orc_dot_tile(c->mode, n, x, y, c->tb, c->e, out);
    else orc_dot_partitions(c->mode, n, x, y, c->partitions, out);
    o->v[0] = out[0]; o->v[1] = out[1]; o->v[2] = out[2];
}

/* cg_solve: cg.py:78-183.  x (w*n) receives the solution words.
 * Histories are written up to hist_cap entries. */
int orc_cg_solve(const orc_cfg *c, int64_t n, const int64_t *rp, const int64_t *ci,
                 const double *va, const double *b, const double *x0, const double *x_star,
                 double *x, int64_t hist_cap, int64_t *h_k, double *h_rel, double *h_true,
                 double *h_err, orc_result *res) {
    int mode = c->mode, w = WORDS[mode];
    int quasi = (mode == M_QDW || mode == M_QTW);
    int norm_r = quasi && c->normalization != NORM_NONE;
    int norm_all = quasi && c->normalization == NORM_EVERY_OP;
    int64_t max_iters = c->max_iterations;
    red_t rd = {c->reduction, c->tb, c->e};
    size_t sz = sizeof(double) * (size_t)w * (size_t)(n > 0 ? n : 1);
    double *q = (double *)calloc(1, sz), *r = (double *)calloc(1, sz), *p = (double *)calloc(1, sz);
    double *ws = (double *)malloc(sizeof(double) * 9 * (size_t)(n > 0 ? n : 1));
    memset(x, 0, sizeof(double) * (size_t)w * (size_t)n);
    if (x0) memcpy(x, x0, sizeof(double) * (size_t)n);

    orc_spmv(mode, n, rp, ci, va, x, n, q);
    orc_residual(mode, n, b, q, r);
    if (norm_r) orc_normalize(mode, n, r);
    memcpy(p, r, sz);
    mw rho; dot_cfg(c, n, r, r, &rho);
    double b_norm = sqrt(orc_sumsq(1, n, b));
    if (b_norm == 0.0) b_norm = 1.0;
#define REL(S) (sqrt(fabs(op_collapse(mode, (S)))) / b_norm)
    int64_t nh = 0;
#define RECORD(K, RELV) do { \
        if (nh < hist_cap) { \
            double e_ = NAN, t_ = NAN; \
            if (c->record_history) \
                norm_metrics(&rd, mode, n, rp, ci, va, x, x_star, b, &e_, &t_, ws); \
            h_k[nh] = (K); h_rel[nh] = (RELV); h_true[nh] = t_; h_err[nh] = e_; \
        } \
        nh++; \
    } while (0)
    int64_t last_rec = -1;
    double rel = REL(rho);
    RECORD(0, rel); last_rec = 0;
    int reason = 0; int64_t kk = 0;
    if (rel < c->epsilon) { reason = REASON_CONVERGED; kk = 0; goto done; }
    for (int64_t k = 1; k <= max_iters; k++) {
        orc_spmv(mode, n, rp, ci, va, p, n, q);
        if (norm_all) orc_normalize(mode, n, q);
        mw pq; dot_cfg(c, n, p, q, &pq);
        double pq_f = op_collapse(mode, pq);
        if (pq_f == 0.0 || !isfinite(pq_f)) { reason = REASON_BREAKDOWN; kk = k - 1; goto done; }
        mw alpha = op_div(mode, rho, pq);
        orc_axpy(mode, n, alpha.v, p, x);
        if (norm_all) orc_normalize(mode, n, x);
        mw na = op_neg(mode, alpha);
        orc_axpy(mode, n, na.v, q, r);
        if (norm_r) orc_normalize(mode, n, r);
        mw rho_new; dot_cfg(c, n, r, r, &rho_new);
        rel = REL(rho_new);
        if (k % c->history_stride == 0) { RECORD(k, rel); last_rec = k; }
        if (rel < c->epsilon) { reason = REASON_CONVERGED; kk = k; goto done; }
        double rho_f = op_collapse(mode, rho_new);
        if (rho_f == 0.0 || !isfinite(rho_f)) { reason = REASON_BREAKDOWN; kk = k; goto done; }
        mw beta = op_div(mode, rho_new, rho);
        orc_scal_add(mode, n, beta.v, p, r);
        if (norm_all) orc_normalize(mode, n, p);
        rho = rho_new;
    }
    reason = REASON_MAX_ITERS; kk = max_iters;
done:
    if (last_rec != kk) RECORD(kk, rel);
    res->iterations = kk;
    res->reason = reason;
    res->final_rel = rel;
    res->n_hist = nh;
    free(q); free(r); free(p); free(ws);
#undef REL
#undef RECORD
    return 0;
}

/* Run `iters` unconditional CG iterations (no stop test, no history) from
 * x0=0: the bounded CPU-baseline sample for bench.py.  Returns the final
 * FP64-collapsed rho so the work cannot be elided. */
double orc_cg_iterations(const orc_cfg *c, int64_t n, const int64_t *rp, const int64_t *ci,
                         const double *va, const double *b, int64_t iters, double *x) {
    int mode = c->mode, w = WORDS[mode];
    int quasi = (mode == M_QDW || mode == M_QTW);
    int norm_r = quasi && c->normalization != NORM_NONE;
    size_t sz = sizeof(double) * (size_t)w * (size_t)n;
    double *q = (double *)calloc(1, sz), *r = (double *)calloc(1, sz), *p = (double *)calloc(1, sz);
    memset(x, 0, sz);
    orc_spmv(mode, n, rp, ci, va, x, n, q);
    orc_residual(mode, n, b, q, r);
    if (norm_r) orc_normalize(mode, n, r);
    memcpy(p, r, sz);
    mw rho; dot_cfg(c, n, r, r, &rho);
    for (int64_t k = 1; k <= iters; k++) {
        orc_spmv(mode, n, rp, ci, va, p, n, q);
        mw pq; dot_cfg(c, n, p, q, &pq);
        mw alpha = op_div(mode, rho, pq);
        orc_axpy(mode, n, alpha.v, p, x);
        mw na = op_neg(mode, alpha);
        orc_axpy(mode, n, na.v, q, r);
        if (norm_r) orc_normalize(mode, n, r);
        mw rho_new; dot_cfg(c, n, r, r, &rho_new);
        mw beta = op_div(mode, rho_new, rho);
        orc_scal_add(mode, n, beta.v, p, r);
        rho = rho_new;
    }
    double out = op_collapse(mode, rho);
    free(q); free(r); free(p);
    return out;
}
