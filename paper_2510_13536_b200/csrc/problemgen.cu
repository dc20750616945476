// problemgen.cu -- native exact problem generation (reference
// problemgen.py:47-108, `generate`).  Host code only.
//
// The reference sums each row with `ExactValue` (oracle.py:35-128, arbitrary-precision
// dyadic rationals in pure Python), rounds the sum to FP64 (ties to even), and absorbs
// the rounding gap into the diagonal, nudging b_i by up to 4 ulps (problemgen.py:37-44)
// until the perturbed diagonal is an FP64 number.  That is exact arithmetic on
// multiples of 2^-1074, so here every exact value is a fixed-point two's-complement
// integer in units of 2^-1074 (34 x 64-bit limbs: 2098 bits of FP64 range + sign +
// 60 bits of row-length headroom).  Adding an FP64 touches two limbs plus a carry;
// rounding finds the top bit and applies round-half-even on the 53-bit window.  Rows
// are independent and split across host threads; the error reported is the one of the
// first failing row, as the reference's sequential loop raises it.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#include "mwcg_internal.h"
#include "../../include/mwcg_cuda.h"

namespace mwcg {
void set_error(const char *fmt, ...);
}

namespace {

constexpr int NL = 34;  // limbs

struct Exact {
    uint64_t w[NL];
    void zero() { memset(w, 0, sizeof w); }
    bool is_zero() const {
        for (int k = 0; k < NL; k++)
            if (w[k]) return false;
        return true;
    }
    bool negative() const { return (int64_t)w[NL - 1] < 0; }
};

inline void add_shifted(Exact &a, uint64_t m, int off, bool neg) {
    int limb = off >> 6, sh = off & 63;
    uint64_t lo = m << sh;
    uint64_t hi = sh ? (m >> (64 - sh)) : 0;
    if (!neg) {
        unsigned __int128 t = (unsigned __int128)a.w[limb] + lo;
        a.w[limb] = (uint64_t)t;
        uint64_t c = (uint64_t)(t >> 64);
        t = (unsigned __int128)a.w[limb + 1] + hi + c;
        a.w[limb + 1] = (uint64_t)t;
        c = (uint64_t)(t >> 64);
        for (int k = limb + 2; c && k < NL; k++) c = (++a.w[k] == 0);
    } else {
        uint64_t old = a.w[limb];
        a.w[limb] = old - lo;
        uint64_t b = old < lo;
        old = a.w[limb + 1];
        uint64_t sub = hi + b;  // hi < 2^63, no overflow
        a.w[limb + 1] = old - sub;
        b = old < sub;
        for (int k = limb + 2; b && k < NL; k++) b = (a.w[k]-- == 0);
    }
}

// a += (neg ? -x : x); x finite
inline void add_fp64(Exact &a, double x, bool neg = false) {
    uint64_t bits;
    memcpy(&bits, &x, 8);
    uint64_t E = (bits >> 52) & 0x7ff, frac = bits & ((1ull << 52) - 1);
    uint64_t m = E ? (frac | (1ull << 52)) : frac;
    if (!m) return;
    int off = E ? (int)E - 1 : 0;  // value = m * 2^(off - 1074)
    add_shifted(a, m, off, ((bits >> 63) != 0) != neg);
}

inline void add_exact(Exact &a, const Exact &b, bool neg) {
    if (!neg) {
        uint64_t c = 0;
        for (int k = 0; k < NL; k++) {
            unsigned __int128 t = (unsigned __int128)a.w[k] + b.w[k] + c;
            a.w[k] = (uint64_t)t;
            c = (uint64_t)(t >> 64);
        }
    } else {
        uint64_t br = 0;
        for (int k = 0; k < NL; k++) {
            unsigned __int128 t = (unsigned __int128)a.w[k] - b.w[k] - br;
            a.w[k] = (uint64_t)t;
            br = (uint64_t)(t >> 64) ? 1 : 0;
        }
    }
}

inline uint64_t bits_at(const uint64_t *w, int pos, int cnt) {  // cnt <= 64, pos >= 0
    int limb = pos >> 6, sh = pos & 63;
    uint64_t v = w[limb] >> sh;
    if (sh && limb + 1 < NL) v |= w[limb + 1] << (64 - sh);
    return cnt == 64 ? v : (v & ((1ull << cnt) - 1));
}

// ExactValue.to_fp64 (oracle.py:115-128): nearest, ties to even, overflow -> +-inf.
// *exact = the value is an FP64 number (false on overflow).
double round_fp64(const Exact &a, bool *exact) {
    uint64_t mag[NL];
    bool neg = a.negative();
    if (neg) {
        uint64_t c = 1;
        for (int k = 0; k < NL; k++) {
            unsigned __int128 t = (unsigned __int128)(~a.w[k]) + c;
            mag[k] = (uint64_t)t;
            c = (uint64_t)(t >> 64);
        }
    } else {
        memcpy(mag, a.w, sizeof mag);
    }
    int L = NL - 1;
    while (L >= 0 && !mag[L]) L--;
    if (L < 0) {
        *exact = true;
        return 0.0;
    }
    int h = L * 64 + 63 - __builtin_clzll(mag[L]);
    double v;
    if (h <= 52) {
        v = ldexp((double)mag[0], -1074);  // exact (subnormal or smallest binade)
        *exact = true;
    } else {
        int s = h - 52;
        uint64_t top = bits_at(mag, s, 53);
        bool half = bits_at(mag, s - 1, 1) != 0;
        bool sticky = false;
        if (s - 1 > 0) {
            int full = (s - 1) >> 6;
            for (int k = 0; k < full && !sticky; k++) sticky = mag[k] != 0;
            int rem = (s - 1) & 63;
            if (!sticky && rem) sticky = (mag[full] & ((1ull << rem) - 1)) != 0;
        }
        if (half && (sticky || (top & 1))) {
            top++;
            if (top == (1ull << 53)) {
                top >>= 1;
                s++;
            }
        }
        v = ldexp((double)top, s - 1074);
        *exact = !half && !sticky && std::isfinite(v);
    }
    return neg ? -v : v;
}

enum RowErr { ROW_OK = 0, ROW_NONFINITE, ROW_OVERFLOW, ROW_NO_DIAG, ROW_NO_REPR };

struct RowOut {
    int err;
    int nudge;
};

// problemgen.py:68-105 for one row
RowOut gen_row(int64_t i, const int64_t *rp, const int64_t *ci, const double *va, double *nv,
               double *b, double *deltas) {
    int64_t lo = rp[i], hi = rp[i + 1];
    Exact s;
    s.zero();
    for (int64_t k = lo; k < hi; k++) {
        if (!std::isfinite(va[k])) return {ROW_NONFINITE, 0};
        add_fp64(s, va[k]);
    }
    // diagonal_index (sparse.py:81-87): searchsorted on the row's columns
    int64_t a = lo, e = hi;
    while (a < e) {
        int64_t mid = a + (e - a) / 2;
        if (ci[mid] < i) a = mid + 1;
        else e = mid;
    }
    int64_t di = (a < hi && ci[a] == i) ? a : -1;
    bool ex;
    double br = round_fp64(s, &ex);
    if (!std::isfinite(br)) return {ROW_OVERFLOW, 0};
    // _nudges (problemgen.py:37-44): x, up1, down1, up2, down2, ...
    double up = br, down = br;
    for (int nc = 0; nc <= 8; nc++) {
        double bi;
        if (nc == 0) bi = br;
        else if (nc & 1) bi = up = nextafter(up, INFINITY);
        else bi = down = nextafter(down, -INFINITY);
        if (!std::isfinite(bi)) return {ROW_NONFINITE, 0};  // ExactValue.from_fp64(inf)
        Exact d;
        d.zero();
        add_fp64(d, bi);
        add_exact(d, s, true);
        if (d.is_zero()) {
            b[i] = bi;
            deltas[i] = 0.0;
            return {ROW_OK, nc};
        }
        if (di < 0) continue;
        add_fp64(d, va[di]);  // new_diag = a_dd + delta
        bool rep;
        double nd = round_fp64(d, &rep);
        if (!std::isfinite(nd)) return {ROW_NONFINITE, 0};  // _representable: from_fp64(inf)
        if (rep) {
            b[i] = bi;
            deltas[i] = 0.0;
            if (nd != va[di]) {
                deltas[i] = nd - va[di];
                nv[di] = nd;
            }
            return {ROW_OK, nc};
        }
    }
    return {di < 0 ? ROW_NO_DIAG : ROW_NO_REPR, 0};
}

}  // namespace

extern "C" int mwcg_problem_generate(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                                     const double *values, double *new_values, double *b,
                                     double *deltas, int64_t *max_ulp_adjustment, int threads) {
    if (n < 0 || (n > 0 && (!row_ptr || !b || !deltas)) || !max_ulp_adjustment) {
        mwcg::set_error("problem_generate: bad arguments");
        return MWCG_ERR_VALUE;
    }
    int64_t nnz = n ? row_ptr[n] : 0;
    if (nnz && new_values != values) memcpy(new_values, values, (size_t)nnz * sizeof(double));
    int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    if (T < 1) T = 1;
    if ((int64_t)T > n / 4096 + 1) T = (int)(n / 4096 + 1);
    std::vector<int64_t> first_err(T, INT64_MAX);
    std::vector<int> err_kind(T, ROW_OK), nudge(T, 0);
    auto work = [&](int t) {
        int64_t r0 = n * t / T, r1 = n * (t + 1) / T;
        int mx = 0;
        for (int64_t i = r0; i < r1; i++) {
            RowOut o = gen_row(i, row_ptr, col_idx, values, new_values, b, deltas);
            if (o.err) {
                first_err[t] = i;
                err_kind[t] = o.err;
                break;
            }
            int u = (o.nudge + 1) / 2;
            if (u > mx) mx = u;
        }
        nudge[t] = mx;
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; t++) pool.emplace_back(work, t);
    work(0);
    for (auto &th : pool) th.join();
    int64_t mx = 0;
    for (int t = 0; t < T; t++) {
        if (first_err[t] != INT64_MAX) {
            int64_t i = first_err[t];
            switch (err_kind[t]) {
            case ROW_NONFINITE: mwcg::set_error("NaN/Inf have no exact dyadic representation"); break;
            case ROW_OVERFLOW: mwcg::set_error("row %lld: exact row sum overflows FP64", (long long)i); break;
            case ROW_NO_DIAG:
                mwcg::set_error("row %lld: inexact row sum but no diagonal entry to absorb the "
                                "rounding gap", (long long)i);
                break;
            default:
                mwcg::set_error("row %lld: no representable diagonal within 4 ulps of the rounded "
                                "row sum", (long long)i);
            }
            return MWCG_ERR_VALUE;
        }
        if (nudge[t] > mx) mx = nudge[t];
    }
    *max_ulp_adjustment = mx;
    return 0;
}
