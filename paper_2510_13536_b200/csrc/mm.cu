// mm.cu -- native Matrix Market (coordinate) parser: the ingestion step of the
// solve path (reference sparse.py:115-196, read_matrix_market
// / _parse_mm).  Host code only.  Same grammar, same error messages and line
// numbers as the reference parser; inputs outside the fast grammar (non-ASCII
// bytes, lone CR line breaks, '_' digit separators, hex floats, integers that
// overflow int64) return MWCG_MM_FALLBACK so the caller can use its exact
// pure-Python restatement instead.
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include "mwcg_internal.h"
#include "../../include/mwcg_cuda.h"

namespace {

// Python str.split() whitespace over ASCII
inline bool is_ws(unsigned char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c ||
           (c >= 0x1c && c <= 0x1f);
}

struct Line {
    const char *b, *e;  // stripped
};

struct Cursor {
    const char *p, *end;
    int64_t lineno = 0;
    // next line (without terminator), false at end of input
    bool next(Line &ln) {
        if (p >= end) return false;
        const char *q = (const char *)memchr(p, '\n', (size_t)(end - p));
        const char *le = q ? q : end;
        ln.b = p;
        ln.e = le;
        p = q ? q + 1 : end;
        lineno++;
        while (ln.b < ln.e && is_ws((unsigned char)*ln.b)) ln.b++;
        while (ln.e > ln.b && is_ws((unsigned char)ln.e[-1])) ln.e--;
        return true;
    }
};

int split(const Line &ln, std::string *tok, int maxtok) {
    int n = 0;
    const char *s = ln.b;
    while (s < ln.e) {
        while (s < ln.e && is_ws((unsigned char)*s)) s++;
        if (s >= ln.e) break;
        const char *t = s;
        while (t < ln.e && !is_ws((unsigned char)*t)) t++;
        if (n < maxtok) tok[n].assign(s, t);
        n++;
        s = t;
    }
    return n;
}

enum { OK = 0, BAD = 1, FALLBACK = 2 };

// Python int(): [+-]?digits (underscore separators -> fallback)
int parse_int(const std::string &t, long long &v) {
    if (t.find('_') != std::string::npos) return FALLBACK;
    size_t i = 0;
    if (i < t.size() && (t[i] == '+' || t[i] == '-')) i++;
    if (i == t.size()) return BAD;
    for (size_t k = i; k < t.size(); k++)
        if (t[k] < '0' || t[k] > '9') return BAD;
    errno = 0;
    v = strtoll(t.c_str(), nullptr, 10);
    if (errno == ERANGE) return FALLBACK;
    return OK;
}

// Python float(): decimal / inf / nan forms (hex, '_' and nan(...) -> fallback)
int parse_float(const std::string &t, double &v) {
    for (char c : t)
        if (c == '_' || c == 'x' || c == 'X' || c == '(' || c == ')') return FALLBACK;
    if (t.empty()) return BAD;
    char *endp = nullptr;
    v = strtod(t.c_str(), &endp);
    if (endp != t.c_str() + t.size()) return BAD;
    return OK;
}

std::string lower(std::string s) {
    for (auto &c : s) c = (char)tolower((unsigned char)c);
    return s;
}

int fail(mwcg_mm_info *info, int64_t line, const std::string &msg) {
    info->error_line = line;
    mwcg::set_error("%s", msg.c_str());
    return MWCG_MM_ERROR;
}

}  // namespace

extern "C" int mwcg_mm_parse(const char *data, int64_t len, mwcg_mm_info *info, int64_t *rows, int64_t *cols,
                             double *vals) {
    if (!info || (len > 0 && !data) || len < 0) {
        mwcg::set_error("bad argument");
        return MWCG_ERR_VALUE;
    }
    info->error_line = -1;
    for (int64_t i = 0; i < len; i++) {
        const unsigned char c = (unsigned char)data[i];
        if (c >= 0x80) return MWCG_MM_FALLBACK;                                 // ascii decode error path
        if (c == '\r' && (i + 1 >= len || data[i + 1] != '\n')) return MWCG_MM_FALLBACK;  // lone CR
    }
    Cursor cur{data, data + len};
    Line ln;
    if (!cur.next(ln)) return fail(info, 1, "empty input, missing banner");
    std::string tok[6];
    int nt = split(ln, tok, 6);
    if (nt != 5 || tok[0] != "%%MatrixMarket")
        return fail(info, 1,
                    "expected '%%MatrixMarket matrix coordinate real|integer general|symmetric' banner");
    const std::string obj = lower(tok[1]), fmt = lower(tok[2]), fld = lower(tok[3]), sym = lower(tok[4]);
    if (obj != "matrix" || fmt != "coordinate")
        return fail(info, 1, "unsupported object/format '" + obj + " " + fmt + "'");
    if (fld != "real" && fld != "integer")
        return fail(info, 1, "unsupported field '" + fld + "' (pattern/complex matrices are not accepted)");
    if (sym != "general" && sym != "symmetric") return fail(info, 1, "unsupported symmetry '" + sym + "'");
    const bool symmetric = sym == "symmetric";
    long long nr = 0, nc = 0, nz = 0;
    bool have_size = false;
    while (cur.next(ln)) {
        if (ln.b == ln.e || *ln.b == '%') continue;
        nt = split(ln, tok, 4);
        if (nt != 3) return fail(info, cur.lineno, "size line must be 'rows cols nnz'");
        long long v[3];
        for (int k = 0; k < 3; k++) {
            const int r = parse_int(tok[k], v[k]);
            if (r == FALLBACK) return MWCG_MM_FALLBACK;
            if (r == BAD) return fail(info, cur.lineno, "size line must be 'rows cols nnz'");
        }
        nr = v[0];
        nc = v[1];
        nz = v[2];
        if (nr < 0 || nc < 0 || nz < 0) return fail(info, cur.lineno, "negative size");
        have_size = true;
        break;
    }
    if (!have_size) return fail(info, cur.lineno, "missing size line");
    if (symmetric && nr != nc) return fail(info, cur.lineno, "symmetric matrix must be square");
    info->n_rows = nr;
    info->n_cols = nc;
    info->nnz = nz;
    info->symmetric = symmetric ? 1 : 0;
    if (!rows) return 0;  // header pass: the caller allocates nnz entries
    long long k = 0;
    char buf[256];
    while (cur.next(ln)) {
        if (ln.b == ln.e || *ln.b == '%') continue;
        nt = split(ln, tok, 4);
        if (nt != 3) return fail(info, cur.lineno, "entry must be 'row col value'");
        long long i = 0, j = 0;
        double v = 0.0;
        int r0 = parse_int(tok[0], i), r1 = r0 == OK ? parse_int(tok[1], j) : r0;
        int r2 = r1 == OK ? parse_float(tok[2], v) : r1;
        if (r0 == FALLBACK || r1 == FALLBACK || r2 == FALLBACK) return MWCG_MM_FALLBACK;
        if (r0 != OK || r1 != OK || r2 != OK) return fail(info, cur.lineno, "entry must be 'row col value'");
        if (k >= nz) {
            snprintf(buf, sizeof buf, "more than the declared %lld entries", nz);
            return fail(info, cur.lineno, buf);
        }
        if (!(1 <= i && i <= nr) || !(1 <= j && j <= nc)) {
            snprintf(buf, sizeof buf, "index (%lld, %lld) out of range for %lldx%lld", i, j, nr, nc);
            return fail(info, cur.lineno, buf);
        }
        if (symmetric && j > i) {
            snprintf(buf, sizeof buf, "symmetric file must store the lower triangle only, got (%lld, %lld)", i,
                     j);
            return fail(info, cur.lineno, buf);
        }
        rows[k] = i - 1;
        cols[k] = j - 1;
        vals[k] = v;
        k++;
    }
    if (k != nz) {
        snprintf(buf, sizeof buf, "declared %lld entries but found %lld", nz, k);
        return fail(info, cur.lineno, buf);
    }
    return 0;
}
