"""Generate golden fixtures from the REAL reference package (`mwcg`).

Run in the build container only (the reference tree is not on the GPU box):

    python tests/golden/make_golden.py [--skip-slow]

The reference imports `gmpy2` for its scalar FMA (eft.py:16, 36-39), which is
absent here.  A shim exposing glibc's correctly rounded `fma` is written to a
temp dir and put on sys.path first; the reference's own
test-suite passes under it (287/287), so its FMA boundary stays pinned.

Outputs (committed, small):
  ops.json       scalar EFT / multi-word ops on adversarial inputs (hex)
  kernels.json   every `_fast.KERNELS[mode][op]` on small seeded inputs (hex)
  cg_small.json  full cg_solve runs on small problems (x words, history; hex)
  cg_c1.json     BASELINE config 1 (256x256 Poisson) for all five arithmetics:
                 iterations, reason, history, sha256 of the solution words
  cg_accept.json acceptance problems (pkg/tests/test_acceptance.py:68-96):
                 iteration counts and partition bands
"""

import argparse
import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

_SHIM = '''
import ctypes, ctypes.util
_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.fma.restype = ctypes.c_double
_libm.fma.argtypes = [ctypes.c_double] * 3
def fma(a, b, c):
    return _libm.fma(float(a), float(b), float(c))
'''


def _import_reference():
    shim_dir = tempfile.mkdtemp(prefix="gmpy2shim")
    with open(os.path.join(shim_dir, "gmpy2.py"), "w") as f:
        f.write(_SHIM)
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba"))
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, shim_dir)
    import mwcg  # noqa: F401
    from mwcg import cg, kernels, multiword, problemgen, sparse
    return cg, kernels, multiword, problemgen, sparse


def hx(v):
    return float(v).hex()


def hxl(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def words_hash(words):
    arr = np.ascontiguousarray(np.stack([np.asarray(w, dtype=np.float64) for w in words]))
    return hashlib.sha256(arr.tobytes()).hexdigest()


def csr_hash(A):
    h = hashlib.sha256()
    for a in (np.ascontiguousarray(A.row_ptr, dtype=np.int64),
              np.ascontiguousarray(A.col_idx, dtype=np.int64),
              np.ascontiguousarray(A.values, dtype=np.float64)):
        h.update(a.tobytes())
    return h.hexdigest()


def csr_json(A):
    return {"n": int(A.n_rows), "row_ptr": [int(v) for v in A.row_ptr],
            "col_idx": [int(v) for v in A.col_idx], "values": hxl(A.values)}


# ---------------------------------------------------------------------------
def adversarial_words(rng, count, w):
    """Multi-word inputs stressing ties, zeros, cancellation, unnormalized words."""
    out = []
    specials = [0.0, -0.0, 1.0, -1.0, 2.0 ** -60, 3.0, 0.1, -0.1]
    for t in range(count):
        kind = t % 6
        if kind == 0:      # normalized-ish random
            hi = rng.standard_normal() * 2.0 ** rng.integers(-20, 20)
            ws = [hi, hi * 2.0 ** -53 * rng.uniform(-1, 1), hi * 2.0 ** -106 * rng.uniform(-1, 1)]
        elif kind == 1:    # unnormalized / overlapping
            ws = list(rng.standard_normal(3))
        elif kind == 2:    # exact ties in magnitude
            v = float(rng.choice([1.0, 0.5, 3.0]))
            ws = [v, -v * 2.0 ** -53, v * 2.0 ** -106]
        elif kind == 3:    # zeros and signed zeros
            ws = [float(rng.choice(specials)) for _ in range(3)]
        elif kind == 4:    # reversed magnitudes
            hi = rng.standard_normal()
            ws = [hi * 2.0 ** -60, hi, hi * 2.0 ** -30]
        else:              # tiny / huge
            e = int(rng.integers(-900, 900))
            ws = [np.ldexp(rng.uniform(1, 2), e), np.ldexp(rng.uniform(-1, 1), e - 55),
                  np.ldexp(rng.uniform(-1, 1), e - 110)]
        out.append([float(v) for v in ws[:w]])
    return out


def gen_ops(mw, eft):
    rng = np.random.default_rng(1234)
    cases = []
    # pair the "a" and "b" operands so ties across operands also occur
    A2 = adversarial_words(rng, 240, 2)
    B2 = adversarial_words(rng, 240, 2)
    for i in range(0, 240, 7):   # force cross-operand ties
        B2[i] = [A2[i][0], -A2[i][1]]
    A3 = adversarial_words(rng, 240, 3)
    B3 = adversarial_words(rng, 240, 3)
    for i in range(0, 240, 5):
        B3[i] = [-A3[i][0], A3[i][2], A3[i][1]]
    for i in range(0, 240, 11):
        B3[i] = [A3[i][1], A3[i][0], -A3[i][2]]
    DW, TW = mw.DoubleWord, mw.TripleWord
    fam = {
        "dw": (DW, A2, B2, mw.dw_add, mw.dw_mul, mw.dxdw_mul, mw.dxdw_add, mw.normalize_dw, mw.dw_div),
        "qdw": (DW, A2, B2, mw.qdw_add, mw.qdw_mul, mw.dxqdw_mul, mw.dxqdw_add, mw.normalize_dw, mw.qdw_div),
        "tw": (TW, A3, B3, mw.tw_add, mw.tw_mul, mw.dxtw_mul, mw.dxtw_add, None, mw.tw_div),
        "qtw": (TW, A3, B3, mw.qtw_add, mw.qtw_mul, mw.dxqtw_mul, mw.dxqtw_add, mw.normalize_tw, mw.qtw_div),
    }
    for mode, (T, As, Bs, add, mul, dxmul, dxadd, norm, div) in fam.items():
        for a, b in zip(As, Bs):
            ta, tb = T(*a), T(*b)
            c = {"mode": mode, "a": hxl(a), "b": hxl(b),
                 "add": hxl(add(ta, tb)), "mul": hxl(mul(ta, tb)),
                 "dxmul": hxl(dxmul(a[0], tb)), "dxadd": hxl(dxadd(a[0], tb))}
            if norm is not None:
                c["normalize"] = hxl(norm(ta))
            try:
                c["div"] = hxl(div(ta, tb))
            except (ZeroDivisionError, OverflowError) as exc:  # pragma: no cover
                c["div_error"] = type(exc).__name__
            cases.append(c)
    eft_cases = []
    for a, b in zip(A2, B2):
        eft_cases.append({"a": hx(a[0]), "b": hx(b[0]),
                          "two_sum": hxl(eft.two_sum(a[0], b[0])),
                          "quick_two_sum": hxl(eft.quick_two_sum(a[0], b[0])),
                          "two_prod": hxl(eft.two_prod_fma(a[0], b[0]))})
    return {"ops": cases, "eft": eft_cases}


def rand_vec(kn, mode, n, seed):
    """pkg/tests/test_kernels.py:14-22 with a third word for TW modes."""
    rng = np.random.default_rng(seed)
    v = kn.MultiwordVector.from_fp64(rng.standard_normal(n), mode)
    if mode != "fp64":
        v.words[1][:] = rng.standard_normal(n) * 1e-20
        if kn.mode_words(mode) == 3:
            v.words[2][:] = rng.standard_normal(n) * 1e-37
    return v


def gen_kernels(kn, mw, sparse):
    out = {"cases": []}
    mats = {"random25": sparse.random_symmetric(25, seed=4),
            "lap5": sparse.laplacian_2d(5)}
    out["matrices"] = {k: csr_json(v) for k, v in mats.items()}
    for mode in kn.MODES:
        w = kn.mode_words(mode)
        for mname, A in mats.items():
            n = A.n_rows
            x = rand_vec(kn, mode, n, 5)
            y = kn.spmv(A, x)
            out["cases"].append({"op": "spmv", "mode": mode, "matrix": mname,
                                 "x": [hxl(wd) for wd in x.words],
                                 "y": [hxl(wd) for wd in y.words]})
        n = 57
        x = rand_vec(kn, mode, n, 8)
        y = rand_vec(kn, mode, n, 9)
        for parts in (1, 3, 7, 57):
            d = kn.dot(x, y, partitions=parts)
            out["cases"].append({"op": "dot", "mode": mode, "partitions": parts,
                                 "x": [hxl(wd) for wd in x.words],
                                 "y": [hxl(wd) for wd in y.words],
                                 "out": hxl(d if w > 1 else [d])})
        # axpy / scal_add with a non-trivial scalar (1/3 in the mode)
        one = kn.scalar_one(mode)
        three = 3.0 if mode == "fp64" else (mw.DoubleWord(3.0, 0.0) if w == 2 else mw.TripleWord(3.0, 0.0, 0.0))
        alpha = kn.scalar_div(mode, one, three)
        xa = rand_vec(kn, mode, 33, 14)
        ya = rand_vec(kn, mode, 33, 15)
        y0 = [hxl(wd) for wd in ya.words]
        kn.axpy(alpha, xa, ya)
        out["cases"].append({"op": "axpy", "mode": mode, "alpha": hxl(alpha if w > 1 else [alpha]),
                             "x": [hxl(wd) for wd in xa.words], "y": y0,
                             "out": [hxl(wd) for wd in ya.words]})
        pa = rand_vec(kn, mode, 33, 16)
        p0 = [hxl(wd) for wd in pa.words]
        kn.scal_then_add(alpha, pa, xa)
        out["cases"].append({"op": "scal_add", "mode": mode, "beta": hxl(alpha if w > 1 else [alpha]),
                             "p": p0, "r": [hxl(wd) for wd in xa.words],
                             "out": [hxl(wd) for wd in pa.words]})
        rng = np.random.default_rng(17)
        b = rng.standard_normal(20)
        q = rand_vec(kn, mode, 20, 17)
        r = kn.residual(b, q)
        out["cases"].append({"op": "residual", "mode": mode, "b": hxl(b),
                             "q": [hxl(wd) for wd in q.words],
                             "out": [hxl(wd) for wd in r.words]})
        if mode in ("qdw", "qtw"):
            v = rand_vec(kn, mode, 30, 19)
            v.words[1][:] = v.words[0] * 0.5
            v0 = [hxl(wd) for wd in v.words]
            kn.normalize_vector(v)
            out["cases"].append({"op": "normalize", "mode": mode, "v": v0,
                                 "out": [hxl(wd) for wd in v.words]})
        # collapsed sequential norm (kernels.py:290-296)
        v = rand_vec(kn, mode, 41, 21)
        out["cases"].append({"op": "norm2", "mode": mode, "v": [hxl(wd) for wd in v.words],
                             "out": hx(kn.norm2_fp64(v))})
    # norm metrics on a DW iterate (kernels.py:305-328)
    A = mats["lap5"]
    xs = np.random.default_rng(3).uniform(-1, 1, A.n_rows)
    b = np.zeros(A.n_rows)
    kn._fast.spmv_fp64(A.row_ptr, A.col_idx, A.values, xs, b)
    for mode in kn.MODES:
        x = rand_vec(kn, mode, A.n_rows, 22)
        err, tr = kn.norm_metrics_tw(x, xs, A, b)
        out["cases"].append({"op": "metrics", "mode": mode, "matrix": "lap5",
                             "x": [hxl(wd) for wd in x.words], "x_star": hxl(xs), "b": hxl(b),
                             "err": hx(err), "true_res": hx(tr)})
    return out


def result_json(res, full_x=True):
    d = {"converged": bool(res.converged), "reason": res.reason,
         "iterations": int(res.iterations),
         "final_rel": hx(res.final_recurrence_residual),
         "history": [[int(h.iteration), hx(h.recurrence_residual), hx(h.true_residual),
                      None if h.error_norm is None else hx(h.error_norm)] for h in res.history],
         "x_sha256": words_hash(res.x.words)}
    if full_x:
        d["x"] = [hxl(wd) for wd in res.x.words]
    return d


def gen_cg_small(cg, kn, sparse, problemgen):
    probs = {}
    probs["identity6"] = (sparse.identity(6), np.arange(1.0, 7.0), None)
    A22 = sparse.CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]),
                           np.array([4.0, 1.0, 1.0, 3.0]))
    probs["spd2"] = (A22, np.array([1.0, 2.0]), None)
    Ab = sparse.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, -1.0]))
    probs["indef2"] = (Ab, np.array([1.0, 1.0]), None)
    p = problemgen.generate(sparse.laplacian_2d(4))
    probs["genlap4"] = (p.matrix, p.b, p.x_star)
    p = problemgen.generate(sparse.laplacian_2d(8))
    probs["genlap8"] = (p.matrix, p.b, p.x_star)
    p = problemgen.generate(sparse.scaled_laplacian_2d(6, decades=3.0, seed=2))
    probs["genslap6"] = (p.matrix, p.b, p.x_star)
    p = problemgen.generate(sparse.random_symmetric(40, seed=5))
    probs["genrand40"] = (p.matrix, p.b, p.x_star)
    out = {"problems": {}, "runs": []}
    for name, (A, b, xs) in probs.items():
        out["problems"][name] = {"A": csr_json(A), "b": hxl(b),
                                 "x_star": None if xs is None else hxl(xs)}
    runs = []
    for name in probs:
        for mode in kn.MODES:
            runs.append((name, dict(mode=mode, epsilon=1e-14 if mode == "fp64" else 1e-26,
                                    history_stride=3)))
    for mode in ("qdw", "qtw"):
        for norm in ("none", "after-axpy", "every-op"):
            for name in ("genlap8", "genslap6"):
                runs.append((name, dict(mode=mode, epsilon=1e-24, normalization=norm,
                                        history_stride=4)))
    for mode in kn.MODES:
        for parts in (2, 5):
            runs.append(("genrand40", dict(mode=mode, epsilon=1e-24 if mode != "fp64" else 1e-14,
                                           partitions=parts, history_stride=7)))
        runs.append(("genslap6", dict(mode=mode, epsilon=1e-300, max_iterations=15,
                                      history_stride=5)))
    for spec in runs:
        name, kw = spec
        A, b, xs = probs[name]
        cfg = cg.SolverConfig(**kw)
        res = cg.cg_solve(A, b, cfg, x_star=xs)
        out["runs"].append({"problem": name, "config": {**kw}, "x0": None,
                            "result": result_json(res)})
    # explicit x0 cases
    A, b, xs = probs["genlap4"]
    x0 = np.random.default_rng(8).uniform(-1, 1, A.n_rows)
    for mode in kn.MODES:
        kw = dict(mode=mode, epsilon=1e-20 if mode != "fp64" else 1e-13, history_stride=2)
        res = cg.cg_solve(A, b, cg.SolverConfig(**kw), x0=x0, x_star=xs)
        out["runs"].append({"problem": "genlap4", "config": kw, "x0": hxl(x0),
                            "result": result_json(res)})
    return out


def c1_problem(sparse, kn):
    A = sparse.laplacian_2d(256)
    x_true = np.random.default_rng(0).uniform(-1.0, 1.0, A.n_rows)
    b = np.zeros(A.n_rows)
    kn._fast.spmv_fp64(A.row_ptr, A.col_idx, A.values, x_true, b)
    return A, b, x_true


def gen_c1(cg, kn, sparse, modes):
    A, b, x_true = c1_problem(sparse, kn)
    out = {"matrix_sha256": csr_hash(A),
           "b_sha256": hashlib.sha256(b.tobytes()).hexdigest(),
           "x_true_sha256": hashlib.sha256(x_true.tobytes()).hexdigest(),
           "runs": []}
    for mode in modes:
        cfg = cg.SolverConfig(mode=mode, epsilon=1e-12, max_iterations=10000,
                              history_stride=100)
        t = time.perf_counter()
        res = cg.cg_solve(A, b, cfg, x_star=x_true)
        dt = time.perf_counter() - t
        d = result_json(res, full_x=False)
        d["seconds"] = dt
        out["runs"].append({"mode": mode, "config": {"epsilon": 1e-12, "max_iterations": 10000,
                                                      "history_stride": 100}, "result": d})
        print(f"C1 {mode}: it={res.iterations} {dt:.1f}s", flush=True)
    return out


def gen_accept(cg, kn, sparse, problemgen, slow):
    out = {"runs": []}
    easy = problemgen.generate(sparse.laplacian_2d(64))
    hard = problemgen.generate(sparse.scaled_laplacian_2d(16, decades=4.0, seed=1))
    out["hard_problem"] = {"A": csr_json(hard.matrix), "b": hxl(hard.b)}
    out["easy_b_sha256"] = hashlib.sha256(easy.b.tobytes()).hexdigest()
    out["easy_matrix_sha256"] = csr_hash(easy.matrix)
    for mode in kn.MODES:
        cfg = cg.SolverConfig(mode=mode, epsilon=1e-32, history_stride=100)
        res = cg.cg_solve(easy.matrix, easy.b, cfg, x_star=easy.x_star)
        out["runs"].append({"problem": "easy", "mode": mode, "normalization": "after-axpy",
                            "partitions": 1, "result": result_json(res, full_x=False)})
        print(f"easy {mode}: it={res.iterations}", flush=True)
    parts_list = (1, 2, 8, 37, 148) if slow else (1,)
    for mode in ("dw", "qdw", "tw", "qtw"):
        for parts in parts_list:
            cfg = cg.SolverConfig(mode=mode, epsilon=1e-24, max_iterations=20000,
                                  partitions=parts, history_stride=100)
            res = cg.cg_solve(hard.matrix, hard.b, cfg, x_star=hard.x_star)
            out["runs"].append({"problem": "hard", "mode": mode, "normalization": "after-axpy",
                                "partitions": parts, "result": result_json(res, full_x=False)})
            print(f"hard {mode} P={parts}: it={res.iterations}", flush=True)
    for mode in ("qdw", "qtw"):
        cfg = cg.SolverConfig(mode=mode, epsilon=1e-24, max_iterations=20000,
                              normalization="none", history_stride=100)
        res = cg.cg_solve(hard.matrix, hard.b, cfg, x_star=hard.x_star)
        out["runs"].append({"problem": "hard", "mode": mode, "normalization": "none",
                            "partitions": 1, "result": result_json(res, full_x=False)})
        print(f"hard {mode} none: it={res.iterations} {res.reason}", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-slow", action="store_true")
    ap.add_argument("--only", default="ops,kernels,small,c1,accept")
    args = ap.parse_args()
    cg, kn, mw, problemgen, sparse = _import_reference()
    from mwcg import eft
    only = set(args.only.split(","))

    def dump(name, obj):
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(obj, f, separators=(",", ":"))
        print("wrote", name, os.path.getsize(os.path.join(HERE, name)), "bytes", flush=True)

    if "ops" in only:
        dump("ops.json", gen_ops(mw, eft))
    if "kernels" in only:
        dump("kernels.json", gen_kernels(kn, mw, sparse))
    if "small" in only:
        dump("cg_small.json", gen_cg_small(cg, kn, sparse, problemgen))
    if "c1" in only:
        modes = ("fp64", "dw", "qdw", "qtw") if args.skip_slow else kn.MODES
        dump("cg_c1.json", gen_c1(cg, kn, sparse, modes))
    if "accept" in only:
        dump("cg_accept.json", gen_accept(cg, kn, sparse, problemgen, not args.skip_slow))


if __name__ == "__main__":
    main()
