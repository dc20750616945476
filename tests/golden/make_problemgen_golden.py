"""Generate tests/golden/problemgen.json from the REAL reference `problemgen.generate`
(problemgen.py:47-108).  Build container only (needs /root/reference):

    python tests/golden/make_problemgen_golden.py

Cases: the reference's own test matrices (pkg/tests/test_problemgen.py), moderate
generator matrices with perturbed (inexact) values, and ~1500 tiny adversarial
matrices (wide exponent ranges, subnormals, near-overflow entries, cancellation,
missing diagonals) so every branch of the nudge / absorption / error logic is hit.
Each case stores the input CSR and either the outputs (hex) or the error message.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import HERE, _import_reference, hx  # noqa: E402


def _csr_case(n, rp, ci, va):
    return {"n": int(n), "row_ptr": [int(v) for v in rp], "col_idx": [int(v) for v in ci],
            "values": [hx(v) for v in va]}


def _adversarial_value(rng):
    kind = rng.integers(0, 9)
    sign = -1.0 if rng.random() < 0.4 else 1.0
    if kind == 0:
        return float(rng.integers(-8, 9))
    if kind == 1:
        return float(rng.standard_normal())
    if kind == 2:
        return sign * float(np.ldexp(1.0 + rng.random(), int(rng.integers(-60, 61))))
    if kind == 3:
        return sign * float(np.ldexp(1.0 + rng.random(), int(rng.integers(-1074, 1024))))
    if kind == 4:
        return sign * float(rng.integers(1, 1 << 20)) * 5e-324
    if kind == 5:
        return sign * (1.7976931348623157e308 - float(rng.integers(0, 4)) * 2.0 ** 970)
    if kind == 6:
        return sign * float(np.ldexp(float(rng.integers(1, 1 << 53)), int(rng.integers(-30, 30))))
    if kind == 7:
        return -0.0 if rng.random() < 0.5 else 0.0
    return sign * (1.0 + float(rng.integers(1, 16)) * 2.0 ** -52)


def _tiny(rng):
    n = int(rng.integers(1, 4))
    rp, ci, va = [0], [], []
    for i in range(n):
        cols = set(int(c) for c in rng.choice(n, size=int(rng.integers(0, n + 1)), replace=False))
        if rng.random() < 0.8:
            cols.add(i)
        for c in sorted(cols):
            ci.append(c)
            va.append(_adversarial_value(rng))
        rp.append(len(ci))
    return n, np.array(rp), np.array(ci), np.array(va, dtype=np.float64)


def main():
    _, _, _, problemgen, sparse = _import_reference()
    cases = []

    def run(name, A):
        c = {"name": name, **_csr_case(A.n_rows, A.row_ptr, A.col_idx, A.values)}
        try:
            p = problemgen.generate(A)
        except ValueError as exc:
            c["error"] = str(exc)
        else:
            c["b"] = [hx(v) for v in p.b]
            c["out_values"] = [hx(v) for v in p.matrix.values]
            c["perturbation_norm"] = hx(p.perturbation_norm)
            c["max_ulp_adjustment"] = int(p.max_ulp_adjustment)
        cases.append(c)

    C = sparse.CsrMatrix
    run("identity5", sparse.identity(5))
    run("laplacian4", sparse.laplacian_2d(4))
    run("random60", sparse.random_symmetric(60, seed=5))
    run("random40", sparse.random_symmetric(40, seed=77))
    run("scaled_laplacian5", sparse.scaled_laplacian_2d(5, decades=3.0, seed=8))
    run("wide_row", C(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]),
                      np.array([1.0, 2.0 ** 60, 2.0 ** 60, 1.0])))
    run("missing_diag_inexact", C(3, 3, np.array([0, 2, 3, 4]), np.array([1, 2, 0, 0]),
                                  np.array([2.0 ** 60, 1.0 + 2.0 ** -52, 2.0 ** 60,
                                            1.0 + 2.0 ** -52])))
    run("missing_diag_exact", C(2, 2, np.array([0, 1, 2]), np.array([1, 0]),
                                np.array([2.0, 2.0])))
    run("overflow", C(2, 2, np.array([0, 2, 3]), np.array([0, 1, 1]),
                      np.array([1.7e308, 1.7e308, 1.0])))
    rng = np.random.default_rng(20251013)
    for k, (A, scale) in enumerate([(sparse.laplacian_2d(20), 1.0),
                                    (sparse.random_symmetric(300, seed=3), 1e-3),
                                    (sparse.scaled_laplacian_2d(16, decades=6.0, seed=2), 1e5)]):
        v = A.values * (1.0 + rng.standard_normal(A.values.size) * 1e-3) * scale
        run(f"perturbed{k}", C(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, v))
    for t in range(1500):
        n, rp, ci, va = _tiny(rng)
        run(f"tiny{t}", C(n, n, rp, ci, va))
    # rows whose rounding gap needs b nudged: a big off-diagonal 2^E, a small one
    # (the new diagonal b - off-diagonals spans > 53 bits unless b lands on 2^E) and
    # a diagonal of about k ulps of 2^E, so the nudge that works is k ulps away
    for t in range(400):
        E = int(rng.integers(55, 120))
        ulp = 2.0 ** (E - 52)
        k = int(rng.integers(0, 6))
        sg = -1.0 if rng.random() < 0.5 else 1.0
        d = sg * ulp * (k + float(rng.uniform(-0.4, 0.4)))
        small = float(rng.integers(1, 99) | 1) * 2.0 ** -int(rng.integers(1, 20))
        vals = [d, sg * 2.0 ** E, small, 1.0, 1.0]
        run(f"nudge{t}", C(3, 3, np.array([0, 3, 4, 5]), np.array([0, 1, 2, 1, 2]), np.array(vals)))
    out = os.path.join(HERE, "problemgen.json")
    with open(out, "w") as f:
        json.dump({"cases": cases}, f, separators=(",", ":"))
    errs = sum("error" in c for c in cases)
    nudged = sum(c.get("max_ulp_adjustment", 0) > 0 for c in cases)
    print(f"wrote {out}: {len(cases)} cases, {errs} errors, {nudged} with nudges")


if __name__ == "__main__":
    main()
