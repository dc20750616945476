"""Device self-verification suites behind ``mwcg verify`` (reference verify.py:1-244).

The reference's suites check its host arithmetic against exact dyadic rationals
(``ExactValue``).  These run the same kinds of checks on the DEVICE code paths,
with ``fractions.Fraction`` as the exact arithmetic:

error_free          two_sum / two_prod on the device are error-free (verify.py:108-129)
precision_floors    DW/QDW/TW/QTW device add/mul within the reference bounds (verify.py:132-164)
normalization       device normalize keeps the value exactly (verify.py:167-190)
problem_generation  generated problems are exactly consistent (verify.py:193-210)
kernel_accuracy     device SpMV / dot in every mode against exact sums
reduction_agreement tile-tree and partition orders agree on a well-conditioned solve
                    (the device analogue of verify.py:213-237's fast == reference check)
"""
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import sparse

__all__ = ["CheckResult", "run_all"]

SEED = 20251013
MODES = ("fp64", "dw", "qdw", "tw", "qtw")
# verify.py:146-153 bounds: 2^-100 (DW), 8 * 2^-100 (QDW), 2^-150 (TW), 8 * 2^-150 (QTW)
_FLOOR_BITS = {"fp64": 52, "dw": 100, "qdw": 97, "tw": 150, "qtw": 147}


@dataclass(frozen=True)
class CheckResult:
    suite: str
    name: str
    passed: bool
    detail: str


def _exact(words):
    return sum((Fraction(float(w)) for w in words), Fraction(0))


def _rel_bits(got, exact, scale=None):
    """-log2 of |got - exact| / |scale or exact| (inf when exact)."""
    err = abs(got - exact)
    ref = abs(exact) if scale is None else scale
    if err == 0:
        return float("inf")
    if ref == 0:
        return float("-inf")
    return float(np.log2(float(ref / err)))


def suite_error_free(n=200):
    from . import eft
    from .multiword import scalar_op
    out = []
    try:  # the reference's import-time fused-fma check (eft.py:42-53), on the device
        eft._check_fused()
        out.append(CheckResult("error_free", "fused_fma", True, "(1+2^-27)^2 error term exact"))
    except eft.FmaUnavailableError as exc:
        out.append(CheckResult("error_free", "fused_fma", False, str(exc)))
    rng = np.random.default_rng(SEED)
    a = rng.standard_normal(n) * np.exp2(rng.integers(-30, 30, n))
    b = rng.standard_normal(n) * np.exp2(rng.integers(-30, 30, n))
    for op, f in (("two_sum", lambda x, y: x + y), ("two_prod", lambda x, y: x * y)):
        bad = 0
        for x, y in zip(a, b):
            s, e, _ = scalar_op(op, "dw", [x], [y])
            bad += Fraction(float(s)) + Fraction(float(e)) != f(Fraction(float(x)), Fraction(float(y)))
        out.append(CheckResult("error_free", op, bad == 0,
                               f"{n} samples exact" if not bad else f"{bad}/{n} inexact"))
    return out


def suite_precision_floors(n=100):
    from .multiword import scalar_op
    rng = np.random.default_rng(SEED + 1)
    out = []
    for mode in ("dw", "qdw", "tw", "qtw"):
        w = 2 if mode in ("dw", "qdw") else 3
        worst = float("inf")
        for _ in range(n):
            xs, ys = [], []
            for v in (xs, ys):
                v.append(float(rng.uniform(1.0, 2.0)))
                for k in range(1, w):
                    v.append(float(np.spacing(v[k - 1]) * rng.uniform(-0.5, 0.5)))
            X, Y = _exact(xs), _exact(ys)
            for op, ex in (("add", X + Y), ("mul", X * Y)):
                got = _exact(scalar_op(op, mode, xs, ys)[:w])
                worst = min(worst, _rel_bits(got, ex))
        floor = _FLOOR_BITS[mode]
        out.append(CheckResult("precision_floors", mode, worst >= floor,
                               f"worst {worst:.1f} bits (floor {floor})"))
    return out


def suite_normalization(n=100):
    from .multiword import scalar_op
    rng = np.random.default_rng(SEED + 2)
    hi = rng.standard_normal(n) * np.exp2(rng.integers(-20, 20, n))
    lo = rng.standard_normal(n) * np.abs(hi) * rng.uniform(0, 2.0 ** -40, n)
    out = []
    # normalize_dw / normalize_tw (multiword.py:330-357) are the quasi renormalisations
    for name, mode, w in (("dw", "qdw", 2), ("tw", "qtw", 3)):
        bad = 0
        for h, l in zip(hi, lo):
            a = [float(h), float(l), float(l) * 2.0 ** -30][:w]
            bad += _exact(scalar_op("normalize", mode, a)[:w]) != _exact(a)
        out.append(CheckResult("normalization", f"normalize_{name}", bad == 0,
                               f"{bad}/{n} value changes"))
    return out


def suite_problem_generation():
    from .problemgen import generate
    out = []
    for name, A in (("laplacian_2d(8)", sparse.laplacian_2d(8)),
                    ("random_symmetric(60)", sparse.random_symmetric(60, seed=5))):
        p = generate(A)
        m, bad = p.matrix, None
        for i in range(m.n_rows):
            if _exact(m.values[m.row_ptr[i]:m.row_ptr[i + 1]]) != Fraction(float(p.b[i])):
                bad = i
                break
        out.append(CheckResult("problem_generation", name, bad is None,
                               "exact residual zero" if bad is None else f"row {bad} inexact"))
    return out


def suite_kernel_accuracy():
    from . import kernels as kn
    rng = np.random.default_rng(SEED + 3)
    A = sparse.laplacian_2d(5)
    n = A.n_rows
    out = []
    for mode in MODES:
        w = kn.mode_words(mode)
        planes = np.zeros((w, n))
        planes[0] = rng.standard_normal(n)
        for k in range(1, w):
            planes[k] = np.spacing(planes[k - 1]) * rng.uniform(-0.5, 0.5, n)
        x = kn.MultiwordVector.from_planes(planes, mode)
        xe = [_exact(planes[:, j]) for j in range(n)]
        y = kn.spmv(A, x).to_host()
        worst = float("inf")
        for i in range(n):
            lo, hi = A.row_ptr[i], A.row_ptr[i + 1]
            terms = [Fraction(float(A.values[k])) * xe[A.col_idx[k]] for k in range(lo, hi)]
            worst = min(worst, _rel_bits(_exact(y[:, i]), sum(terms), sum(abs(t) for t in terms)))
        d = kn.dot(x, x, partitions=3)
        dw = d if isinstance(d, (tuple, list, np.ndarray)) else [d]
        worst = min(worst, _rel_bits(_exact(list(dw)[:w]), sum(v * v for v in xe)))
        floor = _FLOOR_BITS[mode] - 8  # n-term sums lose up to log2(n) bits
        out.append(CheckResult("kernel_accuracy", mode, worst >= floor,
                               f"spmv/dot worst {worst:.1f} bits (floor {floor})"))
    return out


def suite_reduction_agreement():
    from . import cg
    from .problemgen import generate
    p = generate(sparse.laplacian_2d(8))
    out = []
    for mode in MODES:
        its = []
        for red in ("tile", "partitions"):
            cfg = cg.SolverConfig(mode=mode, epsilon=1e-12, reduction=red, partitions=3)
            r = cg.cg_solve(p.matrix, p.b, cfg, x_star=p.x_star)
            its.append((r.converged, r.iterations, r.history[-1].error_norm))
        ok = its[0][0] and its[1][0] and its[0][1] == its[1][1] and \
            max(its[0][2], its[1][2]) < 1e-10
        out.append(CheckResult("reduction_agreement", mode, ok,
                               f"iterations tile {its[0][1]} / partitions {its[1][1]}, "
                               f"error {its[0][2]:.2e} / {its[1][2]:.2e}"))
    return out


SUITES = (suite_error_free, suite_precision_floors, suite_normalization, suite_problem_generation,
          suite_kernel_accuracy, suite_reduction_agreement)


def run_all():
    out = []
    for suite in SUITES:
        out.extend(suite())
    return out
