"""Test problems whose exact solution is known by construction (reference
problemgen.py:1-108), generated natively.

`generate(A)` chooses the all-ones solution, rounds each exact row sum to FP64 for
b, and absorbs the rounding gap into the diagonal (nudging b_i by up to 4 ulps until
the new diagonal is representable).  The exact row sums run in
`libmwcg_cuda.so:mwcg_problem_generate` (csrc/problemgen.cu: fixed-point exact
accumulators over host threads) instead of the reference's pure-Python
`ExactValue` loop (its exact-arithmetic module, lines 35-128), which is
infeasible beyond ~1e5 nonzeros.
Results, error messages and the error row are the reference's.
"""
import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .sparse import CsrMatrix

__all__ = ["GeneratedProblem", "generate"]


@dataclass(frozen=True)
class GeneratedProblem:
    """problemgen.py:26-32."""
    matrix: CsrMatrix
    b: np.ndarray
    x_star: np.ndarray
    perturbation_norm: float     # FP64 2-norm of the diagonal perturbations
    max_ulp_adjustment: int      # largest right-hand-side nudge used


def generate(A, x_star=None, threads=0):
    """Build an exactly consistent problem from ``A`` with solution ones
    (problemgen.py:47-108).  ``threads``: host threads for the row sums (0 = all)."""
    if A.n_rows != A.n_cols:
        raise ValueError("matrix must be square")
    if x_star is not None:
        xs = np.asarray(x_star, dtype=np.float64)
        if xs.shape != (A.n_cols,) or not np.all(xs == 1.0):
            raise ValueError("only the all-ones solution vector is supported")
    n = A.n_rows
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_idx, dtype=np.int64)
    va = np.ascontiguousarray(A.values, dtype=np.float64)
    values = np.empty_like(va)
    b = np.empty(n)
    deltas = np.zeros(n)
    mx = ctypes.c_int64(0)
    L = _lib.load()
    _lib.check(L.mwcg_problem_generate(n, rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
                                       values.ctypes.data, b.ctypes.data, deltas.ctypes.data,
                                       ctypes.byref(mx), int(threads)))
    matrix = CsrMatrix(A.n_rows, A.n_cols, rp.copy(), ci.copy(), values)
    return GeneratedProblem(
        matrix=matrix, b=b, x_star=np.ones(n),
        perturbation_norm=float(np.sqrt(np.sum(deltas * deltas))),
        max_ulp_adjustment=int(mx.value))
