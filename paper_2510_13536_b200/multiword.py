"""Multi-word scalar value types (multiword.py:34-73 of the reference).

Only the value containers live on the host; all multi-word ARITHMETIC runs
on the device (csrc/mw.cuh).  `scalar_op` exposes the device ops one at a
time for the API and for unit parity tests.
"""
from fractions import Fraction
from typing import NamedTuple

import numpy as np


def _decimal_str(words, digits):
    """Exact value of sum(words) in decimal, round-half-even to `digits`
    significant digits (the reference's ExactValue.decimal_str, its exact-
    arithmetic module lines 165-188)."""
    v = sum((Fraction(float(w)) for w in words), Fraction(0))
    if v == 0:
        return "0"
    f, exp10 = abs(v), 0
    while f >= 10:
        f /= 10
        exp10 += 1
    while f < 1:
        f *= 10
        exp10 -= 1
    scaled = f * Fraction(10) ** (digits - 1)
    q, r = divmod(scaled.numerator, scaled.denominator)
    if 2 * r > scaled.denominator or (2 * r == scaled.denominator and q % 2 == 1):
        q += 1
    s = str(q)
    if len(s) > digits:  # rounding carried into a new leading digit
        s = s[:digits]
        exp10 += 1
    body = f"{s[0]}.{s[1:]}" if digits > 1 else s
    return f"{'-' if v < 0 else ''}{body}e{exp10:+d}"

__all__ = [
    "DoubleWord", "TripleWord", "scalar_op",
    "dw_add", "dw_mul", "dw_neg", "dw_sub", "dw_div",
    "qdw_add", "qdw_mul", "qdw_div",
    "tw_add", "tw_mul", "tw_neg", "tw_sub", "tw_div",
    "qtw_add", "qtw_mul", "qtw_div",
    "dxdw_add", "dxdw_mul", "dxqdw_add", "dxqdw_mul",
    "dxtw_add", "dxtw_mul", "dxqtw_add", "dxqtw_mul",
    "normalize_dw", "normalize_tw",
    "dw_from_fp64", "tw_from_fp64", "dw_to_fp64", "tw_to_fp64",
]


class DoubleWord(NamedTuple):
    w0: float
    w1: float

    def to_hex(self):
        return f"{self.w0.hex()} {self.w1.hex()}"

    @classmethod
    def from_hex(cls, text):
        a, b = text.split()
        return cls(float.fromhex(a), float.fromhex(b))

    def decimal_str(self, digits=40):
        return _decimal_str(self, digits)


class TripleWord(NamedTuple):
    w0: float
    w1: float
    w2: float

    def to_hex(self):
        return f"{self.w0.hex()} {self.w1.hex()} {self.w2.hex()}"

    @classmethod
    def from_hex(cls, text):
        a, b, c = text.split()
        return cls(float.fromhex(a), float.fromhex(b), float.fromhex(c))

    def decimal_str(self, digits=60):
        return _decimal_str(self, digits)


def dw_to_fp64(a):
    return a.w0 + a.w1


def tw_to_fp64(a):
    return (a.w0 + a.w1) + a.w2


OPS = {"add": 0, "mul": 1, "dxmul": 2, "dxadd": 3, "normalize": 4, "div": 5, "neg": 6,
       "two_sum": 7, "quick_two_sum": 8, "two_prod": 9, "collapse": 10, "fma": 11}


def scalar_op(op, mode, a, b=None):
    """Run one multi-word scalar op on the device; returns 3 floats."""
    import torch
    from . import _lib
    L = _lib.load()
    dev = torch.device("cuda")
    A = torch.zeros(3, dtype=torch.float64)
    A[:len(a)] = torch.tensor(np.asarray(a, dtype=np.float64))
    B = torch.zeros(3, dtype=torch.float64)
    if b is not None:
        B[:len(b)] = torch.tensor(np.asarray(b, dtype=np.float64))
    A, B = A.to(dev), B.to(dev)
    out = torch.zeros(3, dtype=torch.float64, device=dev)
    _lib.check(L.mwcg_scalar_op(OPS[op], _lib.MODE_ID[mode], _lib.ptr(A), _lib.ptr(B),
                                _lib.ptr(out), _lib.stream_handle()))
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# The reference's scalar API (multiword.py:18-409), each op one device launch
# of the same arithmetic the kernels use (csrc/mw.cuh); results are
# DoubleWord / TripleWord values.
# ---------------------------------------------------------------------------

def _run(op, mode, a, b=None):
    w = 2 if mode in ("dw", "qdw") else 3
    r = scalar_op(op, mode, a, b)
    return DoubleWord(float(r[0]), float(r[1])) if w == 2 else TripleWord(*map(float, r[:3]))


def dw_from_fp64(x):
    return DoubleWord(float(x), 0.0)


def tw_from_fp64(x):
    return TripleWord(float(x), 0.0, 0.0)


def dw_add(a, b): return _run("add", "dw", a, b)           # noqa: E704
def dw_mul(a, b): return _run("mul", "dw", a, b)           # noqa: E704
def dw_neg(a): return _run("neg", "dw", a)                 # noqa: E704
def dw_sub(a, b): return dw_add(a, dw_neg(b))              # noqa: E704  (multiword.py:135-136)
def dw_div(a, b): return _run("div", "dw", a, b)           # noqa: E704
def qdw_add(a, b): return _run("add", "qdw", a, b)         # noqa: E704
def qdw_mul(a, b): return _run("mul", "qdw", a, b)         # noqa: E704
def tw_add(a, b): return _run("add", "tw", a, b)           # noqa: E704
def tw_mul(a, b): return _run("mul", "tw", a, b)           # noqa: E704
def tw_neg(a): return _run("neg", "tw", a)                 # noqa: E704
def tw_sub(a, b): return tw_add(a, tw_neg(b))              # noqa: E704  (multiword.py:259-260)
def tw_div(a, b): return _run("div", "tw", a, b)           # noqa: E704
def qtw_add(a, b): return _run("add", "qtw", a, b)         # noqa: E704
def qtw_mul(a, b): return _run("mul", "qtw", a, b)         # noqa: E704
def dxdw_add(a, b): return _run("dxadd", "dw", [a], b)     # noqa: E704
def dxdw_mul(a, b): return _run("dxmul", "dw", [a], b)     # noqa: E704
def dxqdw_add(a, b): return _run("dxadd", "qdw", [a], b)   # noqa: E704
def dxqdw_mul(a, b): return _run("dxmul", "qdw", [a], b)   # noqa: E704
def dxtw_add(a, b): return _run("dxadd", "tw", [a], b)     # noqa: E704
def dxtw_mul(a, b): return _run("dxmul", "tw", [a], b)     # noqa: E704
def dxqtw_add(a, b): return _run("dxadd", "qtw", [a], b)   # noqa: E704
def dxqtw_mul(a, b): return _run("dxmul", "qtw", [a], b)   # noqa: E704
# normalize_dw is the QuickTwoSum/TwoSum renormalisation of the quasi kernels
# (_fast.py:121-126); normalize_tw the VecSum renormalisation (_fast.py:129-133)
def normalize_dw(a): return _run("normalize", "qdw", a)    # noqa: E704
def normalize_tw(a): return _run("normalize", "qtw", a)    # noqa: E704


# the quasi modes reuse the normalized divisions (multiword.py:405-409)
qdw_div = dw_div
qtw_div = tw_div
