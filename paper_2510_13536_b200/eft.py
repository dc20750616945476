"""Error-free transformations (reference eft.py:1-130) on the device.

Same names and results as the reference: `two_sum`, `quick_two_sum`,
`two_prod_fma` return `Fp64Pair(hi, lo)`; `fma` is one correctly rounded fused
multiply-add.  Each call is one launch of the device op the kernels inline
(csrc/mw.cuh, built with -fmad=false and explicit __fma_rn).  The reference's
import-time check that fma is truly fused (eft.py:42-53) runs here on the
device at the first fma / two_prod_fma call (no GPU is touched at import).
"""
from typing import NamedTuple

__all__ = ["U", "Fp64Pair", "FmaUnavailableError", "fma", "two_sum", "quick_two_sum",
           "two_prod_fma"]

# unit round-off for FP64 with round-to-nearest
U = 2.0 ** -53


class FmaUnavailableError(RuntimeError):
    """Raised when the device fma is not a single-rounding fused multiply-add."""


class Fp64Pair(NamedTuple):
    """Rounded result plus its exact rounding error (hi + lo is exact)."""
    hi: float
    lo: float


_fused_ok = False


def _op(op, a, b, c=0.0):
    from .multiword import scalar_op
    r = scalar_op(op, "dw", [float(a), float(c)], [float(b)])
    return float(r[0]), float(r[1])


def _check_fused():
    # (1 + 2^-27)^2 = 1 + 2^-26 + 2^-54: the error term survives only if fused
    global _fused_ok
    if _fused_ok:
        return
    a = 1.0 + 2.0 ** -27
    if _op("fma", a, a, -(a * a))[0] != 2.0 ** -54:
        raise FmaUnavailableError("device fma is not a single-rounding fused multiply-add; "
                                  "two_prod_fma would silently lose its error term")
    _fused_ok = True


def fma(a, b, c):
    """Fused a*b + c with a single rounding (eft.py:56-68)."""
    _check_fused()
    return _op("fma", a, b, c)[0]


def two_sum(a, b):
    """hi = fl(a+b), hi + lo = a + b exactly (eft.py:78-88)."""
    return Fp64Pair(*_op("two_sum", a, b))


def quick_two_sum(a, b):
    """Error-free sum assuming |a| >= |b| (eft.py:92-117)."""
    return Fp64Pair(*_op("quick_two_sum", a, b))


def two_prod_fma(a, b):
    """hi = fl(a*b), hi + lo = a * b exactly (eft.py:120-130)."""
    _check_fused()
    return Fp64Pair(*_op("two_prod", a, b))
