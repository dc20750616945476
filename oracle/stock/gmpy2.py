"""TEST INFRASTRUCTURE (not product code): stand-in for the absent third-party
`gmpy2` module, so the STOCK reference package (baseline/_ref, installed from
/root/reference/pkg) can be imported and timed.  The reference uses exactly
one gmpy2 function, fma() at eft.py:36-39 (gmpy2.fma at 53-bit precision =
IEEE binary64 fma, correctly rounded); glibc's fma() is correctly rounded,
so this is the same function.  Its fused-ness is checked by the reference's
own import-time self test (eft.py:42-53)."""
import ctypes
import ctypes.util

_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.fma.restype = ctypes.c_double
_libm.fma.argtypes = [ctypes.c_double] * 3


def fma(a, b, c):
    return _libm.fma(float(a), float(b), float(c))
