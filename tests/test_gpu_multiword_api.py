"""The reference's scalar multi-word API (multiword.py:18-409) on the device:
every named op against the golden vectors the real reference produced
(tests/golden/ops.json; same cases as test_gpu_parity.test_scalar_ops_golden)."""
import numpy as np
import pytest

from paper_2510_13536_b200 import multiword as mw
from tests.golden_io import arr, load, same_bits

OPS = load("ops.json")
NAMES = {
    "dw": ("dw_add", "dw_mul", "dxdw_mul", "dxdw_add", "normalize_dw", "dw_div"),
    "qdw": ("qdw_add", "qdw_mul", "dxqdw_mul", "dxqdw_add", "normalize_dw", "qdw_div"),
    "tw": ("tw_add", "tw_mul", "dxtw_mul", "dxtw_add", "normalize_tw", "tw_div"),
    "qtw": ("qtw_add", "qtw_mul", "dxqtw_mul", "dxqtw_add", "normalize_tw", "qtw_div"),
}
KEYS = ("add", "mul", "dxmul", "dxadd", "normalize", "div")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["dw", "qdw", "tw", "qtw"])
def test_named_ops_golden(mode):
    w = 2 if mode in ("dw", "qdw") else 3
    cls = mw.DoubleWord if w == 2 else mw.TripleWord
    n = 0
    for c in (c for c in OPS["ops"] if c["mode"] == mode):
        a, b = cls(*arr(c["a"])[:w]), cls(*arr(c["b"])[:w])
        for key, name in zip(KEYS, NAMES[mode]):
            if key not in c:
                continue
            f = getattr(mw, name)
            if key.startswith("dx"):
                got = f(float(a[0]), b)
            elif key == "normalize":
                got = f(a)
            else:
                got = f(a, b)
            assert isinstance(got, cls)
            assert same_bits(np.array(got), arr(c[key])), (mode, name, c["a"], c["b"])
            n += 1
    assert n > 100


@pytest.mark.gpu
def test_neg_sub_and_conversions():
    a = mw.DoubleWord(1.5, 2.0 ** -60)
    b = mw.DoubleWord(0.25, -(2.0 ** -70))
    assert mw.dw_neg(a) == (-1.5, -(2.0 ** -60))
    assert mw.dw_sub(a, b) == mw.dw_add(a, mw.DoubleWord(-0.25, 2.0 ** -70))
    t = mw.TripleWord(1.0, 2.0 ** -60, 2.0 ** -120)
    assert mw.tw_sub(t, t) == mw.tw_add(t, mw.tw_neg(t))
    assert mw.dw_from_fp64(3.0) == (3.0, 0.0) and mw.tw_from_fp64(3.0) == (3.0, 0.0, 0.0)
    assert mw.dw_to_fp64(a) == 1.5 + 2.0 ** -60
    assert mw.qdw_div is mw.dw_div and mw.qtw_div is mw.tw_div


@pytest.mark.gpu
def test_eft_api_golden():
    """eft.two_sum / quick_two_sum / two_prod_fma against the reference's vectors;
    eft.fma against glibc's correctly rounded fma (the gmpy2 stand-in)."""
    import ctypes
    import ctypes.util
    from paper_2510_13536_b200 import eft
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.fma.restype = ctypes.c_double
    libm.fma.argtypes = [ctypes.c_double] * 3
    for c in OPS["eft"][:80]:
        a, b = float.fromhex(c["a"]), float.fromhex(c["b"])
        for name, key in (("two_sum", "two_sum"), ("quick_two_sum", "quick_two_sum"),
                          ("two_prod_fma", "two_prod")):
            got = getattr(eft, name)(a, b)
            assert isinstance(got, eft.Fp64Pair)
            assert same_bits(np.array(got), arr(c[key])), (name, c["a"], c["b"])
        assert same_bits([eft.fma(a, b, -a * b)], [libm.fma(a, b, -a * b)])
    a = 1.0 + 2.0 ** -27
    assert eft.fma(a, a, -(a * a)) == 2.0 ** -54
