"""Helpers to read the committed golden fixtures (tests/golden/*.json)."""
import json
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def fh(s):
    return float.fromhex(s)


def arr(lst):
    return np.array([float.fromhex(v) for v in lst], dtype=np.float64)


def planes(lst_of_lists):
    return np.stack([arr(w) for w in lst_of_lists])


def csr(d):
    return SimpleNamespace(n_rows=d["n"], n_cols=d["n"],
                           row_ptr=np.array(d["row_ptr"], dtype=np.int64),
                           col_idx=np.array(d["col_idx"], dtype=np.int64),
                           values=arr(d["values"]))


def bits(a):
    """Bit patterns, so that -0.0 != 0.0 and NaN payloads compare exactly."""
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def same_bits(a, b):
    """Bitwise equality; NaNs match any NaN (payload/sign of a generated NaN
    is platform-defined: Python's math.nan, x86's default NaN and the GPU's
    canonical NaN all differ, and IEEE 754 leaves it unspecified)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    return np.array_equal(bits(a[~na]), bits(b[~nb]))
