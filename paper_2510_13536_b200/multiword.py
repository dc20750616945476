"""Multi-word scalar value types (multiword.py:34-73 of the reference).

Only the value containers live on the host; all multi-word ARITHMETIC runs
on the device (csrc/mw.cuh).  `scalar_op` exposes the device ops one at a
time for the API and for unit parity tests.
"""
from typing import NamedTuple

import numpy as np

__all__ = ["DoubleWord", "TripleWord", "scalar_op", "dw_to_fp64", "tw_to_fp64"]


class DoubleWord(NamedTuple):
    w0: float
    w1: float

    def to_hex(self):
        return f"{self.w0.hex()} {self.w1.hex()}"

    @classmethod
    def from_hex(cls, text):
        a, b = text.split()
        return cls(float.fromhex(a), float.fromhex(b))


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


def dw_to_fp64(a):
    return a.w0 + a.w1


def tw_to_fp64(a):
    return (a.w0 + a.w1) + a.w2


OPS = {"add": 0, "mul": 1, "dxmul": 2, "dxadd": 3, "normalize": 4, "div": 5, "neg": 6,
       "two_sum": 7, "quick_two_sum": 8, "two_prod": 9, "collapse": 10}


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
