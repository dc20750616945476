"""ctypes facade over the C oracle (TEST INFRASTRUCTURE -- not product code).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs
import this module, and only as the checker / the CPU baseline.  The C
restatement lives in ``oracle/mwcg_oracle.c``; every function there cites the
reference file:line it follows.  Parity of the oracle itself is pinned by
``tests/golden`` (vectors produced by the real reference).

Vectors are numpy arrays of shape (w, n) float64 (SoA word planes, the layout
the device uses), matrices are (row_ptr, col_idx, values) int64/int64/f64.
"""

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmwcg_oracle.so")

MODES = ("fp64", "dw", "qdw", "tw", "qtw")
WORDS = {"fp64": 1, "dw": 2, "qdw": 2, "tw": 3, "qtw": 3}
MODE_ID = {m: i for i, m in enumerate(MODES)}
NORM_ID = {"none": 0, "after-axpy": 1, "every-op": 2}
REASONS = {1: "converged", 2: "max_iterations", 3: "breakdown"}

# canonical tile-tree shape shared with the device kernels
TILE_THREADS = 256
TILE_ELEMS = 4

_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)


class _Cfg(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("normalization", ctypes.c_int),
                ("reduction", ctypes.c_int), ("tb", ctypes.c_int), ("e", ctypes.c_int),
                ("record_history", ctypes.c_int), ("epsilon", ctypes.c_double),
                ("max_iterations", ctypes.c_int64), ("history_stride", ctypes.c_int64),
                ("partitions", ctypes.c_int64)]


class _Res(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("reason", ctypes.c_int),
                ("final_rel", ctypes.c_double), ("n_hist", ctypes.c_int64)]


def build():
    """Compile the oracle with its Makefile (gcc; no reference sources)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_sumsq.restype = ctypes.c_double
        L.orc_cg_iterations.restype = ctypes.c_double
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    if a.dtype == np.int64:
        return a.ctypes.data_as(_lp)
    return a.ctypes.data_as(_dp)


def _soa(v, mode):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.ndim == 1:
        v = v.reshape(1, -1)
    assert v.shape[0] == WORDS[mode], (v.shape, mode)
    return v


def _csr(A):
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_idx, dtype=np.int64)
    va = np.ascontiguousarray(A.values, dtype=np.float64)
    return rp, ci, va


def set_threads(t):
    lib().orc_set_threads(int(t))


def max_threads():
    return int(lib().orc_max_threads())


def scalar_op(op, mode, a, b=None):
    ops = {"add": 0, "mul": 1, "dxmul": 2, "dxadd": 3, "normalize": 4, "div": 5,
           "neg": 6, "two_sum": 7, "quick_two_sum": 8, "two_prod": 9, "collapse": 10}
    A = np.zeros(3)
    A[:len(a)] = a
    B = np.zeros(3)
    if b is not None:
        B[:len(b)] = b
    out = np.zeros(3)
    lib().orc_scalar_op(ops[op], MODE_ID[mode], _p(A), _p(B), _p(out))
    return out


def spmv(mode, A, x):
    rp, ci, va = _csr(A)
    x = _soa(x, mode)
    n_rows = rp.size - 1
    y = np.zeros((WORDS[mode], n_rows))
    lib().orc_spmv(MODE_ID[mode], ctypes.c_int64(n_rows), _p(rp), _p(ci), _p(va),
                   _p(x), ctypes.c_int64(x.shape[1]), _p(y))
    return y


def dot(mode, x, y, partitions=1, tile=None):
    """partitions=P reference shape, or tile=(TB, E) for the canonical tree."""
    x, y = _soa(x, mode), _soa(y, mode)
    out = np.zeros(3)
    n = ctypes.c_int64(x.shape[1])
    if tile is not None:
        lib().orc_dot_tile(MODE_ID[mode], n, _p(x), _p(y), int(tile[0]), int(tile[1]), _p(out))
    else:
        lib().orc_dot_partitions(MODE_ID[mode], n, _p(x), _p(y),
                                 ctypes.c_int64(partitions), _p(out))
    return out[:WORDS[mode]]


def tile_partials(mode, x, y, out, tile_off):
    """Canonical per-tile partials of x.y written into out[:, tile_off:...]
    (out: (w, ld) float64, C-contiguous)."""
    x, y = _soa(x, mode), _soa(y, mode)
    assert out.flags.c_contiguous and out.dtype == np.float64
    lib().orc_tile_partials(MODE_ID[mode], ctypes.c_int64(x.shape[1]), _p(x),
                            ctypes.c_int64(x.shape[1]), _p(y), ctypes.c_int64(y.shape[1]),
                            TILE_THREADS, TILE_ELEMS, _p(out), ctypes.c_int64(out.shape[1]),
                            ctypes.c_int64(tile_off))


def reduce_partials(mode, parts):
    parts = _soa(parts, mode)
    out = np.zeros(3)
    lib().orc_reduce_partials(MODE_ID[mode], ctypes.c_int64(parts.shape[1]), _p(parts),
                              TILE_THREADS, _p(out))
    return out[:WORDS[mode]]


def axpy(mode, alpha, x, y):
    x, y = _soa(x, mode), _soa(y, mode).copy()
    a = np.zeros(3)
    a[:WORDS[mode]] = alpha
    lib().orc_axpy(MODE_ID[mode], ctypes.c_int64(x.shape[1]), _p(a), _p(x), _p(y))
    return y


def scal_add(mode, beta, p, r):
    p, r = _soa(p, mode).copy(), _soa(r, mode)
    bb = np.zeros(3)
    bb[:WORDS[mode]] = beta
    lib().orc_scal_add(MODE_ID[mode], ctypes.c_int64(p.shape[1]), _p(bb), _p(p), _p(r))
    return p


def residual(mode, b, q):
    q = _soa(q, mode)
    b = np.ascontiguousarray(b, dtype=np.float64)
    r = np.zeros_like(q)
    lib().orc_residual(MODE_ID[mode], ctypes.c_int64(b.size), _p(b), _p(q), _p(r))
    return r


def normalize(mode, v):
    v = _soa(v, mode).copy()
    lib().orc_normalize(MODE_ID[mode], ctypes.c_int64(v.shape[1]), _p(v))
    return v


def sumsq(v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.ndim == 1:
        v = v.reshape(1, -1)
    return float(lib().orc_sumsq(v.shape[0], ctypes.c_int64(v.shape[1]), _p(v)))


def norm_metrics_tw(mode, A, x, x_star, b, tile=False):
    rp, ci, va = _csr(A)
    x = _soa(x, mode)
    b = np.ascontiguousarray(b, dtype=np.float64)
    xs = None if x_star is None else np.ascontiguousarray(x_star, dtype=np.float64)
    err = ctypes.c_double()
    tr = ctypes.c_double()
    lib().orc_norm_metrics_tw(MODE_ID[mode], 1 if tile else 0, TILE_THREADS, TILE_ELEMS,
                              ctypes.c_int64(b.size), _p(rp), _p(ci), _p(va), _p(x), _p(xs),
                              _p(b), ctypes.byref(err), ctypes.byref(tr))
    e = err.value
    return (None if x_star is None else e), tr.value


@dataclass
class OracleResult:
    converged: bool
    reason: str
    iterations: int
    final_recurrence_residual: float
    x: np.ndarray            # (w, n)
    history: list            # [(k, rel, true_res, err|None)]


def cg_solve(A, b, mode="fp64", epsilon=1e-12, max_iterations=None,
             normalization="after-axpy", history_stride=100, partitions=1,
             reduction="partitions", x0=None, x_star=None, record_history=True,
             hist_cap=100000):
    """Oracle cg_solve (cg.py:78-183).  reduction: 'partitions' | 'tile'."""
    rp, ci, va = _csr(A)
    n = rp.size - 1
    b = np.ascontiguousarray(b, dtype=np.float64)
    w = WORDS[mode]
    cfg = _Cfg(MODE_ID[mode], NORM_ID[normalization], 1 if reduction == "tile" else 0,
               TILE_THREADS, TILE_ELEMS, 1 if record_history else 0, float(epsilon),
               int(max_iterations if max_iterations is not None else 10 * n),
               int(history_stride), int(partitions))
    x = np.zeros((w, n))
    hk = np.zeros(hist_cap, dtype=np.int64)
    hr = np.zeros(hist_cap)
    ht = np.zeros(hist_cap)
    he = np.zeros(hist_cap)
    res = _Res()
    x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
    xsa = None if x_star is None else np.ascontiguousarray(x_star, dtype=np.float64)
    lib().orc_cg_solve(ctypes.byref(cfg), ctypes.c_int64(n), _p(rp), _p(ci), _p(va), _p(b),
                       _p(x0a), _p(xsa), _p(x), ctypes.c_int64(hist_cap), _p(hk), _p(hr),
                       _p(ht), _p(he), ctypes.byref(res))
    m = min(res.n_hist, hist_cap)
    hist = [(int(hk[i]), float(hr[i]), float(ht[i]),
             None if x_star is None else float(he[i])) for i in range(m)]
    return OracleResult(res.reason == 1, REASONS[res.reason], int(res.iterations),
                        float(res.final_rel), x, hist)


def cg_iterations(A, b, mode, iters, partitions=1, reduction="partitions"):
    """Bounded CPU-baseline sample: `iters` unconditional CG iterations."""
    rp, ci, va = _csr(A)
    n = rp.size - 1
    b = np.ascontiguousarray(b, dtype=np.float64)
    cfg = _Cfg(MODE_ID[mode], 1, 1 if reduction == "tile" else 0, TILE_THREADS, TILE_ELEMS,
               0, 1e-300, int(iters), 1 << 62, int(partitions))
    x = np.zeros((WORDS[mode], n))
    return float(lib().orc_cg_iterations(ctypes.byref(cfg), ctypes.c_int64(n), _p(rp), _p(ci),
                                         _p(va), _p(b), ctypes.c_int64(iters), _p(x)))
