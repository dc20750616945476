"""Device vectors and the operator-level API (reference kernels.py:17-328).

`MultiwordVector` keeps its words as a (w, n) float64 CUDA tensor of
structure-of-arrays word planes (the reference uses an AoS numpy record
array, kernels.py:39-40; the per-word values are identical).  Every kernel
here calls libmwcg_cuda.so; there is no host fallback.

Reduction shape: `dot(x, y, partitions=P)` with P >= 1 reproduces the
reference's partitioned sequential order exactly (kernels.py:158-162,
_fast.py:342-356); `partitions=0` selects the device tile tree (the order the
fused CG uses).
"""
import ctypes
import warnings
import weakref

import numpy as np
import torch

from . import _lib
from .multiword import DoubleWord, TripleWord

__all__ = ["MODES", "MultiwordVector", "mode_words", "spmv", "dot", "axpy", "scal_then_add",
           "residual", "normalize_vector", "norm2_fp64", "norm_metrics_tw", "scalar_one",
           "scalar_neg", "scalar_div", "scalar_to_fp64", "device_matrix"]

MODES = _lib.MODES


def mode_words(mode):
    if mode not in _lib.WORDS:
        raise ValueError(f"unknown arithmetic mode {mode!r}")
    return _lib.WORDS[mode]


def _cuda():
    if not torch.cuda.is_available():
        raise _lib.MwcgError("no CUDA device: the mwcg B200 path has no CPU fallback")
    return torch.device("cuda")


class MultiwordVector:
    """Fixed-length vector of FP64 / double-word / triple-word elements on the GPU."""

    def __init__(self, mode, length, planes=None):
        w = mode_words(mode)
        self.mode = mode
        if planes is None:
            planes = torch.zeros((w, int(length)), dtype=torch.float64, device=_cuda())
        assert planes.shape == (w, int(length)) and planes.dtype == torch.float64
        self.planes = planes

    @classmethod
    def from_fp64(cls, values, mode):
        v = np.ascontiguousarray(values, dtype=np.float64)
        out = cls(mode, v.size)
        out.planes[0].copy_(torch.from_numpy(v))
        return out

    @classmethod
    def from_planes(cls, planes, mode):
        """planes: (w, n) array-like of FP64 words (host or device)."""
        t = torch.as_tensor(np.ascontiguousarray(planes, dtype=np.float64)) \
            if not isinstance(planes, torch.Tensor) else planes
        t = t.to(device=_cuda(), dtype=torch.float64).contiguous()
        if t.ndim == 1:
            t = t.reshape(1, -1)
        return cls(mode, t.shape[1], t)

    def to_host(self):
        """(w, n) host copy of the word planes through a pinned buffer."""
        h = torch.empty(tuple(self.planes.shape), dtype=torch.float64, pin_memory=True)
        h.copy_(self.planes, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return h.numpy()

    @property
    def words(self):
        """Host snapshot of the word planes, w0 highest (kernels.py:69-74)."""
        h = self.to_host()
        return tuple(h[k] for k in range(h.shape[0]))

    def __len__(self):
        return int(self.planes.shape[1])

    def to_fp64(self):
        """Collapse each element high to low (kernels.py:79-85)."""
        ws = self.words
        out = ws[0].copy()
        for w in ws[1:]:
            out += w
        return out

    def copy(self):
        return MultiwordVector(self.mode, len(self), self.planes.clone())

    def element(self, i):
        col = self.planes[:, i].cpu().numpy()
        if self.mode == "fp64":
            return float(col[0])
        if col.size == 2:
            return DoubleWord(float(col[0]), float(col[1]))
        return TripleWord(*(float(c) for c in col))

    def set_element(self, i, value):
        vals = [value] if self.mode == "fp64" else list(value)
        self.planes[:, i] = torch.tensor(vals, dtype=torch.float64)

    def promote_tw(self):
        v = MultiwordVector("tw", len(self))
        v.planes[:self.planes.shape[0]].copy_(self.planes)
        return v


# ---------------------------------------------------------------- matrices
def device_matrix(A, row_base=0, col_format=-1, col_block=-1):
    """SELL-32 device copy of a CsrMatrix, built once and cached on A.
    row_base: global index of row 0 when A holds a rank's rows with global
    columns (dist.py); col_format: -1 auto / 0 int32 / 1 int16 deltas /
    2 slice-shared offsets, optionally | _lib.SELL_SIGMA / _lib.SELL_NO_SIGMA /
    _lib.DIA_STREAM_VALUES ("auto" is 15 with a flag) (include/mwcg_cuda.h).
    col_block: columns per column block of an irregular (int32-SELL) matrix
    (-1 automatic, 0 none)."""
    h = getattr(A, "_device", None)
    if h is not None:
        return h
    L = _lib.load()
    dev = _cuda()
    if isinstance(A.row_ptr, torch.Tensor):  # DeviceCsrMatrix: arrays already on the GPU
        rp, ci, va = A.row_ptr, A.col_idx, A.values
        ib = rp.element_size()
    else:
        # non_blocking: a DMA straight from the caller's buffers when they are
        # pinned (torch checks); pageable buffers fall back to a staged copy
        # (CsrMatrix arrays are read-only views; torch only reads them here)
        with warnings.catch_warnings():
            warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
            rp = torch.from_numpy(np.ascontiguousarray(A.row_ptr, dtype=np.int64)).to(dev, non_blocking=True)
            ci = torch.from_numpy(np.ascontiguousarray(A.col_idx, dtype=np.int64)).to(dev, non_blocking=True)
            va = torch.from_numpy(np.ascontiguousarray(A.values, dtype=np.float64)).to(dev, non_blocking=True)
        ib = 8
    handle = ctypes.c_void_p()
    _lib.check(L.mwcg_matrix_create_blocked(ctypes.byref(handle), A.n_rows, A.n_cols, A.nnz,
                                            _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(va), ib, int(row_base),
                                            int(col_format), int(col_block), _lib.stream_handle()))
    dm = _DeviceMatrix(handle, A.n_rows, A.n_cols, A.nnz)
    try:
        object.__setattr__(A, "_device", dm)
    except AttributeError:  # pragma: no cover - foreign matrix types
        pass
    return dm


class _DeviceMatrix:
    def __init__(self, handle, n_rows, n_cols, nnz):
        self.handle = handle
        self.n_rows, self.n_cols, self.nnz = n_rows, n_cols, nnz
        self._fin = weakref.finalize(self, _lib.load().mwcg_matrix_destroy, handle)

    def col_bytes(self):
        return int(_lib.load().mwcg_matrix_col_bytes(self.handle))

    def sigma_sorted(self):
        """True when the SELL rows of each tile are stored length-sorted."""
        return bool(_lib.load().mwcg_matrix_sigma_sorted(self.handle))

    def padded_entries(self):
        out = ctypes.c_int64()
        _lib.check(_lib.load().mwcg_matrix_info(self.handle, None, None, None, ctypes.byref(out)))
        return out.value

    def col_blocks(self):
        """Number of column blocks K1 walks (0: the matrix is not blocked)."""
        return int(_lib.load().mwcg_matrix_col_blocks(self.handle))

    def block_columns(self):
        """Columns per column block (0: not blocked)."""
        return int(_lib.load().mwcg_matrix_block_columns(self.handle))

    def stored_values(self):
        """Value entries the layout stores and streams per SpMV (value-uniform
        slices of the slice-shared layout store none)."""
        return int(_lib.load().mwcg_matrix_stored_values(self.handle))


# ---------------------------------------------------------------- scalars
def scalar_one(mode):
    w = mode_words(mode)
    return 1.0 if w == 1 else (DoubleWord(1.0, 0.0) if w == 2 else TripleWord(1.0, 0.0, 0.0))


def scalar_neg(mode, a):
    if mode == "fp64":
        return -a
    return DoubleWord(-a.w0, -a.w1) if mode_words(mode) == 2 else TripleWord(-a.w0, -a.w1, -a.w2)


def _as_words(mode, a):
    return [float(a)] if mode == "fp64" else [float(v) for v in a]


def _from_words(mode, ws):
    w = mode_words(mode)
    if w == 1:
        return float(ws[0])
    return DoubleWord(float(ws[0]), float(ws[1])) if w == 2 else TripleWord(*map(float, ws[:3]))


def scalar_div(mode, a, b):
    """alpha/beta division on the device (dw_div / tw_div, multiword.py:370-409)."""
    from .multiword import scalar_op
    return _from_words(mode, scalar_op("div", mode, _as_words(mode, a), _as_words(mode, b)))


def scalar_to_fp64(mode, a):
    if mode == "fp64":
        return a
    return a.w0 + a.w1 if mode_words(mode) == 2 else (a.w0 + a.w1) + a.w2


def _check_len(a, b):
    if len(a) != len(b):
        raise ValueError(f"length mismatch: {len(a)} vs {len(b)}")


# ---------------------------------------------------------------- kernels
def spmv(A, x, out=None, reference=False):
    """y = A x in the vector's arithmetic (kernels.py:174-197)."""
    if A.n_cols != len(x):
        raise ValueError(f"dimension mismatch: matrix has {A.n_cols} columns, "
                         f"vector has {len(x)} elements")
    if out is None:
        out = MultiwordVector(x.mode, A.n_rows)
    dm = device_matrix(A)
    L = _lib.load()
    _lib.check(L.mwcg_spmv(_lib.MODE_ID[x.mode], dm.handle, _lib.ptr(x.planes), len(x),
                           _lib.ptr(out.planes), len(out), _lib.stream_handle()))
    return out


def dot(x, y, partitions=1, reference=False):
    """Sum of products in the mode's arithmetic (kernels.py:200-223).
    partitions >= 1: the reference order; 0: the device tile tree."""
    _check_len(x, y)
    if x.mode != y.mode:
        raise ValueError("dot operands must share a mode")
    if partitions < 0:
        raise ValueError("partition count must be >= 1")
    L = _lib.load()
    n = len(x)
    work = torch.zeros(int(L.mwcg_dot_work_bytes(n, partitions)) // 8 + 1, dtype=torch.float64,
                       device=_cuda())
    out = torch.zeros(3, dtype=torch.float64, device=_cuda())
    _lib.check(L.mwcg_dot(_lib.MODE_ID[x.mode], n, _lib.ptr(x.planes), n, _lib.ptr(y.planes), n,
                          int(partitions), _lib.ptr(out), _lib.ptr(work), _lib.stream_handle()))
    return _from_words(x.mode, out.cpu().numpy())


def axpy(alpha, x, y, reference=False):
    """y <- y + alpha x (kernels.py:226-238)."""
    _check_len(x, y)
    a = (ctypes.c_double * 3)(*(_as_words(x.mode, alpha) + [0.0, 0.0])[:3])
    _lib.check(_lib.load().mwcg_axpy(_lib.MODE_ID[x.mode], len(x), a, _lib.ptr(x.planes), len(x),
                                     _lib.ptr(y.planes), len(y), _lib.stream_handle()))
    return y


def scal_then_add(beta, p, r, reference=False):
    """p <- r + beta p (kernels.py:241-253)."""
    _check_len(p, r)
    bb = (ctypes.c_double * 3)(*(_as_words(p.mode, beta) + [0.0, 0.0])[:3])
    _lib.check(_lib.load().mwcg_scal_add(_lib.MODE_ID[p.mode], len(p), bb, _lib.ptr(p.planes),
                                         len(p), _lib.ptr(r.planes), len(r), _lib.stream_handle()))
    return p


def residual(b, q, out=None, reference=False):
    """r = b - q for an FP64 b (kernels.py:256-270)."""
    bt = b if isinstance(b, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(b, dtype=np.float64))
    bt = bt.to(_cuda(), torch.float64).contiguous()
    if bt.numel() != len(q):
        raise ValueError("dimension mismatch in residual")
    if out is None:
        out = MultiwordVector(q.mode, len(q))
    _lib.check(_lib.load().mwcg_residual(_lib.MODE_ID[q.mode], len(q), _lib.ptr(bt),
                                         _lib.ptr(q.planes), len(q), _lib.ptr(out.planes), len(out),
                                         _lib.stream_handle()))
    return out


def normalize_vector(v, reference=False):
    """QuickTwoSum/TwoSum (qdw) or VecSum3 (qtw) per element; no-op otherwise."""
    if v.mode not in ("qdw", "qtw"):
        return v
    _lib.check(_lib.load().mwcg_normalize(_lib.MODE_ID[v.mode], len(v), _lib.ptr(v.planes),
                                          len(v), _lib.stream_handle()))
    return v


def norm2_fp64(x):
    """FP64 2-norm of the collapsed vector, sequential accumulation
    (kernels.py:290-296)."""
    if isinstance(x, MultiwordVector):
        c = x.to_fp64() if x.mode != "fp64" else x.words[0]
        # collapsed words: the reference squares (w0+w1)+w2 per element
        v = np.ascontiguousarray(c, dtype=np.float64)
    else:
        v = np.ascontiguousarray(x, dtype=np.float64)
    out = ctypes.c_double()
    _lib.check(_lib.load().mwcg_norm2_host(v.ctypes.data_as(_lib.c_dp), v.size, ctypes.byref(out)))
    return out.value


def norm_metrics_tw(x, x_star, A, b):
    """Relative error and true residual in TW arithmetic (kernels.py:305-328),
    sequential TW sums (partitions=1) exactly like the reference."""
    if A.n_cols != len(x):
        raise ValueError("dimension mismatch in norm metrics")
    xt = x.promote_tw()
    b = np.ascontiguousarray(b, dtype=np.float64)
    q = spmv(A, xt)
    res = residual(b, q)

    def nsq(v):
        s = dot(v, v, partitions=1)
        return (s.w0 + s.w1) + s.w2

    bn = nsq(MultiwordVector.from_fp64(b, "tw")) or 1.0
    true_res = float(np.sqrt(nsq(res) / bn))
    err = None
    if x_star is not None:
        xs = np.ascontiguousarray(x_star, dtype=np.float64)
        diff = residual(xs, xt)
        xn = nsq(MultiwordVector.from_fp64(xs, "tw")) or 1.0
        err = float(np.sqrt(nsq(diff) / xn))
    return err, true_res
