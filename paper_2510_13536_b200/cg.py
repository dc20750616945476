"""Conjugate Gradient in a selectable multi-word arithmetic, on a B200.

Drop-in for the reference solver API (cg.py:23-183): `cg_solve(A, b,
config, x0, x_star, reference)`, `SolverConfig`, `SolverResult`,
`ConvergenceRecord`, `Normalization`, with the same validation errors,
stopping test, breakdown rules, history records and result fields.

The iteration runs entirely on the device (csrc/cg.cu): three fused kernels
per iteration inside a CUDA-graph WHILE loop; the host only wakes up at
history records (every `history_stride` iterations) and at the end.

Two extra config fields (both optional, defaults keep the fast path):
  reduction  "tile"       -- canonical device tile-tree dot products
             "partitions" -- the reference's own P-partition order; the
                             solve is then bitwise identical to the
                             reference's cg_solve(..., partitions=P)
  timing     "graph"      -- whole segments as one graph launch
             "kernels"    -- kernel-by-kernel with CUDA events; fills
                             kernel_seconds per fused stage
`reference=True` forces reduction="partitions" (the reference's operation
order, still executed on the GPU).
"""
import ctypes
import time
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional

import numpy as np
import torch

from . import _lib
from .kernels import MODES, MultiwordVector, device_matrix, mode_words

__all__ = ["Normalization", "SolverConfig", "ConvergenceRecord", "SolverResult", "cg_solve",
           "Solver"]


class Normalization(Enum):
    NONE = "none"
    AFTER_RESIDUAL_AXPY = "after-axpy"
    EVERY_VECTOR_OP = "every-op"


@dataclass(frozen=True)
class SolverConfig:
    mode: str = "fp64"
    epsilon: float = 1e-12
    max_iterations: Optional[int] = None  # defaults to 10 n
    normalization: Normalization = Normalization.AFTER_RESIDUAL_AXPY
    history_stride: int = 100
    partitions: int = 1
    reduction: Optional[str] = None   # None: "partitions" if partitions != 1 else "tile"
    timing: str = "graph"

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"unknown arithmetic mode {self.mode!r}")
        if not (self.epsilon > 0.0):
            raise ValueError("epsilon must be positive")
        if self.history_stride < 1:
            raise ValueError("history_stride must be >= 1")
        if self.partitions < 1:
            raise ValueError("partitions must be >= 1")
        if self.reduction is None:
            # an explicit partition count asks for the reference's own dot
            # order (cg.py:42, kernels.py:158-162); the default P = 1 keeps the
            # fast tile order
            object.__setattr__(self, "reduction", "partitions" if self.partitions != 1 else "tile")
        if self.reduction not in ("tile", "partitions"):
            raise ValueError(f"unknown reduction {self.reduction!r}")
        if self.timing not in ("graph", "kernels"):
            raise ValueError(f"unknown timing {self.timing!r}")
        if isinstance(self.normalization, str):
            object.__setattr__(self, "normalization", Normalization(self.normalization))


@dataclass(frozen=True)
class ConvergenceRecord:
    iteration: int
    recurrence_residual: float
    true_residual: float
    error_norm: Optional[float]


@dataclass
class SolverResult:
    converged: bool
    reason: str
    iterations: int
    final_recurrence_residual: float
    x: MultiwordVector
    history: list = field(default_factory=list)
    elapsed_seconds: float = 0.0
    kernel_seconds: dict = field(default_factory=dict)
    device_seconds: float = 0.0      # CUDA-event time of the iteration loop
    history_seconds: float = 0.0     # CUDA-event time of the history metrics
    gpu_launches: int = 0            # kernels launched by the solve


def _dev_f64(a):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return t.to("cuda", non_blocking=True)


class Solver:
    """A reusable device solver for one (matrix, mode, normalization,
    reduction) combination: owns the work vectors and the captured graph."""

    def __init__(self, A, mode, normalization="after-axpy", reduction="tile", partitions=1):
        if isinstance(normalization, Normalization):
            normalization = normalization.value
        # no reference back to A: A caches its solvers (A._solvers), and a
        # cycle A -> solver -> A would leave every matrix/solver pair to the
        # cyclic GC (freed in bursts, the device pool growing meanwhile)
        self.mode = mode
        self.w = mode_words(mode)
        self.n = A.n_rows
        L = _lib.load()
        self._L = L
        self.dm = device_matrix(A)
        self.x = torch.zeros((self.w, max(self.n, 1)), dtype=torch.float64, device="cuda")
        cfg = _lib.SolverConfigC(_lib.MODE_ID[mode], _lib.NORM_ID[normalization],
                                 _lib.RED_ID[reduction], 0, int(partitions))
        h = ctypes.c_void_p()
        _lib.check(L.mwcg_solver_create(ctypes.byref(h), self.dm.handle, ctypes.byref(cfg),
                                        _lib.ptr(self.x), _lib.stream_handle()))
        self.handle = h
        import weakref
        self._fin = weakref.finalize(self, L.mwcg_solver_destroy, h)

    def describe(self):
        """The kernel configuration the library chose (mwcg_solver_describe)."""
        out = (ctypes.c_int64 * 8)()
        _lib.check(self._L.mwcg_solver_describe(self.handle, out, 8))
        keys = ("grid_k1", "grid_k2", "grid_k3", "grid_init", "tma_k2", "tma_k3", "sell_sigma", "col_blocks")
        return dict(zip(keys, (int(v) for v in out)))

    def solve(self, b_dev, b_norm, x0_dev=None, xs_dev=None, epsilon=1e-12, max_iterations=None,
              history_stride=100, profile=False):
        max_it = int(max_iterations if max_iterations is not None else 10 * self.n)
        cap = max(max_it, 0) // history_stride + 4
        hk = np.zeros(cap, dtype=np.int64)
        hr = np.zeros(cap)
        ht = np.zeros(cap)
        he = np.zeros(cap)
        res = _lib.SolveResultC()
        _lib.check(self._L.mwcg_cg_solve(
            self.handle, _lib.ptr(b_dev), float(b_norm), _lib.ptr(x0_dev), _lib.ptr(xs_dev),
            float(epsilon), max_it, int(history_stride), 1 if profile else 0, ctypes.byref(res),
            cap, hk.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            hr.ctypes.data_as(_lib.c_dp), ht.ctypes.data_as(_lib.c_dp),
            he.ctypes.data_as(_lib.c_dp)))
        m = min(res.n_hist, cap)
        hist = [ConvergenceRecord(int(hk[i]), float(hr[i]), float(ht[i]),
                                  None if xs_dev is None else float(he[i])) for i in range(m)]
        return res, hist


_POOL = None
_SOLVER_CACHE = 2


def _host_pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="mwcg-host")
    return _POOL


def _time_k1(solver, b_dev, b_norm, reps=20):
    """Device µs of one K1 launch (SpMV + p.q + alpha) on a freshly started
    solve: `reps` back-to-back launches between CUDA events."""
    L = solver._L
    _lib.check(L.mwcg_solver_start(solver.handle, _lib.ptr(b_dev), float(b_norm), None, None,
                                   1e-300, 10**9))
    us = ctypes.c_double()
    _lib.check(L.mwcg_solver_time_k1(solver.handle, int(reps), ctypes.byref(us)))
    return us.value


def _b_norm(b):
    out = ctypes.c_double()
    _lib.check(_lib.load().mwcg_norm2_host(b.ctypes.data_as(_lib.c_dp), b.size, ctypes.byref(out)))
    return out.value


def cg_solve(A, b, config=SolverConfig(), x0=None, x_star=None, reference=False):
    """Solve A x = b (A SPD) on the GPU; see module docstring."""
    if A.n_rows != A.n_cols:
        raise ValueError("matrix must be square")
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != A.n_rows:
        raise ValueError("right-hand side length does not match the matrix")
    # the reference raises these from spmv(A, x0) (kernels.py:181-183) and
    # from the first history record's residual(x_star, x) (kernels.py:259-260)
    if x0 is not None:
        x0 = np.asarray(x0, dtype=np.float64).reshape(-1)
        if x0.size != A.n_cols:
            raise ValueError(f"dimension mismatch: matrix has {A.n_cols} columns, "
                             f"vector has {x0.size} elements")
    if x_star is not None:
        x_star = np.asarray(x_star, dtype=np.float64).reshape(-1)
        if x_star.size != A.n_rows:
            raise ValueError("dimension mismatch in residual")
    t0 = time.perf_counter()
    # ||b|| is a sequential host sum (the reference order, kernels.py:290-296);
    # it runs on a host thread (ctypes drops the GIL) while the matrix and
    # solver are set up on the device
    bn_future = _host_pool().submit(_b_norm, b)
    mode = config.mode
    n = A.n_rows
    reduction = "partitions" if reference else config.reduction
    key = (mode, config.normalization.value, reduction,
           config.partitions if reduction == "partitions" else 1)
    cache = getattr(A, "_solvers", None)
    if cache is None:
        cache = {}
        try:
            object.__setattr__(A, "_solvers", cache)
        except AttributeError:  # pragma: no cover
            pass
    solver = cache.pop(key, None)
    if solver is None:
        # at most _SOLVER_CACHE solvers per matrix (each holds 4 w n doubles
        # and a captured graph): a multi-mode run on a large matrix keeps the
        # most recent ones only
        while len(cache) >= _SOLVER_CACHE:
            cache.pop(next(iter(cache)))
        solver = Solver(A, mode, config.normalization, reduction, key[3])
    cache[key] = solver  # most recently used last
    b_dev = _dev_f64(b)
    x0_dev = None if x0 is None else _dev_f64(x0)
    xs_dev = None if x_star is None else _dev_f64(x_star)
    bn = bn_future.result()
    profile = config.timing == "kernels"
    res, hist = solver.solve(b_dev, bn, x0_dev, xs_dev, config.epsilon, config.max_iterations,
                             config.history_stride, profile)
    x = MultiwordVector(mode, n, solver.x[:, :n].clone())
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    ks = {"spmv": 0.0, "dot": 0.0, "axpy": 0.0, "scal_add": 0.0, "residual": 0.0,
          "normalize": 0.0}
    if profile:
        ks["spmv"] = res.stage_ms[0] * 1e-3      # SpMV + fused p.q (+ alpha)
        ks["axpy"] = res.stage_ms[1] * 1e-3      # r update + normalize + r.r (+ beta)
        ks["scal_add"] = res.stage_ms[2] * 1e-3  # x update (deferred axpy) + p = r + beta p
    else:
        # graph mode: the fused iteration loop is one device region (CUDA
        # events around each graph launch); it is reported under "spmv", the
        # kernel that dominates it, so the keys still sum to the device time
        ks["spmv"] = res.loop_ms * 1e-3
    reason = _lib.STATUS[res.status]
    return SolverResult(converged=reason == "converged", reason=reason,
                        iterations=int(res.iterations),
                        final_recurrence_residual=float(res.final_rel), x=x, history=hist,
                        elapsed_seconds=elapsed, kernel_seconds=ks,
                        device_seconds=res.loop_ms * 1e-3, history_seconds=res.history_ms * 1e-3,
                        gpu_launches=int(res.launches))
