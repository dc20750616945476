"""Row-partitioned multi-GPU CG.

Partition on tile boundaries: with TILE = 1024 rows, ntiles = ceil(n / TILE)
and tmax = ceil(ntiles / R), rank r owns tiles [r*tmax, min((r+1)*tmax,
ntiles)), i.e. global rows [r*tmax*TILE, ...).  Each rank keeps

  * its rows of A (SELL-32 on its GPU) with GLOBAL column indices,
  * x, r, q for its rows,
  * a full replica of p, shape (R*tmax*TILE, w) -- interleaved words, the
    layout the kernels gather from: the local slice is written by XPAY and the
    replica is refreshed by ONE all-gather of the contiguous slices,
  * the tile partials of ALL ranks, shape (w, R*tmax): every rank writes its
    own tiles and an all-gather completes the array.

Per iteration:  SpMV(+p.q partials) -> gather partials -> finalize(alpha)
-> update(+r.r partials) -> gather partials -> finalize(beta, stop test)
-> XPAY -> gather p.  The finalize stage reduces all global tiles in the
canonical order on every rank, so alpha/beta/stop decisions are identical on
all ranks and the whole solve is bitwise identical to the 1-GPU tile-order
solve.  There is no floating-point all-reduce anywhere (it would
lose the low words and fix no order).

The exchange is pluggable: `TorchDistExchange` (one rank per process over
torch.distributed: NCCL on B200 / NVLink, gloo on CPU) or `LocalExchange`
(R ranks emulated in one process on one GPU, for parity tests).
"""
import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .kernels import device_matrix, mode_words
from .sparse import CsrMatrix

TILE = 1024

__all__ = ["Partition", "partition", "local_rows", "RankSolver", "LocalExchange",
           "TorchDistExchange", "dist_cg_solve", "DistResult"]


@dataclass(frozen=True)
class Partition:
    n: int
    world: int
    ntiles: int
    tmax: int

    @property
    def nmax(self):
        return self.tmax * TILE

    @property
    def ld_full(self):
        return self.world * self.nmax

    @property
    def part_ld(self):
        return self.world * self.tmax

    def rows(self, r):
        lo = min(r * self.nmax, self.n)
        hi = min((r + 1) * self.nmax, self.n)
        return lo, hi

    def tiles(self, r):
        lo = min(r * self.tmax, self.ntiles)
        return lo, min((r + 1) * self.tmax, self.ntiles)


def partition(n, world):
    ntiles = (n + TILE - 1) // TILE
    tmax = max(1, (ntiles + world - 1) // world)
    return Partition(n, world, ntiles, tmax)


def local_rows(A, lo, hi):
    """Rows [lo, hi) of A with global column indices."""
    rp = A.row_ptr[lo:hi + 1] - A.row_ptr[lo]
    a, b = A.row_ptr[lo], A.row_ptr[hi]
    return CsrMatrix(hi - lo, A.n_cols, rp, A.col_idx[a:b], A.values[a:b])


class RankSolver:
    """Device state of one rank (any device; several may share a GPU)."""

    def __init__(self, A_local, part, rank, mode, normalization="after-axpy", device=None):
        dev = torch.device(device or "cuda")
        self.part, self.rank, self.mode = part, rank, mode
        self.w = w = mode_words(mode)
        self.lo, self.hi = part.rows(rank)
        self.n = self.hi - self.lo
        assert A_local.n_rows == self.n
        self.x = torch.zeros((w, max(self.n, 1)), dtype=torch.float64, device=dev)
        self.p_full = torch.zeros((part.ld_full, w), dtype=torch.float64, device=dev)  # AoS
        self.partials = torch.zeros((w, part.part_ld), dtype=torch.float64, device=dev)
        self.dm = device_matrix(A_local, row_base=self.lo)
        L = _lib.load()
        self._L = L
        cfg = _lib.SolverConfigC(_lib.MODE_ID[mode], _lib.NORM_ID[normalization], 0, 0, 1)
        h = ctypes.c_void_p()
        t_lo, _ = part.tiles(rank)
        _lib.check(L.mwcg_solver_create_dist(
            ctypes.byref(h), self.dm.handle, ctypes.byref(cfg), _lib.ptr(self.x),
            _lib.ptr(self.p_full), part.ld_full, self.lo, _lib.ptr(self.partials), part.part_ld,
            t_lo, part.ntiles, _lib.stream_handle()))
        self.handle = h
        import weakref
        self._fin = weakref.finalize(self, L.mwcg_solver_destroy, h)

    # slices this rank contributes to the gathers
    def p_slice(self):
        return self.rank * self.part.nmax, self.part.nmax

    def part_slice(self):
        return self.rank * self.part.tmax, self.part.tmax

    def segments(self, which):
        """1-D (buffer, offset, count) triples this rank contributes to a
        gather: the AoS p replica is one contiguous block; the SoA tile
        partials are one block per word plane."""
        if which == "p":
            off, cnt = self.p_slice()
            return [(self.p_full.view(-1), off * self.w, cnt * self.w)]
        off, cnt = self.part_slice()
        return [(self.partials[k], off, cnt) for k in range(self.w)]

    def start(self, b_local, b_norm, x0_full, epsilon, max_iterations):
        self._b = b_local          # keep alive: the device state points at it
        self._x0 = x0_full
        _lib.check(self._L.mwcg_solver_start(self.handle, _lib.ptr(b_local), float(b_norm),
                                             _lib.ptr(x0_full), None, float(epsilon),
                                             int(max_iterations)))

    def stage(self, name):
        _lib.check(self._L.mwcg_solver_dist_stage(self.handle, _lib.STAGE[name],
                                                  _lib.stream_handle()))

    def state(self):
        s = _lib.StateC()
        _lib.check(self._L.mwcg_solver_state(self.handle, ctypes.byref(s)))
        return s

    def solution(self):
        return self.x[:, :self.n]


class LocalExchange:
    """R ranks in one process (one GPU): copy each rank's slice to the others."""

    def gather(self, ranks, which):
        for src in ranks:
            for j, (buf, off, cnt) in enumerate(src.segments(which)):
                seg = buf[off:off + cnt]
                for dst in ranks:
                    if dst is not src:
                        dst.segments(which)[j][0][off:off + cnt].copy_(seg)


class TorchDistExchange:
    """One rank per process over torch.distributed (NCCL on GPUs, gloo on CPU):
    an in-place all-gather per word plane of p / of the tile partials."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.nccl = dist.get_backend(group) == "nccl"

    def gather(self, ranks, which):
        (me,) = ranks
        for buf, off, cnt in me.segments(which):
            if self.nccl:  # in-place: each rank's slice already sits at off = rank*cnt
                self.dist.all_gather_into_tensor(buf, buf[off:off + cnt], group=self.group)
            else:
                outs = list(buf.split(cnt))
                tmp = [torch.empty_like(o) for o in outs]
                self.dist.all_gather(tmp, buf[off:off + cnt].clone(), group=self.group)
                for o, t in zip(outs, tmp):
                    o.copy_(t)


@dataclass
class DistResult:
    converged: bool
    reason: str
    iterations: int
    final_recurrence_residual: float


def _iteration(ranks, exchange):
    for rs in ranks:
        rs.stage("spmv")
    exchange.gather(ranks, "part")
    for rs in ranks:
        rs.stage("final_alpha")
    for rs in ranks:
        rs.stage("update")
    exchange.gather(ranks, "part")
    for rs in ranks:
        rs.stage("final_beta")
    for rs in ranks:
        rs.stage("xpay")
    exchange.gather(ranks, "p")


def dist_cg_solve(ranks, exchange, b_norm, epsilon=1e-12, max_iterations=None,
                  check_every=16, graph=False):
    """Drive the SPMD stages over `ranks` (all local ranks of this process).

    graph=True captures `check_every` iterations -- stage kernels and the
    NCCL all-gathers -- into one CUDA graph and replays it, so the host does
    one launch per segment instead of ~10 per iteration.  Stages after the
    stop test early-exit on the device status; the segment's remaining
    exchanges are harmless."""
    part = ranks[0].part
    exchange.gather(ranks, "part")
    for rs in ranks:
        rs.stage("final_init")
    exchange.gather(ranks, "p")
    st = ranks[0].state()
    g = None
    if graph and st.status == 0:
        # one eager segment first (NCCL communicators / lazy init), then capture
        for _ in range(check_every):
            _iteration(ranks, exchange)
        st = ranks[0].state()
        if st.status == 0:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(check_every):
                        _iteration(ranks, exchange)
                g.replay()   # the captured segment is not executed by capture itself
            except Exception:  # pragma: no cover - capture unsupported: stay eager
                g = None
                torch.cuda.synchronize()
            st = ranks[0].state()
    while st.status == 0:
        if g is not None:
            g.replay()
        else:
            for _ in range(check_every):
                _iteration(ranks, exchange)
        st = ranks[0].state()
    reason = _lib.STATUS[st.status]
    return DistResult(reason == "converged", reason, int(st.iterations), float(st.rel))


def solve_partitioned(A, b, world, mode="dw", epsilon=1e-12, max_iterations=None, x0=None,
                      normalization="after-axpy", exchange=None, ranks_here=None,
                      check_every=16, graph=False):
    """Convenience: build the rank solvers for `ranks_here` (default: all
    ranks, emulated in this process) and solve.  Returns (result, x words of
    the local ranks concatenated)."""
    from .cg import _b_norm
    part = partition(A.n_rows, world)
    ranks_here = list(range(world)) if ranks_here is None else list(ranks_here)
    exchange = exchange or LocalExchange()
    b = np.ascontiguousarray(b, dtype=np.float64)
    x0_full = None
    if x0 is not None:
        xf = np.zeros(part.ld_full)
        xf[:A.n_rows] = x0
        x0_full = torch.from_numpy(xf).cuda()
    ranks = []
    for r in ranks_here:
        lo, hi = part.rows(r)
        rs = RankSolver(local_rows(A, lo, hi), part, r, mode, normalization)
        b_loc = torch.from_numpy(np.ascontiguousarray(b[lo:hi])).cuda() if hi > lo else \
            torch.zeros(1, dtype=torch.float64, device="cuda")
        rs.start(b_loc, _b_norm(b), x0_full, epsilon, max_iterations if max_iterations is not None
                 else 10 * A.n_rows)
        ranks.append(rs)
    res = dist_cg_solve(ranks, exchange, _b_norm(b), epsilon, max_iterations, check_every, graph)
    x = torch.cat([rs.solution() for rs in ranks], dim=1)
    return res, x
