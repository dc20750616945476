"""Row-partitioned multi-GPU CG.

Partition on tile boundaries: with TILE = 1024 rows, ntiles = ceil(n / TILE)
and tmax = ceil(ntiles / R), rank r owns tiles [r*tmax, min((r+1)*tmax,
ntiles)), i.e. global rows [r*tmax*TILE, ...).  Each rank keeps

  * its rows of A (SELL-32 on its GPU) with GLOBAL column indices,
  * x, r, q for its rows,
  * a full replica of p, shape (R*tmax*TILE, w) -- interleaved words, the
    layout the kernels gather from: the local slice is written by XPAY and the
    replica is refreshed by ONE all-gather of the contiguous slices,
  * the tile partials of ALL ranks, rank-blocked, shape (R, w, tmax): every
    rank writes its own block and ONE all-gather completes the array.

Pipelined exchange (opt-in, `pipeline=True`; irregular matrices whose p exchange
is the all-gather: C5).  The rank's matrix is cut into column blocks (sell.cu)
whose width divides the ranks' slice of p, so the blocks [s*m, (s+1)*m) hold
exactly the columns owned by rank s.  A row's sum runs left to right through the
blocks, i.e. through the ranks' slices in rank order -- so instead of one
all-gather followed by the whole SpMV, rank s's slice is BROADCAST (R broadcasts,
issued back to back on the communication stream) and the block passes of slice s
start as soon as broadcast s has landed: the transfer of slice s+1.. overlaps the
passes over slice s.  Same additions in the same order: bitwise identical.

Per iteration:  [start the p exchange] -> SpMV of the interior tiles (rows
that read only this rank's slice of p) -> [finish the exchange] -> SpMV of
the boundary tiles (+p.q partials) -> gather partials -> finalize(alpha)
-> update(+r.r partials) -> gather partials -> finalize(beta, stop test)
-> XPAY.  For the stencil / band configs the p exchange is a neighbour halo
and runs concurrently with the interior SpMV; a row is always computed whole
by one of the two SpMV launches, so its left-to-right sum (kernels.py:
175-180) is unchanged.  C5's random global columns leave no interior tiles:
its all-gather cannot overlap the SpMV without changing the reference's
per-row summation order.  The finalize stage reduces all
global tiles in the canonical order on every rank, so alpha/beta/stop
decisions are identical on all ranks and the whole solve is bitwise
identical to the 1-GPU tile-order solve.  There is no floating-point
all-reduce anywhere (it would lose the low words and fix no
order).

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
PIPELINE_BLOCK_COLUMNS = 1 << 21   # widest column block of the pipelined exchange (a 32-MB range of a DW p)

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
    """Rows [lo, hi) of A with global column indices.  A DeviceCsrMatrix (C5,
    built on the GPU) is sliced on the device: no host copy of its ~1e9
    entries."""
    if isinstance(A.row_ptr, torch.Tensor):
        from .sparse import DeviceCsrMatrix
        a, b = int(A.row_ptr[lo]), int(A.row_ptr[hi])
        rp = (A.row_ptr[lo:hi + 1] - A.row_ptr[lo]).contiguous()
        return DeviceCsrMatrix(hi - lo, A.n_cols, rp, A.col_idx[a:b], A.values[a:b])
    rp = A.row_ptr[lo:hi + 1] - A.row_ptr[lo]
    a, b = A.row_ptr[lo], A.row_ptr[hi]
    return CsrMatrix(hi - lo, A.n_cols, rp, A.col_idx[a:b], A.values[a:b])


def tile_column_ranges(A_local):
    """(min, max) global column read by each local tile of TILE rows (rows
    are sorted, so a row's first / last entry hold its extremes); empty tiles
    give (+inf, -inf) as (n_cols, -1)."""
    n = A_local.n_rows
    nt = (n + TILE - 1) // TILE
    if nt == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    rp, ci = A_local.row_ptr, A_local.col_idx
    if isinstance(rp, torch.Tensor):
        rp64 = rp.to(torch.int64)
        lens = rp64[1:] - rp64[:-1]
        nz = lens > 0
        first = torch.where(nz, ci[rp64[:-1].clamp(max=max(ci.numel() - 1, 0))].to(torch.int64)
                            if ci.numel() else torch.zeros_like(rp64[:-1]),
                            torch.full_like(rp64[:-1], A_local.n_cols))
        last = torch.where(nz, ci[(rp64[1:] - 1).clamp(min=0)].to(torch.int64)
                           if ci.numel() else torch.zeros_like(rp64[1:]),
                           torch.full_like(rp64[1:], -1))
        pad = nt * TILE - n
        first = torch.nn.functional.pad(first, (0, pad), value=A_local.n_cols)
        last = torch.nn.functional.pad(last, (0, pad), value=-1)
        return (first.view(nt, TILE).min(1).values.cpu().numpy(),
                last.view(nt, TILE).max(1).values.cpu().numpy())
    rp = np.asarray(rp, dtype=np.int64)
    lens = np.diff(rp)
    nz = lens > 0
    first = np.full(nt * TILE, A_local.n_cols, dtype=np.int64)
    last = np.full(nt * TILE, -1, dtype=np.int64)
    if ci.size:
        first[:n][nz] = ci[rp[:-1][nz]]
        last[:n][nz] = ci[rp[1:][nz] - 1]
    return first.reshape(nt, TILE).min(1), last.reshape(nt, TILE).max(1)


def interior_tiles(A_local, lo, hi):
    """The longest run [ilo, ihi) of local tiles whose rows read p only in
    this rank's own rows [lo, hi): their SpMV needs no exchanged data and
    overlaps the p exchange."""
    tmin, tmax_ = tile_column_ranges(A_local)
    ok = (tmin >= lo) & (tmax_ < hi)
    best, cur = (0, 0), None
    for t, good in enumerate(ok):
        if good:
            cur = (cur[0], t + 1) if cur else (t, t + 1)
            if cur[1] - cur[0] > best[1] - best[0]:
                best = cur
        else:
            cur = None
    return best


class RankSolver:
    """Device state of one rank (any device; several may share a GPU)."""

    def __init__(self, A_local, part, rank, mode, normalization="after-axpy", device=None,
                 pipeline=False):
        dev = torch.device(device or "cuda")
        self.part, self.rank, self.mode = part, rank, mode
        self.w = w = mode_words(mode)
        self.lo, self.hi = part.rows(rank)
        self.n = self.hi - self.lo
        assert A_local.n_rows == self.n
        self.x = torch.zeros((w, max(self.n, 1)), dtype=torch.float64, device=dev)
        self.p_full = torch.zeros((part.ld_full, w), dtype=torch.float64, device=dev)  # AoS
        # rank-blocked tile partials (include/mwcg_cuda.h): rank r's block of
        # w * tmax doubles at r * w * tmax
        self.partials = torch.zeros(part.world * w * part.tmax, dtype=torch.float64, device=dev)
        # pipelined exchange: column blocks aligned with the ranks' slices of p
        # (m blocks per slice, each at most 2^21 columns wide)
        self.blocks_per_slice = 0
        if pipeline:
            m = 1
            while part.nmax // m > PIPELINE_BLOCK_COLUMNS or part.nmax % m:
                m += 1
            self.dm = device_matrix(A_local, row_base=self.lo, col_block=part.nmax // m)
            if self.dm.col_blocks() > 0 and self.dm.block_columns() * m == part.nmax:
                self.blocks_per_slice = m
        else:
            self.dm = device_matrix(A_local, row_base=self.lo)
        L = _lib.load()
        self._L = L
        cfg = _lib.SolverConfigC(_lib.MODE_ID[mode], _lib.NORM_ID[normalization], 0, 0, 1)
        h = ctypes.c_void_p()
        _lib.check(L.mwcg_solver_create_dist(
            ctypes.byref(h), self.dm.handle, ctypes.byref(cfg), _lib.ptr(self.x),
            _lib.ptr(self.p_full), part.ld_full, self.lo, _lib.ptr(self.partials), part.tmax,
            rank * part.tmax, part.ntiles, _lib.stream_handle()))
        self.handle = h
        import weakref
        self._fin = weakref.finalize(self, L.mwcg_solver_destroy, h)
        self.col_range = column_range(A_local)
        self.interior = interior_tiles(A_local, self.lo, self.hi)
        _lib.check(L.mwcg_solver_set_interior(h, *self.interior))

    def p_rows(self, lo, hi):
        """Contiguous views of the p replica for global rows [lo, hi) (AoS:
        one block)."""
        return [self.p_full[lo:hi]]

    # slices this rank contributes to the gathers
    def p_slice(self):
        return self.rank * self.part.nmax, self.part.nmax

    def segments(self, which):
        """1-D (buffer, offset, count) triples this rank contributes to a
        gather: the AoS p replica and the rank-blocked tile partials are one
        contiguous block each (one all-gather per exchange)."""
        if which == "p":
            off, cnt = self.p_slice()
            return [(self.p_full.view(-1), off * self.w, cnt * self.w)]
        blk = self.w * self.part.tmax
        return [(self.partials, self.rank * blk, blk)]

    def start(self, b_local, b_norm, x0_full, epsilon, max_iterations):
        self._b = b_local          # keep alive: the device state points at it
        self._x0 = x0_full
        _lib.check(self._L.mwcg_solver_start(self.handle, _lib.ptr(b_local), float(b_norm),
                                             _lib.ptr(x0_full), None, float(epsilon),
                                             int(max_iterations)))

    def stage(self, name):
        _lib.check(self._L.mwcg_solver_dist_stage(self.handle, _lib.STAGE[name],
                                                  _lib.stream_handle()))

    def spmv_slice(self, src):
        """The block passes over the columns owned by rank `src` (pipelined
        exchange); after src = world - 1 the SpMV and its p.q partials are complete."""
        m = self.blocks_per_slice
        nb = self.dm.col_blocks()
        b0, b1 = min(src * m, nb), min((src + 1) * m, nb)
        if src == self.part.world - 1:
            b1 = nb
        if self.n > 0 and b1 > b0:
            _lib.check(self._L.mwcg_solver_dist_spmv_blocks(self.handle, b0, b1, _lib.stream_handle()))

    def state(self):
        s = _lib.StateC()
        _lib.check(self._L.mwcg_solver_state(self.handle, ctypes.byref(s)))
        return s

    def solution(self):
        return self.x[:, :self.n]


def column_range(A):
    """[min, max] global column referenced by A's rows ((0, -1) if none)."""
    if A.nnz == 0:
        return (0, -1)
    ci = A.col_idx
    if isinstance(ci, torch.Tensor):
        return (int(ci.min()), int(ci.max()))
    return (int(ci.min()), int(ci.max()))


def halo_plan(part, ranges, max_fraction=0.5):
    """Point-to-point pieces of p each rank needs: rank r needs the columns
    [cmin_r, cmax_r] of p; the piece owned by rank s is the overlap with s's
    rows.  Returns {(src, dst): (lo, hi)} row intervals, or None when the
    halo would move more than max_fraction of an all-gather (random columns:
    C5) -- then p is all-gathered."""
    pieces, vol = {}, 0
    for r, (cmin, cmax) in enumerate(ranges):
        for sr in range(part.world):
            if sr == r:
                continue
            lo_s, hi_s = part.rows(sr)
            lo, hi = max(cmin, lo_s), min(cmax + 1, hi_s)
            if lo < hi:
                pieces[(sr, r)] = (lo, hi)
                vol += hi - lo
    full = part.world * (part.world - 1) * part.nmax
    if full == 0 or vol > max_fraction * full:
        return None
    return pieces


class LocalExchange:
    """R ranks in one process (one GPU): copy each rank's slice to the others.
    start() does nothing and finish() copies, so the interior SpMV issued
    between them runs BEFORE the exchanged data lands: a tile wrongly
    classified as interior would read stale p and break the bitwise tests."""

    def __init__(self):
        self.pieces = None

    def setup(self, ranks):
        self.pieces = halo_plan(ranks[0].part, [rs.col_range for rs in ranks])
        self.mode = "halo" if self.pieces is not None else "allgather"

    def start(self, ranks, which):
        return (ranks, which)

    def finish(self, handle):
        self.gather(*handle)

    # pipelined exchange: nothing moves at start; slice s is copied when it is
    # waited for, so a block pass issued before its slice would read stale p
    def start_slices(self, ranks):
        return ranks

    def finish_slice(self, ranks, src):
        for s_rank in ranks:
            if s_rank.rank == src:
                for j, (buf, off, cnt) in enumerate(s_rank.segments("p")):
                    for dst in ranks:
                        if dst is not s_rank:
                            dst.segments("p")[j][0][off:off + cnt].copy_(buf[off:off + cnt])

    def gather(self, ranks, which):
        if which == "p" and self.pieces is not None:
            for (src, dst), (lo, hi) in self.pieces.items():
                for d, s_ in zip(ranks[dst].p_rows(lo, hi), ranks[src].p_rows(lo, hi)):
                    d.copy_(s_)
            return
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
        self.pieces = None

    def setup(self, ranks):
        """All ranks exchange their column ranges once and derive the same
        halo plan (or fall back to the all-gather)."""
        (me,) = ranks
        world = self.dist.get_world_size(self.group)
        dev = me.p_full.device
        t = torch.tensor(list(me.col_range), dtype=torch.int64, device=dev)
        allr = [torch.empty_like(t) for _ in range(world)]
        self.dist.all_gather(allr, t, group=self.group)
        ranges = [tuple(int(v) for v in a.cpu()) for a in allr]
        self.pieces = halo_plan(me.part, ranges)
        self.mode = "halo" if self.pieces is not None else "allgather"

    def _halo(self, me):
        ops = []
        for (src, dst), (lo, hi) in sorted(self.pieces.items()):
            if src == me.rank:
                ops += [self.dist.P2POp(self.dist.isend, seg, dst, group=self.group)
                        for seg in me.p_rows(lo, hi)]
            elif dst == me.rank:
                ops += [self.dist.P2POp(self.dist.irecv, seg, src, group=self.group)
                        for seg in me.p_rows(lo, hi)]
        return self.dist.batch_isend_irecv(ops) if ops else []

    def start(self, ranks, which):
        """Issue the exchange asynchronously (NCCL runs it on its own stream,
        ordered after this stream's work so far); finish() makes the current
        stream wait for it."""
        (me,) = ranks
        if which == "p" and self.pieces is not None:
            return self._halo(me), None
        works, post = [], []
        for buf, off, cnt in me.segments(which):
            if self.nccl:  # in-place: each rank's slice already sits at off = rank*cnt
                works.append(self.dist.all_gather_into_tensor(buf, buf[off:off + cnt],
                                                              group=self.group, async_op=True))
            else:
                outs = list(buf.split(cnt))
                tmp = [torch.empty_like(o) for o in outs]
                works.append(self.dist.all_gather(tmp, buf[off:off + cnt].clone(),
                                                  group=self.group, async_op=True))
                post.append((outs, tmp))
        return works, post

    def finish(self, handle):
        works, post = handle
        for w in works:
            w.wait()
        for outs, tmp in post or ():
            for o, t in zip(outs, tmp):
                o.copy_(t)

    # pipelined exchange: one broadcast per source rank, all issued up front in
    # rank order (the same order on every rank); finish_slice(src) makes the
    # current stream wait for slice src only
    def start_slices(self, ranks):
        (me,) = ranks
        world = self.dist.get_world_size(self.group)
        return [[self.dist.broadcast(buf[s * cnt:(s + 1) * cnt], src=self._global(s), group=self.group,
                                     async_op=True) for buf, _, cnt in me.segments("p")]
                for s in range(world)]

    def _global(self, group_rank):
        return self.dist.get_global_rank(self.group, group_rank) if self.group is not None else group_rank

    def finish_slice(self, works, src):
        for w in works[src]:
            w.wait()

    def gather(self, ranks, which):
        self.finish(self.start(ranks, which))


@dataclass
class DistResult:
    converged: bool
    reason: str
    iterations: int
    final_recurrence_residual: float
    launches: int = 0  # kernels one rank launched (start + stages; graph replays counted)


def _kernels_per_iteration(rs):
    """Kernels one rank launches per iteration: SpMV of the interior and of
    the boundary tiles (each only if non-empty), finalize(alpha), update,
    finalize(beta), XPAY."""
    ilo, ihi = getattr(rs, "interior", (0, 0))
    nt = (rs.n + TILE - 1) // TILE
    dm = getattr(rs, "dm", None)
    per_spmv = max(1, dm.col_blocks()) if dm is not None else 1   # one launch per column block
    if getattr(rs, "blocks_per_slice", 0) > 0:
        return 4 + per_spmv                                     # pipelined: every block once
    return 4 + per_spmv * ((1 if ihi > ilo else 0) + (1 if nt - (ihi - ilo) > 0 else 0))


def _pipelined(ranks, exchange):
    return (getattr(exchange, "mode", None) == "allgather" and hasattr(exchange, "start_slices")
            and all(getattr(rs, "blocks_per_slice", 0) > 0 for rs in ranks))


def _iteration(ranks, exchange):
    if _pipelined(ranks, exchange):
        h = exchange.start_slices(ranks)     # R broadcasts, back to back
        for src in range(ranks[0].part.world):
            exchange.finish_slice(h, src)    # slice src has landed
            for rs in ranks:
                rs.spmv_slice(src)           # ... its block passes overlap the later broadcasts
    else:
        h = exchange.start(ranks, "p")       # p slices written by the last XPAY / init
        for rs in ranks:
            rs.stage("spmv_interior")        # overlaps the exchange
        exchange.finish(h)
        for rs in ranks:
            rs.stage("spmv_boundary")
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


def dist_cg_solve(ranks, exchange, b_norm, epsilon=1e-12, max_iterations=None,
                  check_every=16, graph=False):
    """Drive the SPMD stages over `ranks` (all local ranks of this process).

    graph=True captures `check_every` iterations -- stage kernels and the
    NCCL all-gathers -- into one CUDA graph and replays it, so the host does
    one launch per segment instead of ~10 per iteration.  Stages after the
    stop test early-exit on the device status; the segment's remaining
    exchanges are harmless."""
    part = ranks[0].part
    if getattr(exchange, "setup", None) is not None and getattr(exchange, "_ready", None) is not ranks[0]:
        exchange.setup(ranks)
        exchange._ready = ranks[0]
    exchange.gather(ranks, "part")
    for rs in ranks:
        rs.stage("final_init")
    st = ranks[0].state()
    calls = 0
    cache = getattr(ranks[0], "_graphs", None)
    if cache is None:
        cache = {}
        try:
            ranks[0]._graphs = cache
        except AttributeError:  # pragma: no cover
            pass
    key = (id(exchange), check_every)
    g = cache.get(key) if graph else None
    if graph and g is None and st.status == 0:
        # one eager segment first (NCCL communicators / lazy init), then
        # capture; the graph is kept on the rank (same buffers every solve)
        for _ in range(check_every):
            _iteration(ranks, exchange)
        calls += check_every
        st = ranks[0].state()
        if st.status == 0:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(check_every):
                        _iteration(ranks, exchange)
                g.replay()   # the captured segment is not executed by capture itself
                cache[key] = g
                calls += check_every
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
        calls += check_every
        st = ranks[0].state()
    reason = _lib.STATUS[st.status]
    # start: x0 spread + SpMV + init stage; final_init; then the stage kernels
    launches = 3 + 1 + _kernels_per_iteration(ranks[0]) * calls
    return DistResult(reason == "converged", reason, int(st.iterations), float(st.rel), launches)


def solve_partitioned(A, b, world, mode="dw", epsilon=1e-12, max_iterations=None, x0=None,
                      normalization="after-axpy", exchange=None, ranks_here=None,
                      check_every=16, graph=False, pipeline=False):
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
        rs = RankSolver(local_rows(A, lo, hi), part, r, mode, normalization, pipeline=pipeline)
        b_loc = torch.from_numpy(np.ascontiguousarray(b[lo:hi])).cuda() if hi > lo else \
            torch.zeros(1, dtype=torch.float64, device="cuda")
        rs.start(b_loc, _b_norm(b), x0_full, epsilon, max_iterations if max_iterations is not None
                 else 10 * A.n_rows)
        ranks.append(rs)
    res = dist_cg_solve(ranks, exchange, _b_norm(b), epsilon, max_iterations, check_every, graph)
    x = torch.cat([rs.solution() for rs in ranks], dim=1)
    return res, x
