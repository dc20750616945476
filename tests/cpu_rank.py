"""CPU stand-in for one rank of the partitioned solver (TEST INFRASTRUCTURE).

Same interface as paper_2510_13536_b200.dist.RankSolver (p_full / partials
tensors, p_slice / part_slice, start / stage / state), computed with the C
oracle so the product's distributed driver (`dist_cg_solve`) and its gloo
exchange can be exercised on CPU with world_size > 1.  The scalar steps
restate cg.py:147-181 exactly as csrc/cg.cu:scalar_* do.
"""
import math
from types import SimpleNamespace

import numpy as np
import torch

from oracle import oracle as orc


class CpuRank:
    def __init__(self, A_local, part, rank, mode, normalization="after-axpy", pipeline=False):
        self.part, self.rank, self.mode = part, rank, mode
        # pipelined exchange (dist.py): one "block" per rank slice; spmv_slice(s)
        # records slice s of p AS IT IS when its pass runs, and the SpMV after the
        # last slice uses that record -- a pass issued before its slice arrived
        # would freeze stale data and break the bitwise comparison
        self.blocks_per_slice = 1 if pipeline else 0
        self.w = w = orc.WORDS[mode]
        self.lo, self.hi = part.rows(rank)
        self.n = self.hi - self.lo
        self.A = A_local
        self.p_full = torch.zeros((w, part.ld_full), dtype=torch.float64)
        # rank-blocked partials, as the product's RankSolver (include/mwcg_cuda.h)
        self.partials = torch.zeros(part.world * w * part.tmax, dtype=torch.float64)
        self.x = np.zeros((w, self.n))
        self.r = np.zeros((w, self.n))
        self.q = np.zeros((w, self.n))
        quasi = mode in ("qdw", "qtw")
        self.norm_r = quasi and normalization != "none"
        self.norm_all = quasi and normalization == "every-op"
        self.st = SimpleNamespace(status=0, k=0, iterations=0, rel=0.0)
        ci = A_local.col_idx
        self.col_range = (int(ci.min()), int(ci.max())) if ci.size else (0, -1)
        from paper_2510_13536_b200.dist import interior_tiles
        self.interior = interior_tiles(A_local, self.lo, self.hi)

    def p_slice(self):
        return self.rank * self.part.nmax, self.part.nmax

    def p_rows(self, lo, hi):  # SoA planes: one contiguous view per word
        return [self.p_full[j, lo:hi] for j in range(self.w)]

    def segments(self, which):  # this stand-in keeps p in SoA planes
        if which == "p":
            off, cnt = self.p_slice()
            return [(self.p_full[k], off, cnt) for k in range(self.w)]
        blk = self.w * self.part.tmax
        return [(self.partials, self.rank * blk, blk)]

    def _blocks(self):
        """(w, R*tmax) word planes of the rank-blocked partials (a view)."""
        R, w, t = self.part.world, self.w, self.part.tmax
        return self.partials.view(R, w, t).permute(1, 0, 2).reshape(w, R * t)

    def _pl(self):
        return self.p_full.numpy()[:, self.lo:self.hi]

    def _partials_of(self, x, y):
        blk = self.w * self.part.tmax
        out = np.zeros((self.w, self.part.tmax))
        orc.tile_partials(self.mode, np.ascontiguousarray(x), np.ascontiguousarray(y), out, 0)
        self.partials[self.rank * blk:(self.rank + 1) * blk].copy_(torch.from_numpy(out).reshape(-1))

    def start(self, b_local, b_norm, x0_full, epsilon, max_iterations):
        self.b = np.asarray(b_local, dtype=np.float64)
        self.b_norm = 1.0 if b_norm == 0.0 else b_norm
        self.eps, self.max_it = epsilon, max_iterations
        full = np.zeros((self.w, self.part.ld_full))
        if x0_full is not None:
            full[0] = np.asarray(x0_full)
            self.x[0] = full[0, self.lo:self.hi]
        self.q = orc.spmv(self.mode, self.A, full) if self.n else self.q
        self.stage("init")

    def _div(self, a, b):
        return orc.scalar_op("div", self.mode, a, b)[:self.w]

    def _coll(self, v):
        return float(orc.scalar_op("collapse", self.mode, v)[0])

    def _reduce(self):
        return orc.reduce_partials(self.mode, np.ascontiguousarray(
            self._blocks().numpy()[:, :self.part.ntiles]))

    def stage(self, name):
        st, m = self.st, self.mode
        if name not in ("init", "final_init") and st.status != 0:
            return
        if name == "init":
            if self.n:
                self.r = orc.residual(m, self.b, self.q)
                if self.norm_r:
                    self.r = orc.normalize(m, self.r)
                self.p_full.numpy()[:, self.lo:self.hi] = self.r
                self._partials_of(self.r, self.r)
        elif name == "final_init":
            self.rho = self._reduce()
            st.rel = math.sqrt(abs(self._coll(self.rho))) / self.b_norm
            st.k = 0
            if st.rel < self.eps:
                st.status, st.iterations = 1, 0
            elif self.max_it <= 0:
                st.status, st.iterations = 2, self.max_it
        elif name in ("spmv", "spmv_interior", "spmv_boundary"):
            # rows of the interior tiles are computed before the p exchange
            # lands (dist._iteration): from the stale replica, exactly as the
            # device does -- a misclassified tile would break the bitwise test
            if self.n:
                ilo, ihi = self.interior
                rows = np.zeros(self.n, dtype=bool)
                rows[ilo * 1024:ihi * 1024] = True
                if name == "spmv_boundary":
                    rows = ~rows
                elif name == "spmv":
                    rows[:] = True
                q = orc.spmv(m, self.A, self.p_full.numpy())
                if self.norm_all:
                    q = orc.normalize(m, q)
                self.q[:, rows] = q[:, rows]
                if name != "spmv_interior":
                    self._partials_of(self._pl(), self.q)
        elif name == "final_alpha":
            pq = self._reduce()
            f = self._coll(pq)
            if f == 0.0 or not math.isfinite(f):
                st.status, st.iterations = 3, st.k
                return
            self.alpha = self._div(self.rho, pq)
        elif name == "update":
            if self.n:
                self.x = orc.axpy(m, self.alpha, self._pl(), self.x)
                if self.norm_all:
                    self.x = orc.normalize(m, self.x)
                self.r = orc.axpy(m, -self.alpha, self.q, self.r)
                if self.norm_r:
                    self.r = orc.normalize(m, self.r)
                self._partials_of(self.r, self.r)
        elif name == "final_beta":
            rn = self._reduce()
            st.k += 1
            f = self._coll(rn)
            st.rel = math.sqrt(abs(f)) / self.b_norm
            if st.rel < self.eps:
                st.status, st.iterations = 1, st.k
            elif f == 0.0 or not math.isfinite(f):
                st.status, st.iterations = 3, st.k
            else:
                self.beta = self._div(rn, self.rho)
                self.rho = rn
                if st.k >= self.max_it:
                    st.status, st.iterations = 2, st.k
        elif name == "xpay":
            if self.n:
                pl = orc.scal_add(m, self.beta, self._pl(), self.r)
                if self.norm_all:
                    pl = orc.normalize(m, pl)
                self.p_full.numpy()[:, self.lo:self.hi] = pl

    def spmv_slice(self, src):
        if self.st.status != 0:
            return
        if src == 0:
            self._seen = np.zeros_like(self.p_full.numpy())
        lo = src * self.part.nmax
        self._seen[:, lo:lo + self.part.nmax] = self.p_full.numpy()[:, lo:lo + self.part.nmax]
        if src == self.part.world - 1 and self.n:
            q = orc.spmv(self.mode, self.A, self._seen)
            if self.norm_all:
                q = orc.normalize(self.mode, q)
            self.q = q
            self._partials_of(self._pl(), self.q)

    def state(self):
        s = self.st
        return SimpleNamespace(status=s.status, k=s.k, rel=s.rel,
                               iterations=s.iterations if s.status else s.k)

    def solution(self):
        return torch.from_numpy(self.x)
