"""Column-blocked K1 (sell.cu: column blocks): an irregular matrix whose
gathered vector outgrows the L2 is cut into column ranges and the solver's
SpMV walks them in turn, each row's running sum carried in q.  The additions
and their order are those of the unblocked walk (the reference's per-row
left-to-right order, _fast.py:329-339), so a whole solve is bitwise the
unblocked one and the oracle's."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402
from paper_2510_13536_b200 import cg  # noqa: E402
from paper_2510_13536_b200 import kernels as K  # noqa: E402
from paper_2510_13536_b200.dist import solve_partitioned  # noqa: E402
from paper_2510_13536_b200.sparse import CsrMatrix, random_symmetric  # noqa: E402

from .test_gpu_sell_sigma import _c5, _copy  # noqa: E402


N = 72000 + 77   # far columns beyond +-32767: int32 SELL (the layout C5 gets); ragged last tile / slice


def _blocked(A, cols, monkeypatch):
    """A copy of A whose device matrix (int32 SELL) is built with `cols` columns per block."""
    Ab = _copy(A)
    monkeypatch.setenv("MWCG_COLBLOCK", str(cols))
    dm = K.device_matrix(Ab, col_format=0)
    monkeypatch.delenv("MWCG_COLBLOCK")
    return Ab, dm


def test_blocks_are_built_only_for_irregular_wide_matrices(monkeypatch):
    A = _c5(N)
    Ab, dm = _blocked(A, 12000, monkeypatch)
    assert dm.col_blocks() == 7 and dm.col_bytes() == 4
    du = K.device_matrix(_copy(A))
    assert du.col_bytes() == 4 and du.col_blocks() == 0         # default: only >= 2^22 columns
    monkeypatch.setenv("MWCG_COLBLOCK", "100")
    from paper_2510_13536_b200 import problems
    st = problems.poisson_3d(12)                                 # banded layouts are never blocked
    assert K.device_matrix(st).col_blocks() == 0
    monkeypatch.delenv("MWCG_COLBLOCK")


@pytest.mark.parametrize("cols", [5000, 30000, N - 1])
@pytest.mark.parametrize("mode", orc.MODES)
def test_blocked_solve_bitwise_vs_unblocked_and_oracle(mode, cols, monkeypatch):
    A = _c5(N)                               # column ranges that split tiles
    b = np.random.default_rng(3).uniform(-1, 1, A.n_rows)
    eps = 1e-12 if mode == "fp64" else 1e-24
    conf = cg.SolverConfig(mode=mode, epsilon=eps, history_stride=5)
    Ab, dm = _blocked(A, cols, monkeypatch)
    assert dm.col_blocks() == -(-A.n_cols // cols)
    rb = cg.cg_solve(Ab, b, conf)
    ru = cg.cg_solve(_copy(A), b, conf)
    assert rb.iterations == ru.iterations and rb.reason == ru.reason
    assert np.array_equal(rb.x.planes.cpu().numpy().view(np.uint64), ru.x.planes.cpu().numpy().view(np.uint64))
    assert [(h.iteration, h.recurrence_residual, h.true_residual) for h in rb.history] == \
        [(h.iteration, h.recurrence_residual, h.true_residual) for h in ru.history]
    if cols == 30000:
        o = orc.cg_solve(A, b, mode=mode, epsilon=eps, history_stride=5, reduction="tile")
        assert rb.iterations == o.iterations and rb.reason == o.reason
        assert np.array_equal(rb.x.planes.cpu().numpy().view(np.uint64), o.x.view(np.uint64))


@pytest.mark.parametrize("mode", ["dw", "tw"])
def test_blocked_reference_order_and_every_op_normalization(mode, monkeypatch):
    """The reference's dot order (unfused K1) and every-op normalization
    (q normalised once, after the last block) with blocks."""
    A = random_symmetric(5000, extra_per_row=6, seed=11)
    b = np.random.default_rng(5).uniform(-1, 1, A.n_rows)
    for kw in (dict(reduction="partitions", partitions=3), dict(normalization=cg.Normalization("every-op"))):
        conf = cg.SolverConfig(mode="q" + mode if "normalization" in kw else mode, epsilon=1e-20,
                               history_stride=7, **kw)
        Ab, dm = _blocked(A, 700, monkeypatch)
        assert dm.col_blocks() == 8
        rb = cg.cg_solve(Ab, b, conf)
        Au = _copy(A)
        assert K.device_matrix(Au, col_format=0).col_blocks() == 0
        ru = cg.cg_solve(Au, b, conf)
        assert rb.iterations == ru.iterations and rb.reason == ru.reason
        assert np.array_equal(rb.x.planes.cpu().numpy().view(np.uint64),
                              ru.x.planes.cpu().numpy().view(np.uint64))


def test_blocks_with_empty_ranges(monkeypatch):
    """Column ranges no row touches, and rows without entries in a range."""
    n = 6000
    rows = np.arange(n)
    # diagonal + one far entry in the first 500 or last 500 columns only
    far = np.where(rows % 2 == 0, rows % 500, n - 1 - rows % 500)
    keep = far != rows
    r = np.concatenate([rows, rows[keep], far[keep]])
    c = np.concatenate([rows, far[keep], rows[keep]])
    v = np.concatenate([np.full(n, 40.0), np.full(2 * int(keep.sum()), -0.5)])
    from paper_2510_13536_b200.sparse import csr_from_coo
    A = csr_from_coo(n, n, r, c, v)
    b = np.random.default_rng(6).uniform(-1, 1, n)
    conf = cg.SolverConfig(mode="dw", epsilon=1e-24, history_stride=10**6)
    K.device_matrix(A, col_format=0)
    Ab = _copy(A)
    monkeypatch.setenv("MWCG_COLBLOCK", "400")
    dm = K.device_matrix(Ab, col_format=0)
    monkeypatch.delenv("MWCG_COLBLOCK")
    assert dm.col_blocks() == 15
    rb, ru = cg.cg_solve(Ab, b, conf), cg.cg_solve(A, b, conf)
    assert rb.iterations == ru.iterations
    assert np.array_equal(rb.x.planes.cpu().numpy().view(np.uint64), ru.x.planes.cpu().numpy().view(np.uint64))


@pytest.mark.parametrize("world", [2, 3])
def test_blocked_partitioned_equals_single(world, monkeypatch):
    """Ranks (emulated on one GPU) block their own rows; same bits as one GPU."""
    A = _c5(N)
    b = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    single = cg.cg_solve(_copy(A), b, cg.SolverConfig(mode="dw", epsilon=1e-24, history_stride=10**6))
    monkeypatch.setenv("MWCG_COLBLOCK", "20000")
    res, x = solve_partitioned(_copy(A), b, world, mode="dw", epsilon=1e-24, max_iterations=2000)
    monkeypatch.delenv("MWCG_COLBLOCK")
    assert res.iterations == single.iterations
    assert np.array_equal(x.cpu().numpy().view(np.uint64), single.x.planes.cpu().numpy().view(np.uint64))


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("mode", ["dw", "qtw"])
def test_pipelined_slice_exchange_equals_single(world, mode):
    """dist.py's pipelined exchange: the rank matrices are cut into column
    blocks aligned with the ranks' slices of p and block passes of slice s run
    when slice s has been delivered (LocalExchange copies it only then, so a
    pass issued early would read stale p).  Bitwise the single-GPU solve."""
    from paper_2510_13536_b200.dist import LocalExchange, RankSolver, _pipelined, partition
    A = _c5(N)
    b = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    single = cg.cg_solve(_copy(A), b, cg.SolverConfig(mode=mode, epsilon=1e-24, history_stride=10**6))
    res, x = solve_partitioned(_copy(A), b, world, mode=mode, epsilon=1e-24, max_iterations=2000,
                               pipeline=True)
    assert res.iterations == single.iterations and res.reason == single.reason
    assert np.array_equal(x.cpu().numpy().view(np.uint64), single.x.planes.cpu().numpy().view(np.uint64))
    # the pipelined path really ran: blocks aligned with the slices
    part = partition(A.n_rows, world)
    from paper_2510_13536_b200.dist import local_rows
    lo, hi = part.rows(0)
    rs = RankSolver(local_rows(_copy(A), lo, hi), part, 0, mode, pipeline=True)
    assert rs.blocks_per_slice >= 1 and rs.dm.block_columns() * rs.blocks_per_slice == part.nmax
    ex = LocalExchange()
    ex.mode = "allgather"
    assert _pipelined([rs], ex)


def test_pipelined_exchange_with_several_blocks_per_slice(monkeypatch):
    """Slices wider than a block: m > 1 blocks per slice (forced through a small
    block limit)."""
    import paper_2510_13536_b200.dist as D
    A = _c5(N)
    b = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    single = cg.cg_solve(_copy(A), b, cg.SolverConfig(mode="dw", epsilon=1e-24, history_stride=10**6))
    monkeypatch.setattr(D, "PIPELINE_BLOCK_COLUMNS", 10000)
    res, x = solve_partitioned(_copy(A), b, 2, mode="dw", epsilon=1e-24, max_iterations=2000, pipeline=True)
    assert res.iterations == single.iterations
    assert np.array_equal(x.cpu().numpy().view(np.uint64), single.x.planes.cpu().numpy().view(np.uint64))


def test_automatic_blocks_need_far_gathers():
    """Automatic choice (no MWCG_COLBLOCK, >= 2^22 columns): blocks only when at
    least 10 % of the entries lie 2^21 or more columns away from their row."""
    n = (1 << 22) + 5000
    rows = np.arange(n, dtype=np.int64)
    rng = np.random.default_rng(8)

    def build(far_cols, near=None):
        if near is None:
            near = np.clip(rows + rng.integers(33000, 50000, n), 0, n - 1)   # irregular, beyond int16 deltas
        cols = np.stack([rows, near, far_cols], axis=1)
        cols.sort(axis=1)
        keep = np.ones_like(cols, dtype=bool)
        keep[:, 1:] = cols[:, 1:] != cols[:, :-1]                        # drop duplicate columns
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(keep.sum(axis=1), out=rp[1:])
        return CsrMatrix(n, n, rp, cols[keep], np.ones(int(keep.sum())))

    local = build(np.clip(rows - rng.integers(33000, 50000, n), 0, n - 1))
    dm = K.device_matrix(local)
    assert dm.col_bytes() == 4 and dm.col_blocks() == 0
    local.release_device()
    # two uniform columns per row: a quarter of them >= 2^21 away -> 1/6 of the entries
    spread = build(rng.integers(0, n, n), rng.integers(0, n, n))
    dm = K.device_matrix(spread)
    assert dm.col_bytes() == 4 and dm.col_blocks() == 3 and dm.block_columns() == 1 << 21
