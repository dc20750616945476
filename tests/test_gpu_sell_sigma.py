"""SELL-sigma (rows length-sorted inside their 1024-row tile, sell.cu): the
SpMV, a whole CG solve and the partitioned (emulated ranks) solve must be
bitwise identical to the unsorted SELL layout and to the oracle (the
reference's per-row left-to-right order, _fast.py:329-339; tile-order dots)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402
from paper_2510_13536_b200 import _lib, cg, problems  # noqa: E402
from paper_2510_13536_b200 import kernels as K  # noqa: E402
from paper_2510_13536_b200.dist import solve_partitioned  # noqa: E402
from paper_2510_13536_b200.sparse import CsrMatrix  # noqa: E402

AUTO = 15


def _c5(n, seed=3):
    rp, col, val = problems.random_irregular_spd(n, seed=seed, device="cpu")
    return CsrMatrix(n, n, rp.numpy().astype(np.int64), col.numpy().astype(np.int64), val.numpy())


def _copy(A):
    return CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values)


def _vec(mode, x):
    return K.MultiwordVector.from_planes(x, mode)


@pytest.mark.parametrize("n", [3000, 20000 + 77])   # ragged last tile / slice
@pytest.mark.parametrize("mode", orc.MODES)
def test_sigma_spmv_bitwise(mode, n):
    A = _c5(n)
    As, Au = _copy(A), _copy(A)
    assert K.device_matrix(As, col_format=AUTO | _lib.SELL_SIGMA).sigma_sorted()
    assert not K.device_matrix(Au, col_format=AUTO | _lib.SELL_NO_SIGMA).sigma_sorted()
    assert K.device_matrix(As).padded_entries() < K.device_matrix(Au).padded_entries()
    x = np.random.default_rng(2).standard_normal((orc.WORDS[mode], n))
    ys = K.spmv(As, _vec(mode, x)).planes.cpu().numpy()
    yu = K.spmv(Au, _vec(mode, x)).planes.cpu().numpy()
    want = orc.spmv(mode, A, x)
    assert np.array_equal(ys.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(yu.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("mode", orc.MODES)
def test_sigma_solve_bitwise_vs_oracle(mode):
    A = _c5(30000)
    b = np.random.default_rng(3).uniform(-1, 1, A.n_rows)
    As = _copy(A)
    K.device_matrix(As, col_format=AUTO | _lib.SELL_SIGMA)
    eps = 1e-12 if mode == "fp64" else 1e-24
    r = cg.cg_solve(As, b, cg.SolverConfig(mode=mode, epsilon=eps, history_stride=5))
    o = orc.cg_solve(A, b, mode=mode, epsilon=eps, history_stride=5, reduction="tile")
    assert r.iterations == o.iterations and r.reason == o.reason
    assert np.array_equal(r.x.planes.cpu().numpy().view(np.uint64), o.x.view(np.uint64))
    assert [h.recurrence_residual for h in r.history] == [h[1] for h in o.history]
    # the TW-accurate history (metrics kernel walks sorted rows too)
    assert [h.true_residual for h in r.history] == [h[2] for h in o.history]


def test_sigma_is_automatic_for_irregular_rows():
    A = _c5(20000)
    assert K.device_matrix(_copy(A)).sigma_sorted()
    st = problems.poisson_3d(12)   # stencil: slice-shared offsets, never sorted
    assert not K.device_matrix(st).sigma_sorted()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["dw", "qtw"])
def test_sigma_partitioned_equals_single(mode, world):
    """Ranks (emulated on one GPU) build their own sorted row blocks; the
    partitioned solve equals the single-GPU solve bit for bit."""
    A = _c5(9000)
    b = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    single = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, epsilon=1e-24, history_stride=10**6))
    res, x = solve_partitioned(A, b, world, mode=mode, epsilon=1e-24, max_iterations=2000)
    assert res.iterations == single.iterations
    assert np.array_equal(x.cpu().numpy().view(np.uint64),
                          single.x.planes.cpu().numpy().view(np.uint64))
