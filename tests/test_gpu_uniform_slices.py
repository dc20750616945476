"""Value-uniform slices of the slice-shared-offset layout (common.cuh): a
slice whose slots hold the same value bits in every row that has them keeps
the values in its pattern records and streams no matrix bytes.  Results must
be bitwise those of the streamed layout and of the oracle (spmv_<mode>:
_fast.py:284-290, 329-339, 383-393, 443-455, 501-513)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import oracle as orc  # noqa: E402
from paper_2510_13536_b200 import _lib, cg, kernels as K, problems  # noqa: E402
from paper_2510_13536_b200.sparse import CsrMatrix  # noqa: E402

from .test_gpu_parity import _vec, same_bits  # noqa: E402


def _copy(A, values=None):
    return CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values if values is None else values)


def test_stencil_is_fully_uniform_and_streams_nothing():
    A = problems.config1()["A"]
    du = K.device_matrix(_copy(A))
    ds = K.device_matrix(_copy(A), col_format=15 | _lib.DIA_STREAM_VALUES)
    assert du.col_bytes() == 0 and ds.col_bytes() == 0
    assert du.stored_values() == 0
    assert ds.stored_values() == ds.padded_entries() >= A.nnz
    assert du.padded_entries() == ds.padded_entries()


@pytest.mark.parametrize("mode", orc.MODES)
def test_uniform_equals_streamed_and_oracle(mode):
    A = problems.config1()["A"]
    rng = np.random.default_rng(21)
    x = rng.standard_normal((orc.WORDS[mode], A.n_rows))
    Au, As = _copy(A), _copy(A)
    K.device_matrix(As, col_format=15 | _lib.DIA_STREAM_VALUES)
    yu = K.spmv(Au, _vec(mode, x)).planes.cpu().numpy()
    ys = K.spmv(As, _vec(mode, x)).planes.cpu().numpy()
    assert same_bits(yu, ys) and same_bits(yu, orc.spmv(mode, A, x))


@pytest.mark.parametrize("mode", orc.MODES)
def test_mixed_uniform_and_streamed_slices(mode):
    """Perturb the values of a band of rows: their slices stream, the rest
    stay uniform; rows at the stencil boundary (missing neighbours), a
    partial last slice, signed zeros and values that differ only in the
    last bit."""
    A0 = problems.laplacian_2d(45)  # n = 2025: partial last slice
    v = np.array(A0.values, dtype=np.float64)
    rp = A0.row_ptr
    rng = np.random.default_rng(5)
    for r in range(300, 700):  # non-uniform slices
        v[rp[r]:rp[r + 1]] *= rng.uniform(0.5, 1.5)
    r = 1000  # one row of an otherwise uniform slice differs by one ulp
    v[rp[r]] = np.nextafter(v[rp[r]], 0.0)
    for r in range(1280, 1312):  # a slice whose off-diagonals are -0.0 in every row: uniform
        for k in range(rp[r], rp[r + 1]):
            if A0.col_idx[k] != r:
                v[k] = -0.0
    r = 1400  # +0.0 vs -0.0 in one slot: different bits, not uniform
    v[rp[r]] = 0.0
    v[rp[r + 1] - 1] = -0.0
    A = _copy(A0, v)
    du = K.device_matrix(A, col_format=2)
    assert 0 < du.stored_values() < du.padded_entries()
    As = _copy(A0, v)
    K.device_matrix(As, col_format=2 | _lib.DIA_STREAM_VALUES)
    Ai = _copy(A0, v)
    K.device_matrix(Ai, col_format=0)
    x = rng.standard_normal((orc.WORDS[mode], A.n_rows))
    yu = K.spmv(A, _vec(mode, x)).planes.cpu().numpy()
    assert same_bits(yu, K.spmv(As, _vec(mode, x)).planes.cpu().numpy())
    assert same_bits(yu, K.spmv(Ai, _vec(mode, x)).planes.cpu().numpy())
    assert same_bits(yu, orc.spmv(mode, A, x))


@pytest.mark.parametrize("mode", ["fp64", "dw", "tw", "qtw"])
def test_solve_uniform_equals_streamed(mode):
    c = problems.config1()
    A = c["A"]
    conf = cg.SolverConfig(mode=mode, epsilon=1e-12, history_stride=100)
    got = []
    for flag in (0, _lib.DIA_STREAM_VALUES):
        Af = _copy(A)
        K.device_matrix(Af, col_format=15 | flag)
        got.append(cg.cg_solve(Af, c["b"], conf, x_star=c["x_star"]))
    assert got[0].iterations == got[1].iterations == 853 and got[0].reason == got[1].reason
    assert same_bits(got[0].x.planes.cpu().numpy(), got[1].x.planes.cpu().numpy())
    assert [(h.iteration, h.recurrence_residual, h.true_residual, h.error_norm) for h in got[0].history] == \
        [(h.iteration, h.recurrence_residual, h.true_residual, h.error_norm) for h in got[1].history]
