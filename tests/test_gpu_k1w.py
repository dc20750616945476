"""The windowed SpMV kernel (K1W, cg.cu: cg_spmv_pq_win) against the classic
K1 walk: whole solves bitwise identical (x words, iterations, residual
history) on stencil / band matrices with partial tiles, boundary windows
clipped at both ends of p, every stage height and every arithmetic."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2510_13536_b200 import cg, problems  # noqa: E402
from paper_2510_13536_b200.sparse import laplacian_2d, scaled_laplacian_2d  # noqa: E402


def _solve(A, b, mode, env, **kw):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        A.release_device()
        conf = cg.SolverConfig(mode=mode, history_stride=25, **kw)
        r = cg.cg_solve(A, b, conf)
        desc = A._solvers[next(iter(A._solvers))].describe()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        A.release_device()
    return r, desc


def _problems():
    out = [("lap2d_100", laplacian_2d(100)),                 # 10 tiles, ragged
           ("lap2d_256", laplacian_2d(256)),                 # C1
           ("poisson3d_20", problems.poisson_3d(20)),        # 8000 rows: 3 windows, ragged
           ("scaled16", scaled_laplacian_2d(16, 4, 1)),
           ("band", problems.config4(n=5000)["A"]),          # one 19-wide window
           ("c3_14", problems.config3(k=14)["A"])]           # 27-point: 3 windows
    return out


@pytest.mark.parametrize("vs", ["1", "0"])
@pytest.mark.parametrize("mode", ["fp64", "dw", "qdw", "tw", "qtw"])
def test_k1w_bitwise_equals_classic(mode, vs):
    """vs=1: values staged in the ring with the windows; vs=0: windows only,
    values streamed from HBM."""
    for name, A in _problems():
        xs = np.random.default_rng(7).uniform(-1, 1, A.n_rows)
        b = problems.spmv_fp64_host(A, xs)
        eps = 1e-13 if mode == "fp64" else 1e-22
        r1, d1 = _solve(A, b, mode, {"MWCG_K1W": "1", "MWCG_K1W_VS": vs}, epsilon=eps,
                        max_iterations=400)
        r0, d0 = _solve(A, b, mode, {"MWCG_K1W": "0"}, epsilon=eps, max_iterations=400)
        # whole-tile slots of the 27-slot matrix's values do not fit twice
        if not (name == "c3_14" and vs == "1"):
            assert d1["k1_windowed"] == 1 and d1["k1w_values_staged"] == int(vs), (name, d1)
        assert d0["k1_windowed"] == 0
        assert r1.iterations == r0.iterations, name
        assert [h.recurrence_residual for h in r1.history] == \
            [h.recurrence_residual for h in r0.history], name
        assert torch.equal(r1.x.planes.view(torch.int64), r0.x.planes.view(torch.int64)), name


@pytest.mark.parametrize("mode", ["dw", "qtw"])
def test_k1w_every_op_and_partitions(mode):
    A = laplacian_2d(64)
    b = problems.spmv_fp64_host(A, np.ones(A.n_rows))
    for kw in ({"normalization": "every-op"}, {"reduction": "partitions", "partitions": 5}):
        r1, d1 = _solve(A, b, mode, {"MWCG_K1W": "1"}, epsilon=1e-24, **kw)
        r0, _ = _solve(A, b, mode, {"MWCG_K1W": "0"}, epsilon=1e-24, **kw)
        assert d1["k1_windowed"] == 1
        assert r1.iterations == r0.iterations
        assert torch.equal(r1.x.planes.view(torch.int64), r0.x.planes.view(torch.int64))


def test_k1w_default_on_for_stencils():
    c = problems.config2(k=32)
    r, d = _solve(c["A"], c["b"], "dw", {})
    assert d["k1_windowed"] == 1 and d["k1w_windows"] == 3
    A = problems.config3(k=14)["A"]      # 27 slots per slice: windows only
    r, d = _solve(A, np.ones(A.n_rows), "tw", {})
    assert d["k1_windowed"] == 1 and d["k1w_values_staged"] == 0
