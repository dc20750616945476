"""Edge cases of the cg_solve boundary on the device: non-positive
max_iterations (cg.py:150, 183: finish(False, "max_iterations", max_iters)),
kernel_seconds filled in graph mode, explicit partitions taking the
reference order, stale-cache protection."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402
from paper_2510_13536_b200 import cg, problems  # noqa: E402
from paper_2510_13536_b200.sparse import laplacian_2d  # noqa: E402


@pytest.mark.parametrize("max_it", [0, -3])
@pytest.mark.parametrize("mode", ["fp64", "qtw"])
def test_non_positive_max_iterations(mode, max_it):
    A = laplacian_2d(8)
    b = problems.spmv_fp64_host(A, np.ones(A.n_rows))
    r = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, max_iterations=max_it), x_star=np.ones(64))
    o = orc.cg_solve(A, b, mode=mode, max_iterations=max_it, reduction="tile", x_star=np.ones(64))
    assert (r.reason, r.iterations) == ("max_iterations", max_it) == (o.reason, o.iterations)
    # finish() records k only when it differs from the last record (cg.py:138-141)
    want = [0] if max_it == 0 else [0, max_it]
    assert [h.iteration for h in r.history] == [h[0] for h in o.history] == want


def test_kernel_seconds_graph_mode():
    A = laplacian_2d(32)
    b = problems.spmv_fp64_host(A, np.ones(A.n_rows))
    r = cg.cg_solve(A, b, cg.SolverConfig(mode="dw"))
    assert set(r.kernel_seconds) == {"spmv", "dot", "axpy", "scal_add", "residual", "normalize"}
    assert r.kernel_seconds["spmv"] > 0 and r.kernel_seconds["spmv"] == pytest.approx(r.device_seconds)


def test_explicit_partitions_bitwise_reference_order():
    A = laplacian_2d(16)
    b = problems.spmv_fp64_host(A, np.random.default_rng(1).uniform(-1, 1, A.n_rows))
    r = cg.cg_solve(A, b, cg.SolverConfig(mode="dw", epsilon=1e-24, partitions=3))
    o = orc.cg_solve(A, b, mode="dw", epsilon=1e-24, partitions=3, reduction="partitions")
    assert r.iterations == o.iterations
    assert np.array_equal(r.x.planes.cpu().numpy().view(np.uint64), o.x.view(np.uint64))


def test_release_device_rebuilds():
    A = laplacian_2d(16)
    b = problems.spmv_fp64_host(A, np.ones(A.n_rows))
    r1 = cg.cg_solve(A, b, cg.SolverConfig(mode="dw", epsilon=1e-20))
    A.release_device()
    r2 = cg.cg_solve(A, b, cg.SolverConfig(mode="dw", epsilon=1e-20))
    assert r1.iterations == r2.iterations
    assert torch.equal(r1.x.planes, r2.x.planes)
