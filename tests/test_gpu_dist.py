"""Partitioned multi-GPU solver, ranks emulated on ONE GPU (LocalExchange):
the real CUDA stage kernels of every rank + the product driver; the result
must be bitwise identical to the single-GPU tile-order solve (same x words,
iteration count, recurrence residual).  The NCCL exchange itself is covered
by tests/test_dist_gloo.py (same driver, gloo) and bench.py under torchrun."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2510_13536_b200 import cg, problems  # noqa: E402
from paper_2510_13536_b200.dist import partition, solve_partitioned  # noqa: E402
from paper_2510_13536_b200.sparse import laplacian_2d  # noqa: E402


def _bits(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("mode", ["fp64", "dw", "qdw", "tw", "qtw"])
def test_partitioned_equals_single_gpu(world, mode):
    A = laplacian_2d(100)  # 10 tiles; world=8 leaves ranks without rows
    xs = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    b = problems.spmv_fp64_host(A, xs)
    eps = 1e-12 if mode == "fp64" else 1e-20
    single = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, epsilon=eps, max_iterations=3000,
                                               history_stride=10**6))
    res, x = solve_partitioned(A, b, world, mode=mode, epsilon=eps, max_iterations=3000,
                               check_every=8)
    assert res.iterations == single.iterations
    assert res.reason == single.reason
    assert res.final_recurrence_residual == single.final_recurrence_residual
    assert np.array_equal(_bits(x), _bits(single.x.planes))


def test_partitioned_c1_x0_and_every_op():
    c = problems.config1()
    x0 = np.random.default_rng(9).uniform(-1, 1, c["A"].n_rows)
    for mode in ("qdw", "qtw"):
        conf = cg.SolverConfig(mode=mode, epsilon=1e-14, normalization="every-op",
                               history_stride=10**6)
        single = cg.cg_solve(c["A"], c["b"], conf, x0=x0)
        res, x = solve_partitioned(c["A"], c["b"], 3, mode=mode, epsilon=1e-14, x0=x0,
                                   normalization="every-op")
        assert res.iterations == single.iterations
        assert np.array_equal(_bits(x), _bits(single.x.planes))


def test_partition_geometry():
    p = partition(10_000, 3)
    assert (p.ntiles, p.tmax) == (10, 4)
    assert [p.rows(r) for r in range(3)] == [(0, 4096), (4096, 8192), (8192, 10000)]
    p8 = partition(10_000, 8)
    assert p8.rows(7) == (10_000, 10_000)


@pytest.mark.parametrize("mode", ["dw", "qtw"])
def test_partitioned_graph_replay_equals_eager(mode):
    """The CUDA-graph segment replay (stage kernels + exchanges captured)
    gives the same bits as the eager driver and as one GPU."""
    A = laplacian_2d(100)
    xs = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    b = problems.spmv_fp64_host(A, xs)
    single = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, epsilon=1e-20, history_stride=10**6))
    res, x = solve_partitioned(A, b, 3, mode=mode, epsilon=1e-20, check_every=8, graph=True)
    assert res.iterations == single.iterations
    assert np.array_equal(_bits(x), _bits(single.x.planes))


@pytest.mark.parametrize("mode", ["dw", "tw"])
def test_partitioned_cached_graph_second_solve(mode):
    """A second solve on the same ranks replays the cached segment graph (no
    eager segment, no re-capture) and reproduces the first solve bitwise;
    the banded matrix takes the neighbour-halo exchange."""
    from paper_2510_13536_b200.cg import _b_norm
    from paper_2510_13536_b200.dist import (LocalExchange, RankSolver, dist_cg_solve, local_rows,
                                            partition)
    A = laplacian_2d(100)
    xs = np.random.default_rng(5).uniform(-1, 1, A.n_rows)
    b = problems.spmv_fp64_host(A, xs)
    part = partition(A.n_rows, 3)
    ranks, bl = [], []
    for r in range(3):
        lo, hi = part.rows(r)
        ranks.append(RankSolver(local_rows(A, lo, hi), part, r, mode))
        bl.append(torch.from_numpy(np.ascontiguousarray(b[lo:hi])).cuda())
    ex = LocalExchange()
    out = []
    for _ in range(2):
        for rs, bb in zip(ranks, bl):
            rs.start(bb, _b_norm(b), None, 1e-20, 10 * A.n_rows)
        res = dist_cg_solve(ranks, ex, _b_norm(b), 1e-20, None, check_every=8, graph=True)
        out.append((res, torch.cat([rs.solution() for rs in ranks], dim=1).clone()))
    assert ex.mode == "halo"
    assert len(ranks[0]._graphs) == 1
    (r1, x1), (r2, x2) = out
    assert r1.iterations == r2.iterations and r1.launches == r2.launches
    assert np.array_equal(_bits(x1), _bits(x2))
    single = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, epsilon=1e-20, history_stride=10**6))
    assert r1.iterations == single.iterations
    assert np.array_equal(_bits(x1), _bits(single.x.planes))
