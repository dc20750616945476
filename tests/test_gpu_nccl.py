"""The NCCL exchange path of the partitioned solver, executed for real:
torch.distributed with backend "nccl" at world size 1 (one process, one
B200 -- the only shape this pool offers), eager and CUDA-graph captured,
bitwise against the single-GPU solve.  World > 1 runs the same
TorchDistExchange code (tests/test_dist_gloo.py covers 2-3 ranks on CPU)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2510_13536_b200 import cg, problems  # noqa: E402
from paper_2510_13536_b200.dist import TorchDistExchange, solve_partitioned  # noqa: E402
from paper_2510_13536_b200.sparse import laplacian_2d  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_world1():
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def _bits(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("mode", ["fp64", "dw", "qtw", "tw"])
def test_nccl_world1_equals_single_gpu(nccl_world1, mode, graph):
    A = laplacian_2d(100)
    xs = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    b = problems.spmv_fp64_host(A, xs)
    eps = 1e-12 if mode == "fp64" else 1e-20
    single = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, epsilon=eps, history_stride=10**6))
    ex = TorchDistExchange()
    assert ex.nccl
    res, x = solve_partitioned(A, b, 1, mode=mode, epsilon=eps, exchange=ex, ranks_here=[0],
                               check_every=8, graph=graph)
    assert res.iterations == single.iterations and res.reason == single.reason
    assert res.final_recurrence_residual == single.final_recurrence_residual
    assert np.array_equal(_bits(x), _bits(single.x.planes))


def test_nccl_world1_c2_slice(nccl_world1):
    """A 64^3 7-point problem through the NCCL driver (DW, graph-captured)."""
    c = problems.config2(k=64)
    single = cg.cg_solve(c["A"], c["b"], cg.SolverConfig(mode="dw", epsilon=1e-12,
                                                         history_stride=10**6))
    res, x = solve_partitioned(c["A"], c["b"], 1, mode="dw", epsilon=1e-12,
                               exchange=TorchDistExchange(), ranks_here=[0], graph=True)
    assert res.iterations == single.iterations
    assert np.array_equal(_bits(x), _bits(single.x.planes))


@pytest.mark.parametrize("graph", [False, True])
def test_nccl_world1_pipelined_slice_exchange(nccl_world1, graph):
    """The pipelined exchange (dist.py: NCCL broadcast per rank slice + the
    column-block passes of that slice) through NCCL at world 1, eager and
    graph-captured: an irregular matrix wide enough for int32 columns."""
    from paper_2510_13536_b200.dist import RankSolver, _pipelined, dist_cg_solve, local_rows, partition
    from paper_2510_13536_b200.sparse import CsrMatrix
    from paper_2510_13536_b200.cg import _b_norm
    import paper_2510_13536_b200.dist as D
    n = 72000 + 77
    rp, col, val = problems.random_irregular_spd(n, seed=3, device="cpu")
    A = CsrMatrix(n, n, rp.numpy().astype(np.int64), col.numpy().astype(np.int64), val.numpy())
    b = np.random.default_rng(4).uniform(-1, 1, n)
    single = cg.cg_solve(A, b, cg.SolverConfig(mode="dw", epsilon=1e-24, history_stride=10**6))
    old = D.PIPELINE_BLOCK_COLUMNS
    D.PIPELINE_BLOCK_COLUMNS = 20000   # several blocks inside the one slice
    try:
        part = partition(n, 1)
        rs = RankSolver(local_rows(A, 0, n), part, 0, "dw", pipeline=True)
    finally:
        D.PIPELINE_BLOCK_COLUMNS = old
    assert rs.blocks_per_slice >= 2
    ex = TorchDistExchange()
    bn = _b_norm(b)
    rs.start(torch.from_numpy(b).cuda(), bn, None, 1e-24, 2000)
    res = dist_cg_solve([rs], ex, bn, 1e-24, 2000, check_every=8, graph=graph)
    assert _pipelined([rs], ex)
    assert res.iterations == single.iterations and res.reason == single.reason
    assert np.array_equal(_bits(rs.solution()), _bits(single.x.planes))
