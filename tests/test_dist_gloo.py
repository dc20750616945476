"""World-size-2/3 CPU test of the partitioned solver's distributed logic
(paper_2510_13536_b200.dist: tile-aligned row partition, p replica gather,
tile-partial gather + canonical reduction) over torch.distributed gloo.

The per-rank compute is the C oracle (tests/cpu_rank.py) standing in for the
CUDA kernels; the driver (`dist_cg_solve`) and the exchange
(`TorchDistExchange`) are the product code.  The gathered solution must be
bitwise identical to the single-process oracle solve in the canonical tile
order, i.e. to what one GPU computes."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _matrix(kind, k):
    from paper_2510_13536_b200.sparse import laplacian_2d, random_symmetric
    return laplacian_2d(k) if kind == "lap" else random_symmetric(k * k, seed=3)


def _worker(rank, world, port, mode, k, outdir, kind, pipeline=False):
    import sys
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_13536_b200 import problems
        from paper_2510_13536_b200.dist import (TorchDistExchange, dist_cg_solve, local_rows,
                                                partition)
        from paper_2510_13536_b200.sparse import laplacian_2d
        import importlib.util
        spec = importlib.util.spec_from_file_location(
            "mwcg_cpu_rank", os.path.join(ROOT, "tests", "cpu_rank.py"))
        cpu_rank = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(cpu_rank)
        CpuRank = cpu_rank.CpuRank
        A = _matrix(kind, k)
        xs = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
        b = problems.spmv_fp64_host(A, xs)
        part = partition(A.n_rows, world)
        lo, hi = part.rows(rank)
        rs = CpuRank(local_rows(A, lo, hi), part, rank, mode, pipeline=pipeline)
        s = 0.0
        for v in b:
            s = s + v * v
        rs.start(b[lo:hi], float(np.sqrt(s)), None, 1e-20 if mode != "fp64" else 1e-12, 2000)
        ex = TorchDistExchange()
        res = dist_cg_solve([rs], ex, float(np.sqrt(s)),
                            1e-20 if mode != "fp64" else 1e-12, 2000, check_every=4)
        np.save(os.path.join(outdir, f"x{rank}.npy"), rs.x)
        from paper_2510_13536_b200.dist import _pipelined
        with open(os.path.join(outdir, f"mode{rank}.txt"), "w") as f:
            f.write(ex.mode + ("+pipelined" if _pipelined([rs], ex) else ""))
        np.save(os.path.join(outdir, f"it{rank}.npy"),
                np.array([res.iterations, res.final_recurrence_residual]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode,kind", [(2, "dw", "lap"), (3, "qtw", "lap"),
                                             (2, "fp64", "lap"), (2, "dw", "rand")])
def test_partitioned_solve_gloo_matches_single(world, mode, kind, tmp_path):
    # n = 10,000 (lap) / 3,600 (rand): ragged last tile, uneven ranks for world=3
    k = 100 if kind == "lap" else 60
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, mode, k, str(tmp_path), kind), nprocs=world,
                       join=True, start_method="spawn")
    from oracle import oracle as orc
    from paper_2510_13536_b200 import problems
    A = _matrix(kind, k)
    xs = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    b = problems.spmv_fp64_host(A, xs)
    eps = 1e-20 if mode != "fp64" else 1e-12
    ref = orc.cg_solve(A, b, mode=mode, epsilon=eps, max_iterations=2000, reduction="tile",
                       record_history=False)
    x = np.concatenate([np.load(tmp_path / f"x{r}.npy") for r in range(world)], axis=1)
    its = [np.load(tmp_path / f"it{r}.npy") for r in range(world)]
    assert all(int(i[0]) == ref.iterations for i in its)
    assert all(i[1] == ref.final_recurrence_residual for i in its)
    assert np.array_equal(x.view(np.uint64), ref.x.view(np.uint64))
    # banded matrix: neighbour halo; random columns: all-gather of p
    want = "halo" if kind == "lap" else "allgather"
    assert all((tmp_path / f"mode{r}.txt").read_text() == want for r in range(world))


@pytest.mark.parametrize("world,mode", [(2, "dw"), (3, "qtw")])
def test_pipelined_slice_broadcasts_gloo(world, mode, tmp_path):
    """The pipelined exchange of dist.py (one broadcast per rank slice, the
    passes over slice s issued once broadcast s has completed) over gloo:
    bitwise the single-process solve."""
    k = 60 if world == 2 else 100   # world 3 at n = 3600 would leave a rank without rows and use halos
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, mode, k, str(tmp_path), "rand", True), nprocs=world,
                       join=True, start_method="spawn")
    from oracle import oracle as orc
    from paper_2510_13536_b200 import problems
    A = _matrix("rand", k)
    xs = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    b = problems.spmv_fp64_host(A, xs)
    ref = orc.cg_solve(A, b, mode=mode, epsilon=1e-20, max_iterations=2000, reduction="tile",
                       record_history=False)
    x = np.concatenate([np.load(tmp_path / f"x{r}.npy") for r in range(world)], axis=1)
    its = [np.load(tmp_path / f"it{r}.npy") for r in range(world)]
    assert all(int(i[0]) == ref.iterations for i in its)
    assert np.array_equal(x.view(np.uint64), ref.x.view(np.uint64))
    # random columns -> all-gather, replaced by the slice broadcasts
    want = "allgather+pipelined"
    assert all((tmp_path / f"mode{r}.txt").read_text() == want for r in range(world))


def test_halo_plan():
    from paper_2510_13536_b200.dist import halo_plan, partition, local_rows, column_range
    from paper_2510_13536_b200.sparse import laplacian_2d, random_symmetric
    A = laplacian_2d(200)  # 40,000 rows -> 40 tiles
    part = partition(A.n_rows, 4)
    ranges = [column_range(local_rows(A, *part.rows(r))) for r in range(4)]
    pieces = halo_plan(part, ranges)
    # each rank talks to its neighbours only, one grid line (200 rows) each way
    assert set(pieces) == {(0, 1), (1, 0), (1, 2), (2, 1), (2, 3), (3, 2)}
    for (src, dst), (lo, hi) in pieces.items():
        assert hi - lo == 200
        slo, shi = part.rows(src)
        assert slo <= lo < hi <= shi
    R = random_symmetric(4000, seed=1)
    part = partition(R.n_rows, 2)
    ranges = [column_range(local_rows(R, *part.rows(r))) for r in range(2)]
    assert halo_plan(part, ranges) is None
