"""CPU tests of the BASELINE config-5 generator (problems.random_irregular_spd,
run on the host with torch's CPU generator) and of the host-side argument
checks that mirror the reference's errors (cg.py:85-89, kernels.py:181-183,
259-260)."""
import numpy as np
import pytest

from paper_2510_13536_b200 import problems
from paper_2510_13536_b200.cg import SolverConfig
from paper_2510_13536_b200.sparse import CsrMatrix, laplacian_2d


def _gen(n, seed=3, **kw):
    rp, col, val = problems.random_irregular_spd(n, seed=seed, device="cpu", **kw)
    return CsrMatrix(n, n, rp.numpy().astype(np.int64), col.numpy().astype(np.int64), val.numpy())


@pytest.fixture(scope="module")
def c5small():
    return _gen(20000)


class TestConfig5Generator:
    def test_valid_csr_int32(self):
        rp, col, val = problems.random_irregular_spd(5000, seed=3, device="cpu")
        assert str(rp.dtype) == "torch.int32" and str(col.dtype) == "torch.int32"
        # CsrMatrix validation: sorted strictly increasing columns, bounds
        CsrMatrix(5000, 5000, rp.numpy(), col.numpy(), val.numpy())

    def test_exactly_symmetric(self, c5small):
        A = c5small
        rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
        k1 = rows * A.n_rows + A.col_idx
        k2 = A.col_idx * A.n_rows + rows
        o1, o2 = np.argsort(k1), np.argsort(k2)
        assert np.array_equal(k1[o1], k2[o2])
        # bitwise equal values of (i, j) and (j, i)
        assert np.array_equal(A.values[o1].view(np.uint64), A.values[o2].view(np.uint64))

    def test_diagonal_dominance(self, c5small):
        A = c5small
        n = A.n_rows
        rows = np.repeat(np.arange(n), np.diff(A.row_ptr))
        diag = rows == A.col_idx
        assert diag.sum() == n                       # every row has its diagonal
        off = ~diag
        assert np.all(A.values[off] <= 0.0) and np.all(A.values[off] >= -64.0)
        absrow = np.zeros(n)
        np.add.at(absrow, rows[off], np.abs(A.values[off]))
        d = np.empty(n)
        d[rows[diag]] = A.values[diag]
        # a_ii = 1.01 * sum_j |a_ij| (the generator's row sums are a
        # cumulative-sum difference: equal to rounding, not bitwise)
        assert np.allclose(d, 1.01 * absrow, rtol=1e-9, atol=0)
        assert np.all(d > absrow)                    # strict dominance -> SPD

    def test_row_counts(self, c5small):
        A = c5small
        n = A.n_rows
        lens = np.diff(A.row_ptr)
        # own draws 16..64 (minus diagonal hits / duplicates) plus mirrored ones
        assert lens.min() >= 2 and lens.max() <= 250
        mean_off = (A.nnz - n) / n
        assert 70 < mean_off < 82, mean_off          # ~2 * 40 draws per row, symmetrised
        rows = np.repeat(np.arange(n), lens)
        off = rows != A.col_idx
        near = np.abs(A.col_idx[off] - rows[off]) <= 1024
        # about half the draws land within +-1024 of the diagonal
        assert 0.45 < near.mean() < 0.60
        # no pile-up on the first / last columns (the near window is clipped, not clamped)
        assert lens[0] < 250 and lens[-1] < 250

    def test_deterministic(self):
        a, b = _gen(3000), _gen(3000)
        assert problems.matrix_digest(a) == problems.matrix_digest(b)
        c = _gen(3000, seed=4)
        assert problems.matrix_digest(a) != problems.matrix_digest(c)

    def test_config5_style_shape(self):
        cfg = problems.config5_style(n=4096)
        assert cfg["A"].n_rows == 4096 and cfg["b"].shape == (4096,)
        assert cfg["x_star"] is None and cfg["epsilon"] == 1e-12
        assert np.array_equal(cfg["b"], np.random.default_rng(3).uniform(-1, 1, 4096))


class TestSolverArgs:
    def test_explicit_partitions_select_reference_order(self):
        assert SolverConfig().reduction == "tile"
        assert SolverConfig(partitions=4).reduction == "partitions"
        assert SolverConfig(partitions=4, reduction="tile").reduction == "tile"
        assert SolverConfig(reduction="partitions").reduction == "partitions"

    def test_x0_and_x_star_lengths(self):
        from paper_2510_13536_b200 import cg
        A = laplacian_2d(4)
        b = np.ones(16)
        with pytest.raises(ValueError, match="dimension mismatch: matrix has 16 columns, "
                                             "vector has 15 elements"):
            cg.cg_solve(A, b, x0=np.zeros(15))
        with pytest.raises(ValueError, match="vector has 17 elements"):
            cg.cg_solve(A, b, x0=np.zeros(17))
        with pytest.raises(ValueError, match="dimension mismatch in residual"):
            cg.cg_solve(A, b, x_star=np.zeros(15))
        with pytest.raises(ValueError, match="right-hand side length"):
            cg.cg_solve(A, np.ones(15))

    def test_matrix_arrays_read_only(self):
        A = laplacian_2d(4)
        with pytest.raises(ValueError):
            A.values[0] = 5.0
        with pytest.raises(ValueError):
            A.col_idx[0] = 1
        A.release_device()
        assert A._device is None


class TestPartitionHelpers:
    def test_interior_tiles_banded(self):
        from paper_2510_13536_b200.dist import interior_tiles, local_rows, partition
        A = laplacian_2d(100)               # bandwidth 100, 10 tiles
        part = partition(A.n_rows, 2)
        lo, hi = part.rows(0)
        assert interior_tiles(local_rows(A, lo, hi), lo, hi) == (0, 4)   # tile 4 reads rank 1
        lo, hi = part.rows(1)
        assert interior_tiles(local_rows(A, lo, hi), lo, hi) == (1, 5)   # tile 0 reads rank 0

    def test_interior_tiles_random_has_none(self):
        from paper_2510_13536_b200.dist import interior_tiles, local_rows, partition
        A = _gen(8192)
        part = partition(A.n_rows, 2)
        lo, hi = part.rows(1)
        ilo, ihi = interior_tiles(local_rows(A, lo, hi), lo, hi)
        assert ihi == ilo

    def test_tile_column_ranges_empty_rows(self):
        from paper_2510_13536_b200.dist import tile_column_ranges
        A = CsrMatrix(1500, 1500, np.r_[np.zeros(1025, np.int64), np.arange(1, 477)],
                      np.arange(1024, 1500), np.ones(476))     # rows 0..1023 empty
        mn, mx = tile_column_ranges(A)
        assert list(mn) == [1500, 1024] and list(mx) == [-1, 1499]
