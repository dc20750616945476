"""Exact problem generation (reference problemgen.py:47-108) through the native
row-sum engine (libmwcg_cuda.so: mwcg_problem_generate, host code).

Pinned bit for bit against the real reference on 1912 cases
(tests/golden/problemgen.json, made by tests/golden/make_problemgen_golden.py):
b, the perturbed values, perturbation_norm, max_ulp_adjustment, and the error
message of every failing case.  The other tests restate the reference's own
(pkg/tests/test_problemgen.py) with an exact rational check in place of ExactValue.
"""
from fractions import Fraction

import numpy as np
import pytest

import tests.golden_io as G
from paper_2510_13536_b200.problemgen import GeneratedProblem, generate
from paper_2510_13536_b200.sparse import (CsrMatrix, identity, laplacian_2d, random_symmetric,
                                          scaled_laplacian_2d)


@pytest.fixture(autouse=True, scope="module")
def _lib_built():
    from paper_2510_13536_b200 import _lib
    try:
        _lib.load()
    except Exception:
        pytest.skip("libmwcg_cuda.so not built")


def assert_exactly_consistent(p, rows=None):
    m = p.matrix
    for i in (range(m.n_rows) if rows is None else rows):
        s = sum((Fraction(float(v)) for v in m.values[m.row_ptr[i]:m.row_ptr[i + 1]]), Fraction(0))
        assert Fraction(float(p.b[i])) == s, f"row {i} is not exactly consistent"


def test_golden_against_reference():
    cases = G.load("problemgen.json")["cases"]
    assert len(cases) > 1800
    nudged = errors = 0
    for c in cases:
        A = CsrMatrix(c["n"], c["n"], np.array(c["row_ptr"]), np.array(c["col_idx"]),
                      G.arr(c["values"]))
        if "error" in c:
            errors += 1
            with pytest.raises(ValueError) as ei:
                generate(A)
            assert str(ei.value) == c["error"], c["name"]
            continue
        p = generate(A)
        assert G.same_bits(p.b, G.arr(c["b"])), c["name"]
        assert G.same_bits(p.matrix.values, G.arr(c["out_values"])), c["name"]
        assert G.same_bits([p.perturbation_norm], [G.fh(c["perturbation_norm"])]), c["name"]
        assert p.max_ulp_adjustment == c["max_ulp_adjustment"], c["name"]
        nudged += p.max_ulp_adjustment > 0
    assert errors > 100 and nudged > 50


def test_identity_ones_with_zero_perturbation():
    p = generate(identity(5))
    assert isinstance(p, GeneratedProblem)
    assert np.array_equal(p.b, np.ones(5))
    assert np.array_equal(p.x_star, np.ones(5))
    assert p.perturbation_norm == 0.0 and p.max_ulp_adjustment == 0
    assert_exactly_consistent(p)


def test_laplacian_needs_no_perturbation():
    A = laplacian_2d(4)
    p = generate(A)
    assert p.perturbation_norm == 0.0
    assert np.array_equal(p.matrix.values, A.values)
    assert np.array_equal(generate(laplacian_2d(3)).b, laplacian_2d(3).to_dense().sum(axis=1))
    assert_exactly_consistent(p)


@pytest.mark.parametrize("A", [random_symmetric(60, seed=5), random_symmetric(40, seed=77),
                               scaled_laplacian_2d(5, decades=3.0, seed=8)],
                         ids=["random60", "random40", "scaled-laplacian"])
def test_generated_matrices_exactly_consistent(A):
    before = A.values.copy()
    p = generate(A)
    assert_exactly_consistent(p)
    assert p.max_ulp_adjustment == 0
    assert np.array_equal(A.values, before)


def test_gap_absorbed_into_diagonal():
    A = CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]),
                  np.array([1.0, 2.0 ** 60, 2.0 ** 60, 1.0]))
    p = generate(A)
    assert p.perturbation_norm > 0.0
    assert p.matrix.values[1] == A.values[1] and p.matrix.values[2] == A.values[2]
    d0 = p.matrix.values[0] - A.values[0]
    d1 = p.matrix.values[3] - A.values[3]
    assert p.perturbation_norm == pytest.approx(np.hypot(d0, d1))
    assert_exactly_consistent(p)


def test_missing_diagonal():
    A = CsrMatrix(3, 3, np.array([0, 2, 3, 4]), np.array([1, 2, 0, 0]),
                  np.array([2.0 ** 60, 1.0 + 2.0 ** -52, 2.0 ** 60, 1.0 + 2.0 ** -52]))
    with pytest.raises(ValueError, match="row 0: inexact row sum but no diagonal"):
        generate(A)
    p = generate(CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([1, 0]), np.array([2.0, 2.0])))
    assert np.array_equal(p.b, [2.0, 2.0])


def test_validation():
    assert np.array_equal(generate(identity(3), x_star=np.ones(3)).x_star, np.ones(3))
    with pytest.raises(ValueError, match="all-ones"):
        generate(identity(3), x_star=np.array([1.0, 2.0, 1.0]))
    with pytest.raises(ValueError):
        generate(identity(3), x_star=np.ones(4))
    with pytest.raises(ValueError, match="square"):
        generate(CsrMatrix(1, 2, np.array([0, 1]), np.array([0]), np.array([1.0])))
    with pytest.raises(ValueError, match="row 0: exact row sum overflows"):
        generate(CsrMatrix(2, 2, np.array([0, 2, 3]), np.array([0, 1, 1]),
                           np.array([1.7e308, 1.7e308, 1.0])))


def test_first_failing_row_reported_across_threads():
    # rows 700 and 9000 fail (diagonal 2^60, an off-diagonal 1 + 2^-52: the new
    # diagonal would need > 53 bits whatever the nudge); the first is reported
    A = laplacian_2d(100)
    v = A.values.copy()
    for i in (9000, 700):
        d = A.diagonal_index(i)
        v[d] = 2.0 ** 60
        v[d + 1] = 1.0 + 2.0 ** -52
    B = CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, v)
    for t in (1, 3, 16):
        with pytest.raises(ValueError, match="row 700: no representable diagonal"):
            generate(B, threads=t)


def test_thread_count_invariant_and_scale():
    # |5-point Laplacian| with off-diagonals 1 + j 2^-40 and diagonals 4 + k 2^-50: the
    # row sums need up to 54 bits, so many rows round and absorb the gap
    A = laplacian_2d(300)
    rng = np.random.default_rng(1)
    v = np.abs(A.values)
    off = v != 4.0
    v[off] *= 1.0 + rng.integers(0, 1 << 10, int(off.sum())) * 2.0 ** -40
    v[~off] += rng.integers(0, 1 << 10, int((~off).sum())) * 2.0 ** -50
    A = CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, v)
    p1 = generate(A, threads=1)
    p8 = generate(A, threads=8)
    assert G.same_bits(p1.b, p8.b) and G.same_bits(p1.matrix.values, p8.matrix.values)
    assert p1.perturbation_norm == p8.perturbation_norm > 0.0
    assert_exactly_consistent(p1, rows=range(0, A.n_rows, 997))
