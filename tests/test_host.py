"""CPU-only tests: host-side API logic (mirrors pkg/tests/test_cg.py TestConfig,
pkg/tests/test_sparse.py validation), the C ABI library surface, the build
flags that parity depends on, and the problem generators."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2510_13536_b200 import _lib, problems
from paper_2510_13536_b200.cg import Normalization, SolverConfig
from paper_2510_13536_b200.sparse import (CsrMatrix, csr_from_coo, identity, laplacian_2d,
                                          random_symmetric, scaled_laplacian_2d)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mwcg_cuda.h")


# ------------------------------------------------------------------ config
class TestConfig:
    def test_defaults(self):
        c = SolverConfig()
        assert c.mode == "fp64" and c.epsilon == 1e-12
        assert c.normalization is Normalization.AFTER_RESIDUAL_AXPY
        assert c.history_stride == 100 and c.partitions == 1
        assert c.reduction == "tile"

    def test_string_normalization_coerced(self):
        assert SolverConfig(normalization="none").normalization is Normalization.NONE
        assert SolverConfig(normalization="every-op").normalization is Normalization.EVERY_VECTOR_OP

    @pytest.mark.parametrize("kw", [
        {"mode": "fp32"}, {"epsilon": 0.0}, {"epsilon": -1.0}, {"history_stride": 0},
        {"partitions": 0}, {"reduction": "warp"}, {"timing": "wall"},
        {"normalization": "sometimes"}])
    def test_rejects_bad_values(self, kw):
        with pytest.raises(ValueError):
            SolverConfig(**kw)


# ------------------------------------------------------------------ CSR
class TestCsr:
    def test_validation_messages(self):
        with pytest.raises(ValueError, match="row_ptr must have length"):
            CsrMatrix(2, 2, np.array([0, 1]), np.array([0]), np.array([1.0]))
        with pytest.raises(ValueError, match="start at 0"):
            CsrMatrix(1, 1, np.array([1, 1]), np.array([0]), np.array([1.0]))
        with pytest.raises(ValueError, match="non-decreasing"):
            CsrMatrix(2, 2, np.array([0, 2, 1]), np.array([0]), np.array([1.0]))
        with pytest.raises(ValueError, match="equal length"):
            CsrMatrix(1, 1, np.array([0, 1]), np.array([0]), np.array([1.0, 2.0]))
        with pytest.raises(ValueError, match="out of range"):
            CsrMatrix(1, 1, np.array([0, 1]), np.array([3]), np.array([1.0]))
        with pytest.raises(ValueError, match="row 1: column indices not strictly increasing"):
            CsrMatrix(2, 2, np.array([0, 1, 3]), np.array([0, 1, 1]), np.array([1.0, 1.0, 1.0]))
        with pytest.raises(ValueError, match="negative"):
            CsrMatrix(-1, 1, np.array([0]), np.array([], dtype=np.int64), np.array([]))

    def test_row_boundaries_not_flagged(self):
        # decreasing columns ACROSS a row boundary are fine
        A = CsrMatrix(2, 3, np.array([0, 2, 4]), np.array([1, 2, 0, 1]), np.ones(4))
        assert A.nnz == 4
        # and empty rows in between
        B = CsrMatrix(3, 3, np.array([0, 2, 2, 3]), np.array([1, 2, 0]), np.ones(3))
        assert B.nnz == 3

    def test_dtypes_and_dense(self):
        A = laplacian_2d(3)
        assert A.row_ptr.dtype == np.int64 and A.values.dtype == np.float64
        d = A.to_dense()
        assert np.allclose(d, d.T) and np.all(np.diag(d) == 4.0)
        assert A.diagonal_index(4) is not None
        assert identity(5).nnz == 5

    def test_laplacian_structure(self):
        A = laplacian_2d(256)
        assert A.n_rows == 65536 and A.nnz == 326656
        with pytest.raises(ValueError):
            laplacian_2d(1)

    def test_csr_from_coo_sums_duplicates(self):
        A = csr_from_coo(2, 2, [0, 0, 1, 0], [1, 1, 0, 0], [1.0, 2.0, 5.0, 7.0])
        assert A.to_dense().tolist() == [[7.0, 3.0], [5.0, 0.0]]

    def test_random_and_scaled_are_symmetric(self):
        R = random_symmetric(30, seed=2).to_dense()
        assert np.array_equal(R, R.T)
        S = scaled_laplacian_2d(5, decades=3.0, seed=1).to_dense()
        assert np.array_equal(S, S.T)


# ------------------------------------------------------------------ generators
class TestProblems:
    def test_spmv_fp64_host_is_sequential_unfused(self):
        A = CsrMatrix(1, 3, np.array([0, 3]), np.array([0, 1, 2]), np.array([1.0, 1e16, -1e16]))
        y = problems.spmv_fp64_host(A, np.array([1.0, 1.0, 1.0]))
        # ((0 + 1) + 1e16) + (-1e16) = 0 in FP64 left-to-right
        assert y[0] == 0.0

    def test_config2_shape(self):
        c = problems.config2(k=16)
        A = c["A"]
        assert A.n_rows == 16 ** 3
        assert A.nnz == 7 * 16 ** 3 - 6 * 16 ** 2
        assert np.all(c["b"] == problems.spmv_fp64_host(A, np.ones(A.n_rows)))
        assert np.allclose(A.to_dense(), A.to_dense().T)

    def test_config3_small_is_spd_dominant(self):
        c = problems.config3(k=6)
        d = c["A"].to_dense()
        assert np.array_equal(d, d.T)
        off = np.abs(d).sum(1) - np.abs(np.diag(d))
        assert np.all(np.diag(d) > off)

    def test_config4_small_is_symmetric_positive(self):
        c = problems.config4(n=300)
        d = c["A"].to_dense()
        assert np.array_equal(d, d.T)
        assert np.linalg.eigvalsh(d).min() > 0


# ------------------------------------------------------------------ C ABI
def _header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mwcg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    L = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 25
    for name in syms:
        assert hasattr(L, name), name
    # and the Python binding declares a signature for every one of them
    assert set(syms) == set(_lib.SIGNATURES)


def test_library_loads_without_gpu_and_reports_errors():
    L = _lib.load()
    assert L.mwcg_abi_version() == 1
    assert [L.mwcg_words(m) for m in range(5)] == [1, 2, 2, 3, 3]
    assert L.mwcg_words(9) == -1
    out = ctypes.c_double()
    v = np.array([3.0, 4.0])
    assert L.mwcg_norm2_host(v.ctypes.data_as(_lib.c_dp), 2, ctypes.byref(out)) == 0
    assert out.value == 5.0
    # bad argument -> MWCG_ERR_VALUE with a message, no crash
    assert L.mwcg_scalar_op(99, 1, None, None, None, None) == 1001
    assert b"bad mode or op" in L.mwcg_last_error()


def test_norm2_host_is_sequential_unfused():
    """norm2_fp64 (kernels.py:290-296): sequential, no FMA, no reassociation."""
    L = _lib.load()
    rng = np.random.default_rng(1)
    v = rng.standard_normal(1001) * np.exp(rng.uniform(-30, 30, 1001))
    s = 0.0
    for c in v:
        s = s + c * c
    out = ctypes.c_double()
    L.mwcg_norm2_host(v.ctypes.data_as(_lib.c_dp), v.size, ctypes.byref(out))
    assert out.value == float(np.sqrt(s))


def test_built_for_sm100a_without_contraction():
    from paper_2510_13536_b200 import build as b
    assert "arch=compute_100a,code=sm_100a" in " ".join(b.NVCC_FLAGS)
    assert "-fmad=false" in b.NVCC_FLAGS
    assert "--use_fast_math" not in b.NVCC_FLAGS
    sass = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in sass.stdout


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2510_13536_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower() or f == "__init__.py", f


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_13536_b200 import cg
    with pytest.raises(Exception):
        cg.cg_solve(laplacian_2d(3), np.ones(9), SolverConfig(mode="dw"))


def test_decimal_str_matches_reference():
    """DoubleWord/TripleWord.decimal_str (multiword.py:48-51, 71-75) against the
    reference's strings (tests/golden/decimal.json)."""
    from paper_2510_13536_b200.multiword import DoubleWord, TripleWord
    from tests.golden_io import load
    for c in load("decimal.json")["cases"]:
        dw = DoubleWord(*[float.fromhex(v) for v in c["dw"]])
        tw = TripleWord(*[float.fromhex(v) for v in c["tw"]])
        assert dw.decimal_str(c["digits"]) == c["dw_str"]
        assert tw.decimal_str(c["digits"]) == c["tw_str"]
        assert dw.decimal_str() == c["dw_default"] and tw.decimal_str() == c["tw_default"]
