"""GPU parity: the CUDA path (libmwcg_cuda.so) against the golden vectors of
the real reference and against the C oracle, bit for bit.

Two solver orders are checked:
  * reduction="partitions" (reference=True): the reference's own dot order;
    the device solve must equal the reference's cg_solve bitwise (golden).
  * reduction="tile": the fast device order; must equal the oracle's
    tile-tree restatement bitwise, and its iteration counts must sit inside
    the reference's own reduction-order band (north_star: +-2 %).
"""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402
from paper_2510_13536_b200 import cg, kernels as K, multiword, problems  # noqa: E402
from paper_2510_13536_b200.sparse import (CsrMatrix, identity, laplacian_2d,  # noqa: E402
                                          random_symmetric, scaled_laplacian_2d)
from tests.golden_io import arr, csr, fh, load, planes, same_bits  # noqa: E402

OPS = load("ops.json")
KER = load("kernels.json")
SMALL = load("cg_small.json")
C1 = load("cg_c1.json")
ACC = load("cg_accept.json")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _csrm(d):
    m = csr(d)
    return CsrMatrix(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values)


def _vec(mode, pl):
    return K.MultiwordVector.from_planes(pl, mode)


# ------------------------------------------------------------------ scalar ops
@pytest.mark.parametrize("mode", ["dw", "qdw", "tw", "qtw"])
def test_scalar_ops_golden(mode):
    w = orc.WORDS[mode]
    for c in (c for c in OPS["ops"] if c["mode"] == mode):
        a, b = arr(c["a"]), arr(c["b"])
        for op in ("add", "mul", "dxmul", "dxadd", "normalize", "div"):
            if op not in c:
                continue
            opmode = "qdw" if (op == "normalize" and mode == "dw") else mode
            got = multiword.scalar_op(op, opmode, a, b)[:w]
            assert same_bits(got, arr(c[op])), (mode, op, c["a"], c["b"])


def test_eft_golden():
    for c in OPS["eft"][:60]:
        a, b = [fh(c["a"])], [fh(c["b"])]
        for op in ("two_sum", "quick_two_sum", "two_prod"):
            assert same_bits(multiword.scalar_op(op, "dw", a, b)[:2], arr(c[op]))


# ------------------------------------------------------------------ kernels
@pytest.mark.parametrize("mode", orc.MODES)
def test_kernels_golden(mode):
    mats = {k: _csrm(v) for k, v in KER["matrices"].items()}
    for c in (c for c in KER["cases"] if c["mode"] == mode):
        op = c["op"]
        if op == "spmv":
            y = K.spmv(mats[c["matrix"]], _vec(mode, planes(c["x"])))
            assert same_bits(y.planes.cpu().numpy(), planes(c["y"])), (mode, op)
        elif op == "dot":
            d = K.dot(_vec(mode, planes(c["x"])), _vec(mode, planes(c["y"])),
                      partitions=c["partitions"])
            d = [d] if mode == "fp64" else list(d)
            assert same_bits(d, arr(c["out"])), (mode, c["partitions"])
        elif op == "axpy":
            y = _vec(mode, planes(c["y"]))
            alpha = arr(c["alpha"])
            K.axpy(alpha[0] if mode == "fp64" else alpha, _vec(mode, planes(c["x"])), y)
            assert same_bits(y.planes.cpu().numpy(), planes(c["out"]))
        elif op == "scal_add":
            p = _vec(mode, planes(c["p"]))
            beta = arr(c["beta"])
            K.scal_then_add(beta[0] if mode == "fp64" else beta, p, _vec(mode, planes(c["r"])))
            assert same_bits(p.planes.cpu().numpy(), planes(c["out"]))
        elif op == "residual":
            r = K.residual(arr(c["b"]), _vec(mode, planes(c["q"])))
            assert same_bits(r.planes.cpu().numpy(), planes(c["out"]))
        elif op == "normalize":
            v = _vec(mode, planes(c["v"]))
            K.normalize_vector(v)
            assert same_bits(v.planes.cpu().numpy(), planes(c["out"]))
        elif op == "norm2":
            assert same_bits(K.norm2_fp64(_vec(mode, planes(c["v"]))), fh(c["out"]))
        elif op == "metrics":
            err, tr = K.norm_metrics_tw(_vec(mode, planes(c["x"])), arr(c["x_star"]),
                                        mats[c["matrix"]], arr(c["b"]))
            assert same_bits(err, fh(c["err"])) and same_bits(tr, fh(c["true_res"]))


@pytest.mark.parametrize("mode", orc.MODES)
@pytest.mark.parametrize("n", [0, 1, 31, 1023, 1024, 1025, 70001, 3_000_017])
def test_dot_tile_matches_oracle(mode, n):
    rng = np.random.default_rng(n + 7)
    w = orc.WORDS[mode]
    x = rng.standard_normal((w, n)) * np.array([1.0, 1e-17, 1e-34][:w])[:, None]
    y = rng.standard_normal((w, n)) * np.array([1.0, 1e-17, 1e-34][:w])[:, None]
    d = K.dot(_vec(mode, x), _vec(mode, y), partitions=0)
    want = orc.dot(mode, x, y, tile=(orc.TILE_THREADS, orc.TILE_ELEMS))
    assert same_bits([d] if mode == "fp64" else list(d), want)


@pytest.mark.parametrize("mode", orc.MODES)
def test_spmv_large_matches_oracle(mode):
    """Full BASELINE config-2 matrix (128^3, 14.6M nnz): device SpMV == oracle."""
    c = problems.config2()
    A = c["A"]
    rng = np.random.default_rng(3)
    w = orc.WORDS[mode]
    x = rng.standard_normal((w, A.n_rows)) * np.array([1.0, 1e-17, 1e-34][:w])[:, None]
    orc.set_threads(orc.max_threads())
    want = orc.spmv(mode, A, x)
    got = K.spmv(A, _vec(mode, x)).planes.cpu().numpy()
    assert same_bits(got, want)


# ------------------------------------------------------------------ solver
def _run_small(run, **extra):
    prob = SMALL["problems"][run["problem"]]
    A = _csrm(prob["A"])
    b = arr(prob["b"])
    xs = None if prob["x_star"] is None else arr(prob["x_star"])
    cfg = dict(run["config"])
    x0 = None if run["x0"] is None else arr(run["x0"])
    conf = cg.SolverConfig(**cfg, **extra)
    return A, b, xs, x0, cfg, cg.cg_solve(A, b, conf, x0=x0, x_star=xs)


def _check(got, want, x_bits=True):
    assert got.iterations == want["iterations"]
    assert got.reason == want["reason"]
    assert same_bits(got.final_recurrence_residual, fh(want["final_rel"]))
    assert len(got.history) == len(want["history"])
    for g, h in zip(got.history, want["history"]):
        assert g.iteration == h[0]
        assert same_bits(g.recurrence_residual, fh(h[1]))
        assert same_bits(g.true_residual, fh(h[2]))
        assert (g.error_norm is None) == (h[3] is None)
        if h[3] is not None:
            assert same_bits(g.error_norm, fh(h[3]))
    if x_bits and "x" in want:
        assert same_bits(got.x.planes.cpu().numpy(), planes(want["x"]))


@pytest.mark.parametrize("idx", range(len(SMALL["runs"])))
def test_cg_small_reference_order_golden(idx):
    run = SMALL["runs"][idx]
    *_, res = _run_small(run, reduction="partitions")
    _check(res, run["result"])


def _oracle_tile(A, b, cfg, x0=None, xs=None):
    return orc.cg_solve(A, b, mode=cfg.get("mode", "fp64"), epsilon=cfg["epsilon"],
                        max_iterations=cfg.get("max_iterations"),
                        normalization=cfg.get("normalization", "after-axpy"),
                        history_stride=cfg.get("history_stride", 100), reduction="tile",
                        x0=x0, x_star=xs)


def _check_vs_oracle(got, o):
    assert got.iterations == o.iterations and got.reason == o.reason
    assert same_bits(got.final_recurrence_residual, o.final_recurrence_residual)
    assert len(got.history) == len(o.history)
    for g, h in zip(got.history, o.history):
        assert g.iteration == h[0]
        assert same_bits([g.recurrence_residual, g.true_residual], [h[1], h[2]])
        if h[3] is not None:
            assert same_bits(g.error_norm, h[3])
    assert same_bits(got.x.planes.cpu().numpy(), o.x)


@pytest.mark.parametrize("idx", range(len(SMALL["runs"])))
def test_cg_small_tile_matches_oracle(idx):
    run = SMALL["runs"][idx]
    A, b, xs, x0, cfg, res = _run_small(run, reduction="tile")
    _check_vs_oracle(res, _oracle_tile(A, b, cfg, x0, xs))


@pytest.mark.parametrize("mode", orc.MODES)
def test_c1_reference_order_golden(mode):
    c = problems.config1()
    run = next(r for r in C1["runs"] if r["mode"] == mode)
    res = cg.cg_solve(c["A"], c["b"], cg.SolverConfig(mode=mode, epsilon=1e-12,
                                                       max_iterations=10000, history_stride=100),
                      x_star=c["x_star"], reference=True)
    _check(res, run["result"], x_bits=False)
    assert _sha(res.x.planes.cpu().numpy()) == run["result"]["x_sha256"]


@pytest.mark.parametrize("mode", orc.MODES)
def test_c1_tile_matches_oracle_and_band(mode):
    c = problems.config1()
    cfg = dict(mode=mode, epsilon=1e-12, max_iterations=10000, history_stride=100)
    res = cg.cg_solve(c["A"], c["b"], cg.SolverConfig(**cfg), x_star=c["x_star"])
    orc.set_threads(orc.max_threads())
    _check_vs_oracle(res, _oracle_tile(c["A"], c["b"], cfg, None, c["x_star"]))
    ref = next(r for r in C1["runs"] if r["mode"] == mode)["result"]
    assert abs(res.iterations - ref["iterations"]) <= 0.02 * ref["iterations"]
    ref_err = fh(ref["history"][-1][3])
    assert res.history[-1].error_norm <= 10 * ref_err
    assert res.final_recurrence_residual <= 10 * fh(ref["final_rel"])


def _hard():
    return _csrm(ACC["hard_problem"]["A"]), arr(ACC["hard_problem"]["b"])


@pytest.mark.parametrize("mode", ["dw", "qdw", "tw", "qtw"])
def test_acceptance_hard_tile_band(mode):
    """kappa ~ 3e8, eps 1e-24: iterations within the reference's band over
    partitions {1,2,8,37,148} widened by 2 %; accuracy within
    10x; bitwise equal to the oracle's tile-tree restatement."""
    A, b = _hard()
    cfg = dict(mode=mode, epsilon=1e-24, max_iterations=20000, history_stride=100)
    res = cg.cg_solve(A, b, cg.SolverConfig(**cfg), x_star=np.ones(A.n_rows))
    _check_vs_oracle(res, _oracle_tile(A, b, cfg, None, np.ones(A.n_rows)))
    band = [r["result"] for r in ACC["runs"] if r["problem"] == "hard" and r["mode"] == mode
            and r["normalization"] == "after-axpy"]
    its = [r["iterations"] for r in band]
    assert min(its) * 0.98 <= res.iterations <= max(its) * 1.02
    assert res.converged
    worst_err = max(fh(r["history"][-1][3]) for r in band)
    assert res.history[-1].error_norm <= 10 * worst_err


@pytest.mark.parametrize("mode", orc.MODES)
def test_acceptance_easy_tile(mode):
    """Criterion 6 accuracy ordering (test_acceptance.py:206-220) on the device."""
    A = laplacian_2d(64)
    b = problems.spmv_fp64_host(A, np.ones(A.n_rows))
    res = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, epsilon=1e-32), x_star=np.ones(A.n_rows))
    err = res.history[-1].error_norm
    if mode == "fp64":
        assert 1e-17 <= err <= 1e-12
    elif mode in ("dw", "qdw"):
        assert err <= 1e-22
    else:
        assert err <= 1e-28
    # iteration parity against the reference's own reduction-order band: the
    # oracle (pinned to the reference by tests/golden) over P in {1,2,8,37,148}
    its = [orc.cg_solve(A, b, mode=mode, epsilon=1e-32, partitions=P, record_history=False,
                        x_star=np.ones(A.n_rows)).iterations for P in (1, 2, 8, 37, 148)]
    ref = next(r for r in ACC["runs"] if r["problem"] == "easy" and r["mode"] == mode)["result"]
    assert its[0] == ref["iterations"]
    assert min(its) * 0.98 <= res.iterations <= max(its) * 1.02


@pytest.mark.parametrize("mode", ["qdw", "qtw"])
def test_quasi_without_normalization_fails(mode):
    """Criterion 7 (test_acceptance.py:223-241): without normalization the
    quasi modes never reach 1e-24 on the kappa~3e8 problem."""
    A, b = _hard()
    bare = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, epsilon=1e-24, max_iterations=20000,
                                             normalization="none"), x_star=np.ones(A.n_rows))
    assert not bare.converged
    assert min(h.true_residual for h in bare.history) > 1e-24


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("mode", orc.MODES)
@pytest.mark.parametrize("reduction", ["tile", "partitions"])
def test_identity_and_edge_cases(mode, reduction):
    A = identity(6)
    b = np.arange(1.0, 7.0)
    res = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, reduction=reduction))
    assert res.converged and res.iterations <= 1
    assert np.array_equal(res.x.to_fp64(), b)
    A2 = CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([4.0, 1.0, 1.0, 3.0]))
    z = cg.cg_solve(A2, np.zeros(2), cg.SolverConfig(mode=mode, reduction=reduction))
    assert z.converged and z.iterations == 0 and np.array_equal(z.x.to_fp64(), np.zeros(2))
    ws = cg.cg_solve(A2, np.array([1.0, 2.0]), cg.SolverConfig(mode=mode, epsilon=1e-10,
                                                              reduction=reduction),
                     x0=np.array([1 / 11, 7 / 11]))
    assert ws.converged and ws.iterations == 0
    Ab = CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, -1.0]))
    bd = cg.cg_solve(Ab, np.array([1.0, 1.0]), cg.SolverConfig(mode=mode, reduction=reduction))
    assert bd.reason == "breakdown" and bd.iterations == 0
    mi = cg.cg_solve(laplacian_2d(4), np.ones(16), cg.SolverConfig(mode=mode, epsilon=1e-300,
                                                                   max_iterations=2,
                                                                   reduction=reduction))
    assert mi.reason == "max_iterations" and mi.iterations == 2


def test_empty_system():
    A = CsrMatrix(0, 0, np.array([0]), np.array([], dtype=np.int64), np.array([]))
    res = cg.cg_solve(A, np.zeros(0), cg.SolverConfig(mode="dw"))
    assert res.converged and res.iterations == 0 and len(res.x) == 0


def test_ragged_rows_and_empty_rows():
    """Rows of very different lengths (incl. > 32 entries and a zero row
    handled by a unit diagonal) through SELL-32: device == oracle."""
    rng = np.random.default_rng(5)
    n = 300
    rows, cols, vals = [], [], []
    for i in range(n):
        k = [0, 1, 3, 40, 90][i % 5]
        js = rng.choice(n, size=min(k, n), replace=False)
        for j in js:
            if j != i:
                v = -rng.uniform(0.1, 1.0)
                rows += [i, j]
                cols += [j, i]
                vals += [v, v]
    from paper_2510_13536_b200.sparse import csr_from_coo
    off = csr_from_coo(n, n, rows, cols, vals)
    absrow = np.zeros(n)
    np.add.at(absrow, np.repeat(np.arange(n), np.diff(off.row_ptr)), np.abs(off.values))
    d = np.arange(n)
    A = csr_from_coo(n, n, np.concatenate([np.repeat(np.arange(n), np.diff(off.row_ptr)), d]),
                     np.concatenate([off.col_idx, d]), np.concatenate([off.values, absrow + 1.0]))
    b = rng.standard_normal(n)
    for mode in orc.MODES:
        x = rng.standard_normal((orc.WORDS[mode], n))
        assert same_bits(K.spmv(A, _vec(mode, x)).planes.cpu().numpy(), orc.spmv(mode, A, x))
        cfg = dict(mode=mode, epsilon=1e-20 if mode != "fp64" else 1e-13, history_stride=7)
        res = cg.cg_solve(A, b, cg.SolverConfig(**cfg))
        _check_vs_oracle(res, _oracle_tile(A, b, cfg))


@pytest.mark.parametrize("mode", orc.MODES)
def test_repeat_runs_identical(mode):
    c = problems.config1()
    cfg = cg.SolverConfig(mode=mode, epsilon=1e-12, history_stride=1000)
    a = cg.cg_solve(c["A"], c["b"], cfg)
    b2 = cg.cg_solve(c["A"], c["b"], cfg)
    assert a.iterations == b2.iterations
    assert same_bits(a.x.planes.cpu().numpy(), b2.x.planes.cpu().numpy())


def test_profiled_timing_matches_graph_bits():
    c = problems.config1()
    g = cg.cg_solve(c["A"], c["b"], cg.SolverConfig(mode="dw", history_stride=1000))
    p = cg.cg_solve(c["A"], c["b"], cg.SolverConfig(mode="dw", history_stride=1000,
                                                    timing="kernels"))
    assert g.iterations == p.iterations
    assert same_bits(g.x.planes.cpu().numpy(), p.x.planes.cpu().numpy())
    assert p.kernel_seconds["spmv"] > 0 and p.kernel_seconds["axpy"] > 0
    assert sum(p.kernel_seconds.values()) <= p.elapsed_seconds


@pytest.mark.parametrize("mode", orc.MODES)
def test_c2_full_size_iterations_bitwise(mode):
    """Full BASELINE config 2 (n = 2.1M): 4 device iterations (tile order)
    equal the oracle's 4 iterations bit for bit (x words)."""
    c = problems.config2()
    A, b = c["A"], c["b"]
    res = cg.cg_solve(A, b, cg.SolverConfig(mode=mode, epsilon=1e-300, max_iterations=4,
                                            history_stride=10**9))
    orc.set_threads(orc.max_threads())
    o = orc.cg_solve(A, b, mode=mode, epsilon=1e-300, max_iterations=4, history_stride=10**9,
                     reduction="tile", record_history=False)
    assert res.iterations == o.iterations == 4
    assert same_bits(res.x.planes.cpu().numpy(), o.x)
    assert same_bits(res.final_recurrence_residual, o.final_recurrence_residual)


@pytest.mark.parametrize("mode", orc.MODES)
def test_int16_delta_and_int32_columns_agree(mode):
    """The three matrix layouts (slice-shared offsets, int16 column deltas,
    int32 columns) give the same bits; the stencil picks slice-shared
    offsets automatically and a matrix with far columns falls back to
    int32."""
    c = problems.config1()
    A = c["A"]
    mats = {f: CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values) for f in (-1, 1, 0, 2)}
    assert K.device_matrix(mats[-1]).col_bytes() == 0
    assert K.device_matrix(mats[1], col_format=1).col_bytes() == 2
    assert K.device_matrix(mats[0], col_format=0).col_bytes() == 4
    assert K.device_matrix(mats[2], col_format=2).col_bytes() == 0
    rng = np.random.default_rng(11)
    x = rng.standard_normal((orc.WORDS[mode], A.n_rows))
    ys = [K.spmv(m, _vec(mode, x)).planes.cpu().numpy() for m in mats.values()]
    want = orc.spmv(mode, A, x)
    assert all(same_bits(y, want) for y in ys)
    far = random_symmetric(40000, extra_per_row=2, seed=3)
    assert K.device_matrix(far).col_bytes() == 4
    xf = rng.standard_normal((orc.WORDS[mode], far.n_rows))
    assert same_bits(K.spmv(far, _vec(mode, xf)).planes.cpu().numpy(), orc.spmv(mode, far, xf))


def _banded_with_holes(n, half, seed, drop):
    """Banded SPD-ish matrix whose rows miss random off-diagonal entries
    (slices mix several offset patterns), including rows with only the
    diagonal and a partial last slice."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        for o in range(-half, half + 1):
            j = i + o
            if 0 <= j < n and (o == 0 or rng.random() > drop):
                rows.append(i)
                cols.append(j)
                vals.append(4.0 * half if o == 0 else rng.uniform(-1.0, 0.0))
    order = np.lexsort((cols, rows))
    r, c, v = np.array(rows)[order], np.array(cols)[order], np.array(vals)[order]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    return CsrMatrix(n, n, np.cumsum(rp), c.astype(np.int64), v)


@pytest.mark.parametrize("mode", orc.MODES)
def test_slice_shared_offsets_edge_cases(mode):
    """Slice-shared offsets (forced) on slices that mix offset patterns,
    rows holding only the diagonal and a partial last slice: SpMV bitwise
    equal to the oracle and to the int32 SELL layout."""
    A = _banded_with_holes(1000 + 13, 3, seed=5, drop=0.35)
    Ad = CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values)
    As = CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values)
    assert K.device_matrix(Ad, col_format=2).col_bytes() == 0
    assert K.device_matrix(As, col_format=0).col_bytes() == 4
    rng = np.random.default_rng(12)
    x = rng.standard_normal((orc.WORDS[mode], A.n_rows))
    yd = K.spmv(Ad, _vec(mode, x)).planes.cpu().numpy()
    ys = K.spmv(As, _vec(mode, x)).planes.cpu().numpy()
    assert same_bits(yd, orc.spmv(mode, A, x)) and same_bits(yd, ys)


@pytest.mark.parametrize("mode", ["dw", "qtw"])
def test_slice_shared_offsets_solve_equals_sell(mode):
    """A whole CG solve gives the same bits in the slice-shared-offset and
    the SELL layouts."""
    A = _banded_with_holes(3000, 4, seed=7, drop=0.2)
    b = problems.spmv_fp64_host(A, np.ones(A.n_rows))
    conf = cg.SolverConfig(mode=mode, epsilon=1e-20, history_stride=50)
    got = []
    for fmt in (2, 1):
        Af = CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values)
        K.device_matrix(Af, col_format=fmt)
        got.append(cg.cg_solve(Af, b, conf, x_star=np.ones(A.n_rows)))
    assert got[0].iterations == got[1].iterations and got[0].reason == got[1].reason
    assert same_bits(got[0].x.planes.cpu().numpy(), got[1].x.planes.cpu().numpy())
    assert [(h.iteration, h.recurrence_residual) for h in got[0].history] == \
        [(h.iteration, h.recurrence_residual) for h in got[1].history]


def test_slice_shared_offsets_rejected_and_forced_error():
    """Random columns: the automatic choice falls back to SELL; forcing the
    slice-shared layout is a ValueError (too many distinct offsets)."""
    far = random_symmetric(4000, extra_per_row=6, seed=9)
    assert K.device_matrix(CsrMatrix(far.n_rows, far.n_cols, far.row_ptr, far.col_idx,
                                     far.values)).col_bytes() in (2, 4)
    with pytest.raises(ValueError):
        K.device_matrix(CsrMatrix(far.n_rows, far.n_cols, far.row_ptr, far.col_idx, far.values),
                        col_format=2)
