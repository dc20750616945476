"""The `mwcg` command line on the device path (reference cli.py; tests restate
pkg/tests/test_cli.py and the CLI acceptance criteria of
pkg/tests/test_acceptance.py:268-300).

Parity: tests/golden/cli.json holds the bytes the REAL reference CLI wrote for
solve (--no-timing, explicit --threads) and generate; the product CLI with the
same argv must write the same bytes (solve: on the GPU, through the reference's
partition reduction order; generate: host, native problem generator).
"""
import csv
import json
import os

import numpy as np
import pytest

import tests.golden_io as G
from paper_2510_13536_b200 import cli
from paper_2510_13536_b200.sparse import read_matrix_market


def read_csv(path):
    with open(path, newline="", encoding="ascii") as f:
        return list(csv.reader(f))


# ---- exit codes and parsing (no GPU work) ----

@pytest.mark.parametrize("argv", [
    ["solve", "--synthetic", "identity:4", "--mode", "fp128"],
    ["solve"],
    ["solve", "--synthetic", "identity:4", "--eps", "0.0"],
    ["solve", "--synthetic", "identity:4", "--reps", "0"],
    ["solve", "--synthetic", "identity:4", "--threads", "0"],
    ["bench", "--synthetic", "identity:4", "--kernel", "gemm"],
    ["solve", "--synthetic", "identity:4", "--reduction", "pairwise"],
])
def test_usage_errors_exit_one(argv):
    with pytest.raises(SystemExit) as exc:
        cli.main(argv)
    assert exc.value.code == cli.EXIT_USAGE


def test_malformed_matrix_file_is_two(tmp_path, capsys):
    bad = tmp_path / "bad.mtx"
    bad.write_text("this is not a matrix\n1 1 1\n1 1 1.0\n")
    assert cli.main(["solve", "--matrix", str(bad)]) == cli.EXIT_INPUT
    assert "line 1" in capsys.readouterr().err


def test_input_errors_exit_two(tmp_path, capsys, monkeypatch):
    assert cli.main(["solve", "--matrix", str(tmp_path / "nope.mtx")]) == cli.EXIT_INPUT
    assert "cannot read" in capsys.readouterr().err
    assert cli.main(["solve", "--synthetic", "hilbert:5"]) == cli.EXIT_INPUT
    assert "unknown synthetic matrix 'hilbert'" in capsys.readouterr().err
    assert cli.main(["solve", "--synthetic", "identity:x"]) == cli.EXIT_INPUT
    assert "malformed synthetic spec 'identity:x'" in capsys.readouterr().err
    monkeypatch.setenv("MW_THREADS", "zebra")
    assert cli.main(["solve", "--synthetic", "identity:4"]) == cli.EXIT_INPUT
    assert "MW_THREADS='zebra' is not an integer" in capsys.readouterr().err


def test_non_square_and_generation_failure_are_two(tmp_path, capsys):
    m = tmp_path / "r.mtx"
    m.write_text("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1.0\n")
    assert cli.main(["solve", "--matrix", str(m)]) == cli.EXIT_INPUT
    assert "matrix is not square" in capsys.readouterr().err
    # pkg/tests/test_problemgen.py's missing-diagonal case: row 0 sums inexactly
    m.write_text("%%MatrixMarket matrix coordinate real general\n3 3 4\n"
                 "1 2 1152921504606846976.0\n1 3 1.0000000000000002\n"
                 "2 1 1152921504606846976.0\n3 1 1.0000000000000002\n")
    assert cli.main(["generate", "--matrix", str(m), "--out-matrix", str(tmp_path / "a"),
                     "--out-rhs", str(tmp_path / "b")]) == cli.EXIT_INPUT
    err = capsys.readouterr().err
    assert "problem generation failed: row 0: inexact row sum but no diagonal" in err


def test_version_flag(capsys):
    with pytest.raises(SystemExit) as exc:
        cli.main(["--version"])
    assert exc.value.code == 0
    assert capsys.readouterr().out.startswith("mwcg ")


def test_generate_matches_reference_bytes(tmp_path, capsys):
    for c in G.load("cli.json")["cases"]:
        if c["argv"][0] != "generate":
            continue
        m, b = tmp_path / "m.mtx", tmp_path / "b.mtx"
        assert cli.main(c["argv"] + ["--out-matrix", str(m), "--out-rhs", str(b)]) == c["code"]
        assert m.read_text() == c["files"]["matrix"], c["argv"]
        assert b.read_text() == c["files"]["rhs"], c["argv"]
        assert "perturbation norm" in capsys.readouterr().out


def test_generate_output_parses_back(tmp_path):
    om, orhs = tmp_path / "m.mtx", tmp_path / "b.mtx"
    assert cli.main(["generate", "--synthetic", "random:30:7", "--out-matrix", str(om),
                     "--out-rhs", str(orhs)]) == cli.EXIT_OK
    m, symmetric = read_matrix_market(str(om))
    assert not symmetric and m.n_rows == 30
    lines = orhs.read_text().splitlines()
    assert lines[0].startswith("%%MatrixMarket matrix array") and lines[1] == "30 1"
    assert np.array([float(v) for v in lines[2:]]).size == 30


def test_solve_without_gpu_fails_loudly():
    """No CPU fallback: without a device the solve raises instead of computing."""
    import torch
    from paper_2510_13536_b200._lib import MwcgError
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(MwcgError, match="no CPU fallback"):
        cli.main(["solve", "--synthetic", "identity:4"])


# ---- device runs ----

@pytest.mark.gpu
def test_solve_matches_reference_bytes(tmp_path, monkeypatch):
    """--no-timing + --threads P: the device solve in the reference's P-partition
    order writes the reference CLI's summary, history and JSON byte for byte
    (synthetic inputs and a symmetric Matrix Market file)."""
    monkeypatch.chdir(os.path.dirname(G.GOLDEN.rstrip("/")) + "/..")
    n = 0
    for c in G.load("cli.json")["cases"]:
        if c["argv"][0] != "solve":
            continue
        s, h, j = tmp_path / "s.csv", tmp_path / "h.csv", tmp_path / "o.json"
        code = cli.main(c["argv"] + ["--no-timing", "--out-summary", str(s), "--out-history",
                                     str(h), "--json", str(j)])
        assert code == c["code"]
        assert s.read_text() == c["files"]["summary"], c["argv"]
        assert h.read_text() == c["files"]["history"], c["argv"]
        assert j.read_text() == c["files"]["json"], c["argv"]
        n += 1
    assert n == 8


@pytest.mark.gpu
def test_identity_single_row(tmp_path):
    out = tmp_path / "s.csv"
    assert cli.main(["solve", "--synthetic", "identity:5", "--out-summary", str(out)]) == 0
    rows = read_csv(out)
    assert rows[0][:3] == ["matrix", "mode", "eps"] and len(rows) == 2
    rec = dict(zip(rows[0], rows[1]))
    assert rec["mode"] == "fp64" and rec["converged"] == "1"
    assert int(rec["iterations"]) <= 1 and float(rec["final_error_norm"]) == 0.0
    assert "seconds" in rows[0]


@pytest.mark.gpu
def test_five_modes_best_marker_and_history(tmp_path):
    s, h = tmp_path / "s.csv", tmp_path / "h.csv"
    argv = ["solve", "--synthetic", "laplacian2d:4", "--eps", "1e-10", "--no-timing",
            "--out-summary", str(s)]
    for m in ("fp64", "dw", "qdw", "tw", "qtw"):
        argv += ["--mode", m]
    assert cli.main(argv) == 0
    rows = read_csv(s)
    assert len(rows) == 6 and "seconds" not in rows[0]
    assert len([r for r in rows[1:] if r[rows[0].index("best")] == "1"]) == 1
    assert cli.main(["solve", "--synthetic", "laplacian2d:4", "--mode", "dw", "--eps", "1e-20",
                     "--stride", "5", "--out-summary", str(s), "--out-history", str(h)]) == 0
    iters = int(dict(zip(*read_csv(s)[:2]))["iterations"])
    ks = [int(r[3]) for r in read_csv(h)[1:]]
    assert ks[0] == 0 and ks[-1] == iters
    assert len(ks) == len(range(5, iters, 5)) + 2


@pytest.mark.gpu
def test_no_timing_byte_identical_tile_order(tmp_path):
    """Default (device tile-tree) order is deterministic too (acceptance criterion 09)."""
    outs = []
    for name in ("a", "b"):
        s, h = tmp_path / f"s-{name}.csv", tmp_path / f"h-{name}.csv"
        assert cli.main(["solve", "--synthetic", "laplacian2d:8", "--mode", "dw", "--mode", "qtw",
                         "--eps", "1e-24", "--stride", "10", "--no-timing",
                         "--out-summary", str(s), "--out-history", str(h)]) == 0
        outs.append(s.read_bytes() + h.read_bytes())
    assert outs[0] == outs[1]


@pytest.mark.gpu
def test_json_and_stdout(tmp_path, capsys):
    j = tmp_path / "out.json"
    assert cli.main(["solve", "--synthetic", "laplacian2d:3", "--mode", "tw", "--eps", "1e-30",
                     "--json", str(j), "--out-summary", str(tmp_path / "s.csv")]) == 0
    payload = json.loads(j.read_text())
    assert payload["n"] == 9 and payload["matrix"] == "laplacian2d:3"
    (entry,) = payload["runs"]
    assert entry["mode"] == "tw" and entry["converged"] is True
    assert entry["history"][0][0] == 0 and "seconds" in entry and "kernel_seconds" in entry
    assert cli.main(["solve", "--synthetic", "identity:3", "--no-timing"]) == 0
    assert capsys.readouterr().out.splitlines()[0].startswith("matrix,mode,eps")


@pytest.mark.gpu
def test_bench_csv(tmp_path, capsys):
    out = tmp_path / "b.csv"
    assert cli.main(["bench", "--synthetic", "laplacian2d:4", "--kernel", "spmv", "--mode",
                     "fp64", "--mode", "dw", "--reps", "2", "--out-summary", str(out)]) == 0
    rows = read_csv(out)
    assert rows[0] == ["matrix", "kernel", "mode", "n", "nnz", "seconds_best", "bytes_model",
                       "gbps"]
    assert len(rows) == 3 and rows[1][2] == "fp64" and rows[2][2] == "dw"
    assert int(rows[1][3]) == 16 and float(rows[1][5]) > 0
    assert cli.main(["bench", "--synthetic", "identity:100", "--kernel", "dot", "--mode", "tw",
                     "--reps", "1", "--out-summary", str(out)]) == 0
    assert int(read_csv(out)[1][6]) == 2 * 100 * 3 * 8
    assert cli.main(["bench", "--synthetic", "identity:10", "--kernel", "dot", "--reps", "1"]) == 0
    assert ",fp64," in capsys.readouterr().out


@pytest.mark.gpu
def test_verify_passes(capsys):
    assert cli.main(["verify"]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "FAIL" not in out and "checks passed" in out


@pytest.mark.gpu
def test_threads_env_fallback_matches_reference(tmp_path, monkeypatch):
    """MW_THREADS stands in for --threads (cli.py:110-120): same bytes as the
    reference CLI's --threads 2 run."""
    c = next(c for c in G.load("cli.json")["cases"] if "--threads" in c["argv"]
             and c["argv"][c["argv"].index("--threads") + 1] == "2")
    argv = list(c["argv"])
    i = argv.index("--threads")
    del argv[i:i + 2]
    monkeypatch.setenv("MW_THREADS", "2")
    s, h = tmp_path / "s.csv", tmp_path / "h.csv"
    assert cli.main(argv + ["--no-timing", "--out-summary", str(s), "--out-history", str(h)]) == 0
    assert s.read_text() == c["files"]["summary"]
    assert h.read_text() == c["files"]["history"]
