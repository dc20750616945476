"""Generate tests/golden/cli.json from the REAL reference CLI (cli.py:135-331).
Build container only (needs /root/reference):

    python tests/golden/make_cli_golden.py

Each case runs `mwcg.cli.main(argv)` with --no-timing and an explicit --threads
(the reference's partition count), and stores the exit code and the bytes of
every file it wrote; `generate` cases store the Matrix Market outputs.  The
product CLI with the same argv (threads given -> the reference's partition
reduction order on the device) must write the same bytes.
"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import HERE, _import_reference  # noqa: E402

SOLVE = [
    ["solve", "--synthetic", "laplacian2d:8", "--mode", "dw", "--mode", "qtw", "--eps", "1e-24",
     "--threads", "2", "--stride", "10"],
    ["solve", "--synthetic", "laplacian2d:4", "--mode", "fp64", "--mode", "dw", "--mode", "qdw",
     "--mode", "tw", "--mode", "qtw", "--eps", "1e-10", "--threads", "1"],
    ["solve", "--synthetic", "scaled-laplacian2d:6", "--mode", "tw", "--mode", "qdw",
     "--eps", "1e-20", "--eps", "1e-8", "--threads", "3", "--stride", "7"],
    ["solve", "--synthetic", "random:30:7", "--mode", "fp64", "--mode", "dw", "--eps", "1e-12",
     "--threads", "1", "--normalize", "none", "--stride", "3"],
    ["solve", "--synthetic", "identity:5", "--threads", "1"],
    ["solve", "--synthetic", "laplacian2d:6", "--mode", "qdw", "--threads", "4",
     "--max-iters", "5", "--eps", "1e-30", "--stride", "2"],
]
# a symmetric Matrix Market input (lower triangle of a scaled Laplacian); the
# path is relative to the repo root because it is the `matrix` label in the outputs
MTX = os.path.join("tests", "golden", "cli_sym.mtx")
SOLVE += [
    ["solve", "--matrix", MTX, "--mode", "qtw", "--mode", "dw", "--eps", "1e-26", "--threads", "2",
     "--normalize", "every-op", "--stride", "4", "--reps", "2"],
    ["solve", "--matrix", MTX, "--mode", "tw", "--mode", "fp64", "--eps", "1e-14", "--threads", "5",
     "--normalize", "none"],
]
GENERATE = [
    ["generate", "--synthetic", "random:30:7"],
    ["generate", "--synthetic", "scaled-laplacian2d:5:3:8"],
]


def _write_fixture(sparse):
    A = sparse.scaled_laplacian_2d(7, 4.0, 5)
    ents = [(i, int(A.col_idx[k]), float(A.values[k])) for i in range(A.n_rows)
            for k in range(A.row_ptr[i], A.row_ptr[i + 1]) if A.col_idx[k] <= i]
    with open(os.path.join(HERE, "..", "..", MTX), "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n")
        f.write(f"{A.n_rows} {A.n_cols} {len(ents)}\n")
        for i, j, v in ents:
            f.write(f"{i + 1} {j + 1} {v!r}\n")


def main():
    _, _, _, _, sparse = _import_reference()
    _write_fixture(sparse)
    os.chdir(os.path.join(HERE, "..", ".."))
    from mwcg import cli
    cases = []
    with tempfile.TemporaryDirectory() as d:
        for argv in SOLVE:
            s, h, j = (os.path.join(d, f) for f in ("s.csv", "h.csv", "o.json"))
            full = argv + ["--no-timing", "--out-summary", s, "--out-history", h, "--json", j]
            code = cli.main(full)
            cases.append({"argv": argv, "code": code,
                          "files": {k: open(p).read() for k, p in
                                    (("summary", s), ("history", h), ("json", j))}})
        for argv in GENERATE:
            m, b = os.path.join(d, "m.mtx"), os.path.join(d, "b.mtx")
            code = cli.main(argv + ["--out-matrix", m, "--out-rhs", b])
            cases.append({"argv": argv, "code": code,
                          "files": {"matrix": open(m).read(), "rhs": open(b).read()}})
    out = os.path.join(HERE, "cli.json")
    with open(out, "w") as f:
        json.dump({"cases": cases}, f, indent=0)
    print("wrote", out, len(cases), "cases")


if __name__ == "__main__":
    main()
