"""Time the STOCK reference (TEST / BASELINE INFRASTRUCTURE, never product code).

Runs the unmodified reference package `mwcg` (pip-installed into
baseline/_ref from /root/reference/pkg; Python + numba, single-threaded by
design -- SURVEY §0) through its own public API `mwcg.cg.cg_solve`, with the
gmpy2 shim in oracle/stock/.  One process per measurement, pinned to ONE
host core (the reference is single-threaded: `--threads` only changes its
dot-product shape, cli.py:20-25).

    python oracle/stock_reference.py --config C1 --mode dw [--iters K]

--iters K: K unconditional iterations (epsilon 1e-300, max_iterations K),
reported as a per-iteration time; without it, a full solve to the config's
epsilon.  Prints one JSON object.  The numba JIT is warmed on a 4x4 problem
first (not timed).
"""
import argparse
import json
import os
import platform
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.path.join(ROOT, "baseline", "_ref")


def available():
    return os.path.isdir(os.path.join(REF, "mwcg"))


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--mode", default="dw")
    ap.add_argument("--iters", type=int, default=0)
    a = ap.parse_args()
    try:
        core = sorted(os.sched_getaffinity(0))[-1]
        os.sched_setaffinity(0, {core})
    except (AttributeError, OSError):
        core = None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "mwcg_numba_cache"))
    os.environ["NUMBA_NUM_THREADS"] = "1"
    sys.path[:0] = [os.path.join(HERE, "stock"), REF, ROOT]
    import numpy as np
    from mwcg import cg as rcg, sparse as rsp  # the stock reference
    from paper_2510_13536_b200 import problems  # the pinned BASELINE generators

    cfg = problems.CONFIGS[a.config]()
    A0 = cfg["A"]
    A = rsp.CsrMatrix(A0.n_rows, A0.n_cols, np.array(A0.row_ptr), np.array(A0.col_idx),
                      np.array(A0.values))                      # reference validation (sparse.py:46-68)
    b = np.array(cfg["b"])
    # JIT warm-up on a tiny problem (numba compiles the mode's kernels)
    T = rsp.laplacian_2d(4)
    rcg.cg_solve(T, np.ones(16), rcg.SolverConfig(mode=a.mode, max_iterations=3))
    if a.iters:
        conf = rcg.SolverConfig(mode=a.mode, epsilon=1e-300, max_iterations=a.iters,
                                history_stride=10 ** 9)
    else:
        conf = rcg.SolverConfig(mode=a.mode, epsilon=cfg["epsilon"],
                                max_iterations=cfg["max_iterations"], history_stride=10 ** 9)
    t0 = time.perf_counter()
    r = rcg.cg_solve(A, b, conf)
    dt = time.perf_counter() - t0
    ks = sum(r.kernel_seconds.values())
    print(json.dumps({"config": a.config, "mode": a.mode, "iterations": r.iterations,
                      "reason": r.reason, "final_rel": r.final_recurrence_residual,
                      "seconds": dt, "s_per_iter": dt / max(1, r.iterations),
                      "kernel_seconds": ks, "full_solve": not a.iters, "cores": 1,
                      "core_id": core, "cpu_model": cpu_model(),
                      "impl": "stock reference mwcg 0.1.0 (Python + numba, baseline/_ref)"}))


if __name__ == "__main__":
    main()
