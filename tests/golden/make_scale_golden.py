"""Scale goldens for the parity-at-scale GPU tests (tests/test_gpu_scale.py).

The reference's own order -- cg_solve(..., partitions=1), its default
(cg.py:42; sequential dot _fast.py:342-356; bounds kernels.py:158-162) --
run by the pinned C oracle (bitwise equal to the reference on every golden in
tests/golden, see tests/test_oracle_golden.py) on the BASELINE configs the
reference itself cannot finish in a test budget (C2-C4, and a C5-style
instance at n = 1e6).  Recorded per (config, mode): iterations, reason, final
recurrence residual, TW-accurate true residual and forward error
(norm_metrics_tw, kernels.py:305-328), plus a SHA-256 of the generated matrix
so the GPU test can prove it solved the same problem.

    python tests/golden/make_scale_golden.py [--only C4:dw,C4:qtw] [--threads 8]

Resumable: entries already in scale.json are skipped.  C4 takes ~1-2 h per
mode on 8 host cores (1.4e5 iterations, two sequential n = 1e6 dots each).
"""
import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from paper_2510_13536_b200 import problems  # noqa: E402

OUT = os.path.join(HERE, "scale.json")
PLAN = [("C2", m) for m in ("fp64", "dw", "qdw", "qtw", "tw")] + \
       [("C3", m) for m in ("fp64", "dw", "qdw", "qtw")] + \
       [("C5s", m) for m in ("dw", "qtw")] + \
       [("C4s", m) for m in ("fp64", "dw", "qdw", "qtw", "tw")] + \
       [("C4", m) for m in ("dw", "qtw", "fp64", "qdw")] + [("C3", "tw"), ("C4", "tw")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=OUT, help="result file (merge several partial files by hand)")
    a = ap.parse_args()
    plan = PLAN
    if a.only:
        want = {tuple(s.split(":")) for s in a.only.split(",")}
        plan = [p for p in PLAN if p in want]
    orc.set_threads(a.threads)
    out = json.load(open(a.out)) if os.path.exists(a.out) else {}
    cache = {}
    for name, mode in plan:
        if mode in out.get(name, {}).get("runs", {}):
            continue
        if name not in cache:
            cache.clear()
            t = time.time()
            cache[name] = problems.CONFIGS[name]()
            print(name, "generated in %.1f s" % (time.time() - t), flush=True)
        cfg = cache[name]
        A = cfg["A"]
        ent = out.setdefault(name, {"n": A.n_rows, "nnz": A.nnz, "epsilon": cfg["epsilon"],
                                    "max_iterations": cfg["max_iterations"],
                                    "digest": problems.matrix_digest(A), "runs": {}})
        t = time.time()
        r = orc.cg_solve(A, cfg["b"], mode=mode, epsilon=cfg["epsilon"],
                         max_iterations=cfg["max_iterations"], history_stride=1 << 40,
                         partitions=1, reduction="partitions", x_star=cfg["x_star"])
        dt = time.time() - t
        k, rel, tres, err = r.history[-1]
        ent["runs"][mode] = {"iterations": r.iterations, "reason": r.reason,
                             "final_rel": r.final_recurrence_residual, "true_residual": tres,
                             "error_norm": err, "partitions": 1, "seconds": round(dt, 1),
                             "threads": a.threads}
        print(name, mode, json.dumps(ent["runs"][mode]), flush=True)
        json.dump(out, open(a.out, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
