"""Parity at scale (SURVEY §8(c) tier 3).

The reference CPU path cannot finish C3/C4 (days for TW).  The device's
reduction="partitions" mode is bitwise identical to the reference's
cg_solve(partitions=P) (pinned on C1 and the acceptance problems by
tests/test_gpu_parity.py), so it serves as the scale oracle: for each config
and arithmetic, solve in the reference order for several P (the reference's
own reduction-order band) and in the fast tile order, and record iteration
counts, final recurrence residual, TW-accurate true residual and forward
error.  north_star: tile-order iterations within +-2 % of the band, final
residual / error within 10x.

    python tools/scale_parity.py --configs C2,C4 --out gpurun_out/scale.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_13536_b200 import cg, problems  # noqa: E402


def run(cfg, mode, reduction, P, stride):
    conf = cg.SolverConfig(mode=mode, epsilon=cfg["epsilon"], max_iterations=cfg["max_iterations"],
                           history_stride=stride, reduction=reduction, partitions=P)
    t = time.perf_counter()
    r = cg.cg_solve(cfg["A"], cfg["b"], conf, x_star=cfg["x_star"])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    h = r.history[-1]
    return {"reduction": reduction, "P": P, "iterations": r.iterations, "reason": r.reason,
            "final_rel": r.final_recurrence_residual, "true_residual": h.true_residual,
            "error_norm": h.error_norm, "seconds": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C4")
    ap.add_argument("--modes", default="fp64,dw,qdw,tw,qtw")
    ap.add_argument("--parts", default="256,1024,4096")
    ap.add_argument("--out", default="gpurun_out/scale_parity.json")
    a = ap.parse_args()
    out = {}
    if os.path.exists(a.out):
        out = json.load(open(a.out))
    for name in a.configs.split(","):
        cfg = problems.CONFIGS[name]()
        out.setdefault(name, {"n": cfg["A"].n_rows, "nnz": cfg["A"].nnz,
                              "epsilon": cfg["epsilon"], "runs": {}})
        for mode in a.modes.split(","):
            rows = out[name]["runs"].setdefault(mode, [])
            done = {(r["reduction"], r["P"]) for r in rows}
            todo = [("tile", 1)] + [("partitions", int(p)) for p in a.parts.split(",")]
            for red, P in todo:
                if (red, P) in done:
                    continue
                rec = run(cfg, mode, red, P, 10 ** 9)
                rows.append(rec)
                print(name, mode, json.dumps(rec), flush=True)
                json.dump(out, open(a.out, "w"), indent=1)
        del cfg
        torch.cuda.empty_cache()
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
