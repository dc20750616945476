"""A/B sweep of the K1 variants on one config: for each environment variant
(MWCG_K1W, MWCG_K1W_NC, MWCG_K1W_R ...) and arithmetic, the K1 launch time
(20 back-to-back launches, CUDA events) and the µs per CG iteration of a full
solve (graph loop, device-resident inputs).

    python tools/k1w_sweep.py --config C2 --modes dw,qtw \
        --variants 'MWCG_K1W=0;MWCG_K1W=1,MWCG_K1W_NC=512;MWCG_K1W=1,MWCG_K1W_NC=256'
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_13536_b200 import problems  # noqa: E402
from paper_2510_13536_b200.cg import Solver, _b_norm, _time_k1  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--modes", default="fp64,dw,qdw,tw,qtw")
    ap.add_argument("--variants", default="MWCG_K1W=0;MWCG_K1W=1")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfg = problems.CONFIGS[a.config]()
    A, b = cfg["A"], cfg["b"]
    bd = torch.from_numpy(b).cuda()
    bn = _b_norm(b)
    rows = []
    for var in a.variants.split(";"):
        env = dict(kv.split("=") for kv in var.split(",") if kv)
        for m in a.modes.split(","):
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                A.release_device()
                s = Solver(A, m)
                d = s.describe()
            finally:
                for k, v in old.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
            k1 = _time_k1(s, bd, bn, reps=20)
            s.solve(bd, bn, None, None, cfg["epsilon"], cfg["max_iterations"], 10**9)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r, _ = s.solve(bd, bn, None, None, cfg["epsilon"], cfg["max_iterations"], 10**9)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e-3
            pr, _ = s.solve(bd, bn, None, None, cfg["epsilon"], cfg["max_iterations"], 10**9, profile=True)
            it = max(1, pr.iterations)
            row = {"config": a.config, "variant": var, "mode": m, "k1_us": round(k1, 2),
                   "us_per_iter": round(1e6 * t / max(1, r.iterations), 2), "iterations": r.iterations,
                   "stage_us": [round(1e3 * pr.stage_ms[i] / it, 2) for i in range(3)], "describe": d}
            rows.append(row)
            print(json.dumps(row), flush=True)
            del s
            torch.cuda.empty_cache()
    if a.out:
        json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
