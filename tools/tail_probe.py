"""K1 launch time with and without its serial tail (MWCG_NOTAIL), per mode."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_13536_b200 import problems
from paper_2510_13536_b200.cg import Solver, _b_norm, _time_k1
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = problems.CONFIGS[cfgname]()
A, b = cfg["A"], cfg["b"]
bd = torch.from_numpy(b).cuda(); bn = _b_norm(b)
for m in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("fp64", "dw", "qdw", "tw", "qtw")):
    s = Solver(A, m)
    os.environ.pop("MWCG_NOTAIL", None)
    full = min(_time_k1(s, bd, bn, reps=50) for _ in range(3))
    os.environ["MWCG_NOTAIL"] = "1"
    notail = min(_time_k1(s, bd, bn, reps=50) for _ in range(3))
    os.environ.pop("MWCG_NOTAIL", None)
    print(json.dumps({"config": cfgname, "mode": m, "k1_us": round(full, 2), "k1_notail_us": round(notail, 2),
                      "tail_us": round(full - notail, 2)}), flush=True)
