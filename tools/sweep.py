"""Kernel-variant sweep: per-stage µs/iteration of the fused CG kernels for
libraries built with different compile-time knobs.

Build (here, CPU):   python tools/sweep.py build NAME -D MWCG_SP_U_OVERRIDE=8 ...
Run (GPU box):       python tools/sweep.py run --cfg C2 --modes dw,qtw [NAMES...]

Each variant runs in its own process (MWCG_LIB points at build_var/NAME.so);
the matrix is generated once per process.  Not a bench number: a tuning aid.
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VAR = os.path.join(ROOT, "build_var")
sys.path.insert(0, ROOT)


def do_build(name, defines):
    from paper_2510_13536_b200 import build as b
    os.makedirs(VAR, exist_ok=True)
    b.build(force=True, defines=defines, out=os.path.join(VAR, name + ".so"))
    with open(os.path.join(VAR, name + ".json"), "w") as f:
        json.dump(defines, f)


def child(cfg, modes, iters):
    import torch
    from paper_2510_13536_b200 import cg, problems
    t0 = time.time()
    c = problems.CONFIGS[cfg]()
    A, b = c["A"], c["b"]
    gen = time.time() - t0
    out = {"gen_s": round(gen, 1)}
    for mode in modes:
        conf_k = cg.SolverConfig(mode=mode, epsilon=1e-300, max_iterations=iters, history_stride=10**9,
                                 timing="kernels")
        cg.cg_solve(A, b, conf_k)  # warm (graph build, matrix upload)
        r = cg.cg_solve(A, b, conf_k)
        ks = {k: round(v / r.iterations * 1e6, 2) for k, v in r.kernel_seconds.items() if v}
        conf_g = cg.SolverConfig(mode=mode, epsilon=1e-300, max_iterations=iters, history_stride=10**9)
        cg.cg_solve(A, b, conf_g)
        best = 1e30
        for _ in range(3):
            rg = cg.cg_solve(A, b, conf_g)
            best = min(best, rg.device_seconds / rg.iterations * 1e6)
        out[mode] = {"stages_us": ks, "graph_us_per_iter": round(best, 2)}
        torch.cuda.synchronize()
    print("RESULT " + json.dumps(out), flush=True)


def do_run(cfg, modes, iters, names):
    names = names or ["default"]
    res = {}
    for nm in names:
        env = dict(os.environ)
        lib, _, envs = nm.partition(":")  # NAME[:VAR=V,VAR=V]
        if lib != "default":
            env["MWCG_LIB"] = os.path.join(VAR, lib + ".so")
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        p = subprocess.run([sys.executable, __file__, "child", "--cfg", cfg, "--modes", ",".join(modes),
                            "--iters", str(iters)], env=env, capture_output=True, text=True)
        line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT ")]
        if p.returncode or not line:
            res[nm] = {"error": (p.stderr or p.stdout)[-600:]}
        else:
            res[nm] = json.loads(line[-1][7:])
        print(nm, json.dumps(res[nm]), flush=True)
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["build", "run", "child"])
    ap.add_argument("names", nargs="*")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--cfg", default="C2")
    ap.add_argument("--modes", default="dw")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    if a.cmd == "build":
        do_build(a.names[0], a.defines)
    elif a.cmd == "child":
        child(a.cfg, a.modes.split(","), a.iters)
    else:
        r = do_run(a.cfg, a.modes.split(","), a.iters, a.names)
        if a.out:
            with open(a.out, "w") as f:
                json.dump(r, f, indent=1)
