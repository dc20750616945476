"""Phase breakdown of bench.py's e2e step (public cg_solve on a fresh host
CsrMatrix each step, x words back to pinned host memory)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_13536_b200 import cg, problems, kernels
from paper_2510_13536_b200.sparse import CsrMatrix

c = problems.config2()
A, b = c["A"], c["b"]
n = A.n_rows
pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
       for k, v in (("rp", A.row_ptr), ("ci", A.col_idx), ("va", A.values), ("b", b))}
conf = cg.SolverConfig(mode="dw", epsilon=1e-12, max_iterations=20000, history_stride=10**9)
T = {}
def timed(name, f):
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t0
        return r
    return g
kernels.device_matrix = timed("device_matrix", kernels.device_matrix)
cg.device_matrix = kernels.device_matrix
cg.Solver.__init__ = timed("solver_init", cg.Solver.__init__)
cg.Solver.solve = timed("solver_solve", cg.Solver.solve)
cg._b_norm = timed("b_norm", cg._b_norm)
for it in range(int(os.environ.get("E2E_STEPS", "5"))):
    T.clear()
    Ah = CsrMatrix.__new__(CsrMatrix)
    for k, v in (("n_rows", n), ("n_cols", n), ("row_ptr", pin["rp"].numpy()), ("col_idx", pin["ci"].numpy()),
                 ("values", pin["va"].numpy()), ("_device", None)):
        object.__setattr__(Ah, k, v)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = cg.cg_solve(Ah, pin["b"].numpy(), conf)
    t1 = time.perf_counter()
    xw = r.x.to_host()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"step {it}: total {1e3*(t2-t0):.1f} ms  cg_solve {1e3*(t1-t0):.1f}  to_host {1e3*(t2-t1):.1f}  "
          + "  ".join(f"{k} {1e3*v:.1f}" for k, v in T.items()) + f"  device_loop {1e3*r.device_seconds:.1f}", flush=True)
