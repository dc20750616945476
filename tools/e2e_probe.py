"""Break down one e2e step (public API, host inputs) into phases."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_13536_b200 import cg, problems, kernels
from paper_2510_13536_b200.sparse import CsrMatrix

c = problems.config2()
A, b = c["A"], c["b"]
pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
       for k, v in (("rp", A.row_ptr), ("ci", A.col_idx), ("va", A.values), ("b", b))}

def fresh():
    Ah = CsrMatrix.__new__(CsrMatrix)
    for k, v in (("n_rows", A.n_rows), ("n_cols", A.n_cols), ("row_ptr", pin["rp"].numpy()),
                 ("col_idx", pin["ci"].numpy()), ("values", pin["va"].numpy()), ("_device", None)):
        object.__setattr__(Ah, k, v)
    return Ah

conf = cg.SolverConfig(mode="dw", epsilon=1e-12, max_iterations=20000, history_stride=10**9)
for it in range(4):
    Ah = fresh()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dm = kernels.device_matrix(Ah); torch.cuda.synchronize(); t1 = time.perf_counter()
    sv = cg.Solver(Ah, "dw"); torch.cuda.synchronize(); t2 = time.perf_counter()
    object.__setattr__(Ah, "_solvers", {("dw", "after-axpy", "tile", 1): sv})
    r = cg.cg_solve(Ah, pin["b"].numpy(), conf); t3 = time.perf_counter()
    xw = r.x.to_host(); t4 = time.perf_counter()
    print(f"step {it}: matrix {1e3*(t1-t0):.1f} ms  solver(graph) {1e3*(t2-t1):.1f} ms  "
          f"cg_solve {1e3*(t3-t2):.1f} ms (device loop {1e3*r.device_seconds:.1f}, hist {1e3*r.history_seconds:.1f})  "
          f"x->host {1e3*(t4-t3):.1f} ms", flush=True)
