"""Why is one e2e step of bench.py slow?  Runs the e2e step 12 times and prints
per-step ms, the gc counters and the collections that ran (E2E_GC=0 disables
the cyclic collector during the loop)."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_13536_b200 import cg, problems
from paper_2510_13536_b200.sparse import CsrMatrix

c = problems.config2()
A, b = c["A"], c["b"]
n = A.n_rows
pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
       for k, v in (("rp", A.row_ptr), ("ci", A.col_idx), ("va", A.values), ("b", b))}
conf = cg.SolverConfig(mode="dw", epsilon=1e-12, max_iterations=20000, history_stride=10**9)
events = []
gc.callbacks.append(lambda phase, info: events.append((phase, info["generation"], info.get("collected", 0)))
                    if phase == "stop" else None)


def step():
    Ah = CsrMatrix.__new__(CsrMatrix)
    for k, v in (("n_rows", n), ("n_cols", n), ("row_ptr", pin["rp"].numpy()), ("col_idx", pin["ci"].numpy()),
                 ("values", pin["va"].numpy()), ("_device", None)):
        object.__setattr__(Ah, k, v)
    r = cg.cg_solve(Ah, pin["b"].numpy(), conf)
    return r, r.x.to_host()


for _ in range(2):
    step()
if os.environ.get("E2E_GC") == "0":
    gc.collect()
    gc.disable()
for i in range(12):
    events.clear()
    t = time.perf_counter()
    step()
    dt = 1e3 * (time.perf_counter() - t)
    print(f"step {i}: {dt:.1f} ms  gc_count={gc.get_count()}  collections={events}", flush=True)
