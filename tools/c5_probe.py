"""BASELINE config 5 on one B200: generate on device, solve DW and QTW."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_13536_b200 import cg, problems, kernels

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
t = time.time()
c = problems.config5(n=n) if n == 16_000_000 else dict(
    name="C5s", A=problems.random_irregular_spd(n), b=np.random.default_rng(3).uniform(-1, 1, n),
    epsilon=1e-12, max_iterations=20000)
torch.cuda.synchronize()
A = c["A"]
print(f"gen {time.time()-t:.1f}s n={A.n_rows} nnz={A.nnz} ({A.nnz/A.n_rows:.1f}/row) "
      f"mem {torch.cuda.max_memory_allocated()/1e9:.1f} GB", flush=True)
t = time.time()
dm = kernels.device_matrix(A)
torch.cuda.synchronize()
print(f"sell {time.time()-t:.1f}s padded={dm.padded_entries()} ({dm.padded_entries()/A.nnz:.3f}x) "
      f"col_bytes={dm.col_bytes()}", flush=True)
for mode in sys.argv[2].split(",") if len(sys.argv) > 2 else ("dw", "qtw"):
    kern = os.environ.get("C5_KERNELS") == "1"  # kernel-by-kernel launches (for ncu)
    conf = cg.SolverConfig(mode=mode, epsilon=c["epsilon"] if not kern else 1e-300,
                           max_iterations=c["max_iterations"] if not kern else 6,
                           history_stride=10**9, timing="kernels" if kern else "graph")
    r = cg.cg_solve(A, c["b"], conf)
    r = cg.cg_solve(A, c["b"], conf)
    B = 12 * A.nnz + 4 * (A.n_rows + 1) + 72 * {"fp64": 1, "dw": 2, "qdw": 2, "tw": 3, "qtw": 3}[mode] * A.n_rows
    us = r.device_seconds * 1e6 / max(1, r.iterations)
    print(f"{mode}: {r.reason} it={r.iterations} rel={r.final_recurrence_residual:.3e} "
          f"loop {r.device_seconds*1e3:.1f} ms  {us:.0f} us/it  "
          f"{B/us/1e3:.0f} GB/s ({B/us/1e3/6553:.2f} of HBM)", flush=True)
