"""Profiling driver: a few C2 iterations per mode, kernel-by-kernel (for ncu)."""
import argparse
import ctypes
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_13536_b200 import cg, problems, _lib

ap = argparse.ArgumentParser()
ap.add_argument("--modes", default="dw")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--peak", action="store_true")
ap.add_argument("--red", default="tile")
a = ap.parse_args()
if a.peak:
    L = _lib.load()
    ops, ms = ctypes.c_double(), ctypes.c_double()
    for _ in range(3):
        _lib.check(L.mwcg_fp64_peak(ctypes.byref(ops), ctypes.byref(ms), _lib.stream_handle()))
        print("fp64 peak: %.3f Tops/s (%.2f ms)" % (ops.value / 1e12, ms.value), flush=True)
c = problems.config2()
for mode in a.modes.split(","):
    r = cg.cg_solve(c["A"], c["b"], cg.SolverConfig(mode=mode, epsilon=1e-300, max_iterations=a.iters,
                                                    history_stride=10**9, timing="kernels",
                                                    reduction=a.red, partitions=256))
    print(mode, r.iterations, {k: v for k, v in r.kernel_seconds.items() if v}, flush=True)
