import sys, os, ctypes, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2510_13536_b200 import _lib, kernels as kn
L = _lib.load()
n = 2096704
for mode in ("fp64", "dw", "tw"):
    x = kn.MultiwordVector.from_fp64(np.random.default_rng(0).standard_normal(n), mode)
    work = torch.zeros(int(L.mwcg_dot_work_bytes(n, 0)) // 8 + 1, dtype=torch.float64, device="cuda")
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    st = _lib.stream_handle()
    f = lambda: L.mwcg_dot(_lib.MODE_ID[mode], n, _lib.ptr(x.planes), n, _lib.ptr(x.planes), n, 0, _lib.ptr(out), _lib.ptr(work), st)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(50): f()
    e1.record(); e1.synchronize()
    print(mode, "kernel-only us/call %.1f" % (e0.elapsed_time(e1) / 50 * 1e3))
