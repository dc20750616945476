"""Memory-safety evidence without compute-sanitizer (closed on this GPU pool):
libmwcg_cuda_bounds.so is the product library compiled with -DMWCG_BOUNDS --
every pattern-record, value-slot and gathered-column index of the matrix walks
is checked on the device and a violation traps.  One subprocess loads it
(MWCG_LIB) and runs every layout (slice-shared uniform / streamed, int16
deltas, int32, SELL-sigma, column blocks; ragged tiles, partial slices, empty
rows) through the operator SpMV and whole solves; it must finish cleanly with
the same bits as the product library."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BOUNDS = os.path.join(ROOT, "paper_2510_13536_b200", "libmwcg_cuda_bounds.so")

CHILD = r"""
import hashlib, json, os, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2510_13536_b200 import _lib, cg, kernels as K, problems
from paper_2510_13536_b200.sparse import CsrMatrix, laplacian_2d, random_symmetric
def copy(A, v=None):
    return CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values if v is None else v)
out = {}
def solve(tag, A, fmt, mode, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    Af = copy(A)
    dm = K.device_matrix(Af, col_format=fmt)
    for k in (env or {}):
        os.environ.pop(k)
    b = problems.spmv_fp64_host(A, np.ones(A.n_rows))
    r = cg.cg_solve(Af, b, cg.SolverConfig(mode=mode, epsilon=1e-20, max_iterations=60, history_stride=20),
                    x_star=np.ones(A.n_rows))
    x = np.random.default_rng(1).standard_normal((K.mode_words(mode), A.n_rows))
    y = K.spmv(Af, K.MultiwordVector.from_planes(x, mode)).planes.cpu().numpy()
    h = hashlib.sha256(r.x.planes.cpu().numpy().tobytes() + y.tobytes()).hexdigest()
    out[tag] = [r.iterations, r.reason, h, dm.col_bytes(), dm.col_blocks(), dm.stored_values()]
lap = laplacian_2d(45)                       # n = 2025: partial last slice and tile
v = np.array(lap.values); v[lap.row_ptr[300]:lap.row_ptr[700]] *= 1.25
mixed = copy(lap, v)                          # uniform and streamed slices
rnd = random_symmetric(3000 + 13, extra_per_row=5, seed=2)
rp, col, val = problems.random_irregular_spd(72000 + 77, seed=3, device="cpu")
c5 = CsrMatrix(72077, 72077, rp.numpy().astype(np.int64), col.numpy().astype(np.int64), val.numpy())
for mode in ("fp64", "dw", "tw", "qtw"):
    solve(f"lap-uniform-{mode}", lap, 15, mode)
    solve(f"lap-streamed-{mode}", lap, 15 | _lib.DIA_STREAM_VALUES, mode)
    solve(f"mixed-{mode}", mixed, 2, mode)
    solve(f"rnd-int16-{mode}", rnd, 1, mode)
    solve(f"rnd-int32-sigma-{mode}", rnd, 0 | _lib.SELL_SIGMA, mode)
    solve(f"rnd-int32-nosigma-{mode}", rnd, 0 | _lib.SELL_NO_SIGMA, mode)
for mode in ("dw", "qtw"):
    solve(f"c5-blocks-{mode}", c5, 0, mode, {"MWCG_COLBLOCK": "9000"})
    solve(f"c5-{mode}", c5, 15, mode)
print("RESULT " + json.dumps(out))
"""


def _run(lib):
    env = dict(os.environ)
    if lib:
        env["MWCG_LIB"] = lib
    p = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-2000:])
    assert "MWCG_BOUNDS" not in p.stdout + p.stderr
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    return json.loads(line[7:])


def test_every_layout_runs_clean_under_device_bounds_checks():
    assert os.path.exists(BOUNDS), "build the debug library: python -m paper_2510_13536_b200.build --all"
    checked = _run(BOUNDS)
    product = _run(None)
    assert checked == product
    assert checked["lap-uniform-dw"][5] == 0 and checked["lap-streamed-dw"][5] > 0
    assert 0 < checked["mixed-dw"][5] < checked["lap-streamed-dw"][5]
    assert checked["c5-blocks-dw"][4] == 9 and checked["c5-dw"][4] == 0
    assert checked["rnd-int16-dw"][3] == 2 and checked["rnd-int32-sigma-dw"][3] == 4
