#!/usr/bin/env python
"""bench.py -- CG iterations/s and time-to-solution on B200 (BASELINE.json).

Workload (N=1): BASELINE config 2 -- 3-D 7-point Poisson on a 128^3 grid
(n = 2,097,152, nnz = 14,581,760), b = A*ones, x0 = 0, eps = 1e-12; one
step = one complete CG solve in the headline arithmetic (DW by default),
including the solver's start/end TW-accurate history records.  Config 1 is
CPU-runnable and is a parity-test case (tests/), not a bench line.

  value    : whole-job CG iterations/s with A, b resident in HBM
  e2e      : the same metric through the public API `cg_solve(A, b)` with
             HOST inputs in pinned memory: every step re-uploads the CSR
             matrix (int64 indices, as the reference's CsrMatrix holds them)
             and b, rebuilds the device SELL layout and graph, solves, and
             reads the solution words back
  roofline : K1 (SpMV + fused p.q) -- the dominant kernel
  per_arithmetic : one timed solve per arithmetic (fp64/dw/qdw/tw/qtw)
  cpu_baseline   : the C oracle (a port of the reference path) on the host
                   cores, bounded sample of CG iterations of the same config

`--impl reference` times the reference's CPU path (the oracle port, all host
threads) on the same config and metric.  Under torchrun (N>1) every rank
solves its own copy of the problem (replicas; the row-partitioned solver is
DESIGN.md's multi-GPU section) and value = total iterations / max-over-ranks
time.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODES = ("fp64", "dw", "qdw", "tw", "qtw")
WORDS = {"fp64": 1, "dw": 2, "qdw": 2, "tw": 3, "qtw": 3}
# FP64 ops per iteration F = f_nnz*nnz + f_n*n
FLOPS = {"fp64": (2, 10), "dw": (17, 90), "qdw": (11, 63), "tw": (96, 540), "qtw": (33, 237)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4"])
    ap.add_argument("--mode", default="dw", choices=MODES)
    ap.add_argument("--no-per-arith", action="store_true")
    ap.add_argument("--extra-configs", default="C1,C3,C4,C5",
                    help="comma list of other BASELINE configs to time per arithmetic and "
                         "report under 'configs' (not part of value); '' for none")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-stock", action="store_true",
                    help="--impl reference: skip timing the stock Python/numba reference")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--partitioned", action="store_true",
                    help="force the row-partitioned NCCL path (also at N=1 under torchrun)")
    ap.add_argument("--pipeline", action="store_true",
                    help="partitioned run: pipelined p exchange (one broadcast per rank slice, the "
                         "column-block passes of a slice start when it has landed; dist.py)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas instead of the row-partitioned solver")
    ap.add_argument("--c5-rows", type=int, default=16_000_000,
                    help="rows of the C5 problem of the partitioned (N>1) run")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def algorithmic_bytes(n, nnz, w):
    """one CG iteration = A once (f64 + int32 col) + int32
    row_ptr + 9 vector passes of 8w n bytes."""
    return 12 * nnz + 4 * (n + 1) + 72 * w * n


def k1_bytes(n, nnz, w):
    """K1 (SpMV + p.q): A once + row descriptors + p gathered once + q written."""
    return 12 * nnz + 4 * (n + 1) + 16 * w * n


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.k0 = 0

    def mark(self):
        """Start of the timed region: summary() uses the samples from here on
        (the sampler is started before warm-up so nvidia-smi's own start-up
        does not land in the timed region)."""
        self.k0 = len(self.lines)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in (self.lines[self.k0:] or self.lines[-1:]):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_problem(name):
    from paper_2510_13536_b200 import problems
    return problems.CONFIGS[name]()


def workload_name(cfg, mode):
    A = cfg["A"]
    desc = {"C1": "2-D 5-point Poisson 256^2", "C2": "3-D 7-point Poisson 128^3",
            "C3": "3-D 27-point stencil 160^3", "C4": "banded ill-conditioned SPD n=1e6",
            "C5": "random irregular SPD n=16e6 (GPU-built)",
            "C5s": "random irregular SPD (host-built)"}[cfg["name"]]
    return f"{cfg['name']} {desc}, CG in {mode.upper()} to {cfg['epsilon']:g} (n={A.n_rows}, nnz={A.nnz})"


def cpu_sample(cfg, mode, seconds, threads):
    """The oracle port (oracle/mwcg_oracle.c, reference algorithm) on the host
    cores: bounded number of unconditional CG iterations."""
    from oracle import oracle as orc
    orc.set_threads(threads)
    A, b = cfg["A"], cfg["b"]
    t0 = time.perf_counter()
    orc.cg_iterations(A, b, mode, 2, partitions=threads)
    t_it = max((time.perf_counter() - t0) / 2, 1e-6)
    iters = int(max(3, min(2000, seconds / t_it)))
    t0 = time.perf_counter()
    orc.cg_iterations(A, b, mode, iters, partitions=threads)
    dt = time.perf_counter() - t0
    return iters, dt


# ---------------------------------------------------------------------------
def base_config(cfg, mode):
    """The `config` dict of BOTH arms (same workload, same keys)."""
    A = cfg["A"]
    w = WORDS[mode]
    return {"workload": workload_name(cfg, mode), "mode": mode, "n": int(A.n_rows), "nnz": int(A.nnz),
            "epsilon": cfg["epsilon"],
            "l2": f"inputs larger than L2 (A {12 * A.nnz / 1e6:.0f} MB + vectors "
                  f"{4 * 8 * w * A.n_rows / 1e6:.0f} MB > 126 MB)"}


def stock_reference(budget_s=150.0):
    """The UNMODIFIED reference package (Python + numba, baseline/_ref) through
    its public cg_solve on ONE host core (it is single-threaded): C1 full
    solves (TW: a 30-iteration sample, its full solve takes ~100 s) and a
    10-iteration C2 DW sample.  Each run is a subprocess
    (oracle/stock_reference.py) pinned to one core; JIT warm-up untimed."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import stock_reference as sr
    if not sr.available():
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref "
                               "/root/reference/pkg)"}
    runs = [("C1", m, 0) for m in ("fp64", "dw", "qdw", "qtw")] + [("C1", "tw", 30), ("C2", "dw", 10)]
    out, t0 = [], time.perf_counter()
    for cfg, mode, iters in runs:
        left = budget_s - (time.perf_counter() - t0)
        if left < 10:
            out.append({"config": cfg, "mode": mode, "skipped": "time budget"})
            continue
        cmd = [sys.executable, os.path.join(ROOT, "oracle", "stock_reference.py"), "--config", cfg,
               "--mode", mode] + (["--iters", str(iters)] if iters else [])
        try:
            pr = subprocess.run(cmd, capture_output=True, text=True, timeout=left)
            out.append(json.loads(pr.stdout.strip().splitlines()[-1]))
        except Exception as exc:  # pragma: no cover - reported, never fatal
            out.append({"config": cfg, "mode": mode, "error": f"{type(exc).__name__}: {exc}"[:200]})
    return {"runs": out, "cores": 1,
            "note": "stock mwcg 0.1.0 (reference package, Python + numba, single-threaded by design)"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc
    cfg = load_problem(a.config)
    threads = orc.max_threads()
    orc.set_threads(threads)
    per_step = max(1.0, a.cpu_seconds / max(1, a.steps))
    for _ in range(max(0, min(a.warmup, 1))):
        cpu_sample(cfg, a.mode, 0.5, threads)
    tot_it, tot_t = 0, 0.0
    for _ in range(a.steps):
        it, dt = cpu_sample(cfg, a.mode, per_step, threads)
        tot_it += it
        tot_t += dt
    v = tot_it / tot_t
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import stock_reference as sr
    line = {
        "impl": "reference", "metric": "CG iterations/s", "value": v, "unit": "iter/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * tot_t / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": base_config(cfg, a.mode),
        "cpu_baseline": {"value": v, "unit": "iter/s", "cores": threads, "kind": "port",
                         "cpu_model": sr.cpu_model(),
                         "sample": f"{tot_it} unconditional CG iterations of {cfg['name']} in "
                                   f"{a.mode} (oracle/mwcg_oracle.c: the reference algorithm in C, "
                                   f"OpenMP over rows, partitions={threads} dot shape)"},
        "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not a.no_stock:
        line["stock_reference"] = stock_reference()
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# per config: modes solved to the config's epsilon (full), the rest timed on
# a bounded sample of unconditional iterations (their full solves take
# minutes: C4 TW ~1.4e5 iterations)
EXTRA_PLAN = {"C1": {"full": MODES}, "C3": {"full": MODES},
              "C4": {"full": ("fp64", "dw", "qtw"), "sample": 3000},
              "C5": {"full": ("dw", "qtw")}}


def extra_config(name, hbm, fp64_peak, torch):
    """One BASELINE config on one GPU: per arithmetic µs per iteration,
    iterations to solution, roofline fractions (9-pass bytes / counted FP64
    ops).  C5 here is the N=1 point of the N>1 strong-scaling run."""
    from paper_2510_13536_b200 import _lib, kernels
    from paper_2510_13536_b200.cg import Solver, _b_norm
    t0 = time.perf_counter()
    ec = load_problem(name)
    EA, Eb = ec["A"], ec["b"]
    en, ennz = EA.n_rows, EA.nnz
    ebd = torch.from_numpy(Eb).cuda()
    ebn = _b_norm(Eb)
    gen_s = time.perf_counter() - t0
    plan = EXTRA_PLAN.get(name, {"full": MODES})
    modes = plan["full"] + tuple(m for m in MODES if m not in plan["full"] and plan.get("sample")
                                 and name != "C5")
    stride = 10 ** 9
    rows = {}
    for m in modes:
        sv = Solver(EA, m)
        full = m in plan["full"]
        eps, mx = (ec["epsilon"], ec["max_iterations"]) if full else (1e-300, plan["sample"])
        sv.solve(ebd, ebn, None, None, 1e-300, 5, stride)   # warm-up: 5 iterations
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r, _ = sv.solve(ebd, ebn, None, None, eps, mx, stride)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        it = max(1, int(r.iterations))
        wm = WORDS[m]
        # the iteration loop alone (CUDA events around the graph launches): `t` also
        # holds the start/end history records (a TW-accurate residual each: two TW
        # SpMVs and dots), which weigh on a short solve (C5: 37 iterations)
        tl = r.loop_ms * 1e-3 if r.loop_ms > 0 else t
        bw = algorithmic_bytes(en, ennz, wm) * it / tl / 1e9
        fn, fx = FLOPS[m]
        fl = (fn * ennz + fx * en) * it / tl
        rows[m] = {"iterations": int(r.iterations), "reason": _lib.STATUS[r.status],
                   "final_rel": r.final_rel, "solve": "full" if full else f"{mx} unconditional iterations",
                   "time_s": t, "loop_s": tl, "us_per_iter": 1e6 * tl / it,
                   "us_per_iter_with_history_records": 1e6 * t / it, "hbm_frac": bw / hbm,
                   "fp64_frac": fl / fp64_peak, "roofline_frac": max(bw / hbm, fl / fp64_peak),
                   "bound": "fp64" if fl / fp64_peak > bw / hbm else "hbm",
                   "kernels": sv.describe()}
        del sv
        torch.cuda.empty_cache()
    out = {"workload": workload_name(ec, "all"), "n": en, "nnz": ennz, "generate_s": gen_s,
           "col_bytes": kernels.device_matrix(EA).col_bytes(), "per_arithmetic": rows}
    if name == "C5":
        out["note"] = ("N=1 point of the strong-scaling run (bench.py --gpus N>1: same matrix, "
                       "same full DW solve, row-partitioned)")
    return out


def run_ours(a):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or a.partitioned:
        if "RANK" not in os.environ:  # plain `python bench.py --partitioned`: one rank
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(_free_port()))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_13536_b200 import cg, kernels, _lib
    from paper_2510_13536_b200.cg import Solver, _b_norm

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    if (world > 1 and not a.replicas) or a.partitioned:
        return run_partitioned(a, world, rank, local, dist, torch)
    cfg = load_problem(a.config)
    A, b, xs = cfg["A"], cfg["b"], cfg["x_star"]
    n, nnz, mode = A.n_rows, A.nnz, a.mode
    w = WORDS[mode]
    eps, max_it = cfg["epsilon"], cfg["max_iterations"]
    stride = 10 ** 9  # start/end records only (the reference records them too)
    hbm, hbm_src = peaks()
    L = _lib.load()
    import ctypes
    fp64_ops, fp64_ms = ctypes.c_double(), ctypes.c_double()
    _lib.check(L.mwcg_fp64_peak(ctypes.byref(fp64_ops), ctypes.byref(fp64_ms), _lib.stream_handle()))
    fp64_peak = fp64_ops.value  # FP64 ops/s (FMA = 1), measured live

    b_dev = torch.from_numpy(b).cuda()
    bn = _b_norm(b)

    def device_solve(solver, profile=False):
        return solver.solve(b_dev, bn, None, None, eps, max_it, stride, profile)

    # ---- value: device-resident inputs ------------------------------------
    solver = Solver(A, mode)
    dmat = kernels.device_matrix(A)
    cb = dmat.col_bytes()
    layout = {"format": {0: "slice-shared offsets (SELL-32 slices, pattern table)", 2: "SELL-32 int16 deltas",
                         4: "SELL-32 int32"}[cb],
              "col_bytes_per_entry": cb, "padded_entries": dmat.padded_entries(), "nnz": nnz,
              # value entries K1 actually streams: value-uniform slices keep their
              # values in the (L1-resident) pattern records (0 for C1/C2)
              "stored_values": dmat.stored_values(), "col_blocks": dmat.col_blocks()}
    with ClockSampler(local) as clk:
        for _ in range(max(3, a.warmup)):
            device_solve(solver)
        iters, launches = 0, 0
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        clk.mark()
        ev0.record()
        for _ in range(a.steps):
            res, _ = device_solve(solver)
            iters += int(res.iterations)
            launches += int(res.launches)
        ev1.record()
        barrier()
    dt = ev0.elapsed_time(ev1) * 1e-3
    dt_max = max_over_ranks(dt)
    total_iters = sum_over_ranks(iters)
    value = total_iters / dt_max
    ms_per_step = 1e3 * dt_max / a.steps
    reason = _lib.STATUS[res.status]
    iters_per_solve = int(res.iterations)

    # ---- roofline of K1 (profiled solve: per-stage CUDA events) ------------
    pres, _ = device_solve(solver, profile=True)
    it_p = max(1, int(pres.iterations))
    k1_s = pres.stage_ms[0] * 1e-3 / it_p
    k2_s = pres.stage_ms[1] * 1e-3 / it_p
    k3_s = pres.stage_ms[2] * 1e-3 / it_p
    # K1's launch duration: back-to-back launches between CUDA events on the
    # solver's stream (the per-stage events above also carry launch gaps)
    from paper_2510_13536_b200.cg import _time_k1
    k1_launch_s = _time_k1(solver, b_dev, bn, reps=20) * 1e-6
    k1_achieved = k1_bytes(n, nnz, w) / k1_launch_s / 1e9
    traffic, prof = None, {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            prof = json.load(f)
        traffic = prof.get("k1_dram_bytes_per_launch", {}).get(a.config, {}).get(mode)
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": k1_achieved, "peak": hbm, "unit": "GB/s",
                "frac": k1_achieved / hbm, "traffic": traffic,
                "traffic_source": prof.get("source"),
                "traffic_note": "achieved/frac use the ALGORITHMIC (canonical CSR) bytes; traffic is the DRAM "
                                "bytes ncu measured per launch -- below the algorithmic bytes when the layout "
                                "streams no column indices / no values for value-uniform slices",
                "kernel": "cg_spmv_pq (SpMV + fused p.q + alpha)",
                "algorithmic_bytes_per_launch": k1_bytes(n, nnz, w),
                "launch_us": k1_launch_s * 1e6, "peak_source": hbm_src,
                "launch_timing": "20 back-to-back K1 launches between CUDA events (solver stream)",
                "stage_us": {"K1_spmv_pq": k1_s * 1e6, "K2_update_r_rr": k2_s * 1e6,
                             "K3_xpay_x": k3_s * 1e6},
                "vector_passes": {"canonical": 9, "implemented": 10,
                                  "schedule": "K1: p gathered, q written; K2: r, q read, r written; "
                                              "K3: r, p, x read, p, x written"},
                "matrix_layout": layout,
                "iteration": {"us": 1e6 * dt / max(1, iters),
                              "algorithmic_bytes": algorithmic_bytes(n, nnz, w),
                              "achieved_gbs": algorithmic_bytes(n, nnz, w) * iters / dt / 1e9,
                              "frac": algorithmic_bytes(n, nnz, w) * iters / dt / 1e9 / hbm}}

    # ---- e2e through the public API with host inputs -------------------------
    # (measured right after the headline, before the per-arithmetic and the other
    # configs' solves: their deferred frees -- C5 alone releases tens of GB -- used to
    # land inside one timed e2e step, 50-140 ms against 45)
    e2e = None
    if not a.no_e2e:
        import gc
        import torch as _t
        gc.collect()
        torch.cuda.synchronize()
        pin = {k: _t.from_numpy(np.ascontiguousarray(v)).pin_memory()
               for k, v in (("rp", A.row_ptr), ("ci", A.col_idx), ("va", A.values), ("b", b))}
        from paper_2510_13536_b200.sparse import CsrMatrix
        h2d = sum(t.numel() * t.element_size() for t in pin.values())
        d2h = w * n * 8
        conf = cg.SolverConfig(mode=mode, epsilon=eps, max_iterations=max_it, history_stride=stride)

        def e2e_step():
            Ah = CsrMatrix.__new__(CsrMatrix)  # pinned arrays, validated once below
            object.__setattr__(Ah, "n_rows", n)
            object.__setattr__(Ah, "n_cols", n)
            object.__setattr__(Ah, "row_ptr", pin["rp"].numpy())
            object.__setattr__(Ah, "col_idx", pin["ci"].numpy())
            object.__setattr__(Ah, "values", pin["va"].numpy())
            object.__setattr__(Ah, "_device", None)
            r = cg.cg_solve(Ah, pin["b"].numpy(), conf)
            xw = r.x.to_host()  # solution words back to the host (pinned)
            return r, xw

        CsrMatrix(n, n, A.row_ptr, A.col_idx, A.values)  # validation (not timed)
        for _ in range(max(1, min(a.warmup, 2))):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        e_it = 0
        step_ms = []
        for _ in range(a.steps):
            ts = time.perf_counter()
            r, _ = e2e_step()
            e_it += int(r.iterations)
            step_ms.append(1e3 * (time.perf_counter() - ts))
        barrier()
        e_dt = max_over_ranks(time.perf_counter() - t0)
        print("e2e step ms: " + " ".join(f"{v:.1f}" for v in step_ms), file=sys.stderr, flush=True)
        e2e = {"value": sum_over_ranks(e_it) / e_dt, "unit": "iter/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * e_dt / a.steps,
               "ms_per_step_median": statistics.median(step_ms),
               "path": "cg_solve(CsrMatrix(host, pinned), b host) -> x words to host"}

    # ---- per-arithmetic solves (device-resident) -----------------------------
    per = {}
    if not a.no_per_arith:
        for m in MODES:
            sv = solver if m == mode else Solver(A, m)
            device_solve(sv)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r, _ = device_solve(sv)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e-3
            it = max(1, int(r.iterations))
            wm = WORDS[m]
            B = algorithmic_bytes(n, nnz, wm)
            fn, fx = FLOPS[m]
            F = fn * nnz + fx * n
            bw = B * it / t / 1e9
            fl = F * it / t
            hfrac, ffrac = bw / hbm, fl / fp64_peak
            per[m] = {"iterations": int(r.iterations), "reason": _lib.STATUS[r.status],
                      "final_rel": r.final_rel, "time_to_solution_s": t,
                      "iter_per_s": it / t, "us_per_iter": 1e6 * t / it,
                      "hbm_gbs": bw, "hbm_frac": hfrac, "fp64_tops": fl / 1e12,
                      "fp64_frac": ffrac, "roofline_frac": max(hfrac, ffrac),
                      "bound": "fp64" if ffrac > hfrac else "hbm"}
            # FP64-pipe utilisation of the three kernels from the committed ncu
            # launch list (profiles/ncu_summary.json): the instruction-level
            # view of the FP64 roofline (counted ops exclude the compares and
            # selects the exact TW merge needs)
            pipe = prof.get("fp64_pipe_pct", {}).get(a.config, {}).get(m)
            if pipe:
                per[m]["ncu_fp64_pipe_pct"] = pipe
            if sv is not solver:
                del sv
            torch.cuda.empty_cache()

    # ---- other BASELINE configs (reported, not part of value) ---------------
    extra = {}
    for name in [c for c in a.extra_configs.split(",") if c]:
        try:
            extra[name] = extra_config(name, hbm, fp64_peak, torch)
        except Exception as exc:  # pragma: no cover - reported, never fatal
            extra[name] = {"error": f"{type(exc).__name__}: {exc}"}
        torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0, N=1 only) -------------------------------------
    cpu = None
    if world == 1 and rank == 0:
        try:
            from oracle import oracle as orc
            thr = orc.max_threads()
            it, cdt = cpu_sample(cfg, mode, a.cpu_seconds, thr)
            cpu = {"value": it / cdt, "unit": "iter/s", "cores": thr, "kind": "port",
                   "sample": f"{it} unconditional CG iterations of {cfg['name']} in {mode} "
                             f"(oracle/mwcg_oracle.c, partitions={thr}), {cdt:.1f} s"}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "iter/s", "cores": 0, "kind": "port",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": "CG iterations/s", "value": value, "unit": "iter/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": base_config(cfg, mode),
            "solve": {"iterations_per_solve": iters_per_solve, "reason": reason,
                      "time_to_solution_s": ms_per_step * 1e-3,
                      "parallelism": "replicas" if world > 1 else "single",
                      "reduction": "canonical tile tree (bitwise-reproducible)",
                      "kernels": solver.describe()},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "fp64_peak_tops_measured": fp64_peak / 1e12,
            "per_arithmetic": per,
            "configs": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_partitioned(a, world, rank, local, dist, torch):
    """Row-partitioned CG over NCCL, STRONG scaling on BASELINE
    config 5: random irregular SPD, n = 16M, ~1.3e9 nnz, built on every
    rank's GPU from the same seed (identical matrix), each rank keeping its
    tile-aligned row block (sliced on the device).  One step = one full CG
    solve to 1e-12 (a few dozen iterations: 1.01 diagonal dominance keeps C5
    well conditioned); value = global CG iterations / s (max over ranks).
    p is all-gathered each iteration (C5's random columns leave no interior
    tiles to overlap), the tile partials gathered in one
    all-gather and reduced in the canonical order on every rank."""
    from paper_2510_13536_b200 import problems
    from paper_2510_13536_b200.cg import _b_norm
    from paper_2510_13536_b200.dist import (RankSolver, TorchDistExchange, dist_cg_solve,
                                            local_rows, partition)
    mode = a.mode
    n = a.c5_rows
    t0 = time.perf_counter()
    Afull = problems.random_irregular_spd(n, seed=3)
    nnz = Afull.nnz
    b = np.random.default_rng(3).uniform(-1.0, 1.0, n)
    bn = _b_norm(b)
    part = partition(n, world)
    lo, hi = part.rows(rank)
    Aloc = local_rows(Afull, lo, hi)
    Aloc.row_ptr, Aloc.col_idx, Aloc.values = (Aloc.row_ptr.clone(), Aloc.col_idx.clone(),
                                               Aloc.values.clone())
    del Afull
    torch.cuda.empty_cache()
    rs = RankSolver(Aloc, part, rank, mode, pipeline=a.pipeline)
    del Aloc
    torch.cuda.empty_cache()
    setup_s = time.perf_counter() - t0
    b_loc = torch.from_numpy(np.ascontiguousarray(b[lo:hi])).cuda() if hi > lo else \
        torch.zeros(1, dtype=torch.float64, device="cuda")
    ex = TorchDistExchange()
    eps, max_it = 1e-12, 20000
    seg = [8]

    def solve():
        rs.start(b_loc, bn, None, eps, max_it)
        # eager stages (each iteration's GPU work, ~ms, dwarfs the host's
        # launch cost); after the first solve the segment length is the known
        # iteration count, so a step runs exactly the solve's iterations
        return dist_cg_solve([rs], ex, bn, eps, max_it, check_every=seg[0], graph=False)

    first = solve()
    seg[0] = max(1, first.iterations)
    with ClockSampler(local) as clk:
        for _ in range(max(3, a.warmup)):
            solve()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk.mark()
        e0.record()
        its = launches = 0
        for _ in range(a.steps):
            r = solve()
            its += r.iterations
            launches += r.launches
        e1.record()
        torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) * 1e-3
    # e2e: the same steps with this rank's b copied in from pinned host
    # memory and its solution words copied back every step
    b_host = torch.from_numpy(np.ascontiguousarray(b[lo:hi])).pin_memory()
    x_host = torch.empty(tuple(rs.solution().shape), dtype=torch.float64).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    its_e = 0
    for _ in range(a.steps):
        if hi > lo:
            b_loc.copy_(b_host, non_blocking=True)
        its_e += solve().iterations
        x_host.copy_(rs.solution(), non_blocking=True)
    e3.record()
    torch.cuda.synchronize()
    dte = e2.elapsed_time(e3) * 1e-3
    t = torch.tensor([dt, dte], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt, dte = (float(v) for v in t.tolist())
    w = WORDS[mode]
    hbm, hbm_src = peaks()
    value = its / dt
    per_gpu_bytes = algorithmic_bytes(n, nnz, w) / world
    if rank == 0:
        line = {
            "metric": "CG iterations/s", "value": value, "unit": "iter/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5 random irregular SPD n={n} (nnz={nnz}), CG in {mode.upper()}, "
                                   f"row-partitioned over {world} GPU(s)",
                       "n": n, "nnz": nnz, "mode": mode, "epsilon": eps,
                       "step": "one full CG solve to 1e-12",
                       "iterations_per_solve": r.iterations, "reason": r.reason,
                       "final_rel": r.final_recurrence_residual,
                       "time_to_solution_s": dt / a.steps,
                       "parallelism": f"row partition over {world} GPUs: p exchange = NCCL "
                                      f"{'neighbour halo (send/recv)' if ex.mode == 'halo' else 'all-gather'}"
                                      " + one tile-partial all-gather per dot, canonical MW reduction",
                       "p_exchange": ex.mode, "interior_tiles": list(rs.interior),
                       "setup_s": setup_s,
                       "scaling_base": "the N=1 default run reports the same C5 solve under configs.C5"},
            "roofline": {"bound": "hbm", "unit": "GB/s", "peak": hbm, "peak_source": hbm_src,
                         "achieved": per_gpu_bytes * its / dt / 1e9,
                         "frac": per_gpu_bytes * its / dt / 1e9 / hbm, "traffic": None,
                         "kernel": "whole iteration per GPU (canonical 9-pass bytes / N)"},
            "e2e": {"value": its_e / dte, "unit": "iter/s",
                    "h2d_bytes_per_step": 8 * (hi - lo),
                    "d2h_bytes_per_step": 8 * int(x_host.numel()),
                    "note": "per rank: b slice in, solution words out, every step"},
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
