"""Summarise ncu reports / launch lists into profiles/ (tracked)."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d["Kernel Name"][:80]}
        for k in KEYS:
            if k in d:
                e[k] = f"{d[k]} {u[k]}".strip()
        stalls = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""), float(d[k])) for k in hdr
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")
            and d[k].replace(".", "", 1).isdigit()), key=lambda kv: -kv[1])[:6]
        e["top_stalls"] = stalls
        res.append(e)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (int(d["ID"]), d["Kernel Name"][:60])
            data.setdefault(key, {})[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}"
    return [{"id": k[0], "kernel": k[1], **v} for k, v in sorted(data.items())]


def launches_agg(path, command, note):
    """Launch list plus a per-kernel aggregate (count, mean/total time, share)."""
    ls = launches(path)
    agg = {}
    for e in ls:
        t = float(e["gpu__time_duration.sum"].split()[0].replace(",", ""))
        a = agg.setdefault(e["kernel"].split("(")[0], {"launches": 0, "total_ns": 0.0})
        a["launches"] += 1
        a["total_ns"] += t
    tot = sum(a["total_ns"] for a in agg.values())
    for a in agg.values():
        a["mean_ns"] = a["total_ns"] / a["launches"]
        a["share"] = a["total_ns"] / tot
    return {"command": command, "note": note, "per_kernel": agg, "launches": ls}


def k1_summary(path, cfg, source):
    """Per-mode medians of the fused kernels from a launch list of
    tools/prof_c2.py --modes fp64,dw,qdw,tw,qtw (one mode after another):
    K1 DRAM bytes per launch (bench.py roofline.traffic) and FP64-pipe
    utilisation of K1/K2/K3."""
    import statistics
    ls = launches(path)
    modes = ["fp64", "dw", "qdw", "tw", "qtw"]
    out = {"source": source, "k1_dram_bytes_per_launch": {cfg: {}}, "fp64_pipe_pct": {cfg: {}},
           "k1_us": {cfg: {}}}
    for k, kname in ((0, "cg_spmv_pq"), (1, "cg_update"), (2, "cg_xpay")):
        per = {}
        for e in ls:
            if kname not in e["kernel"]:
                continue
            m = modes[int(e["kernel"].split("<")[1].split(",")[0].split(">")[0])]
            per.setdefault(m, []).append(e)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "ns": 1e-3, "us": 1.0,
                 "msecond": 1e3, "%": 1.0}
        def val(x, key):
            v, _, u = x[key].partition(" ")
            return float(v.replace(",", "")) * scale.get(u.strip(), 1.0)
        for m, es in per.items():
            es = es[1:] if len(es) > 2 else es
            f = lambda key: statistics.median(val(x, key) for x in es if key in x)
            out["fp64_pipe_pct"][cfg].setdefault(m, {})[kname] = f(
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
            if k == 0:
                out["k1_dram_bytes_per_launch"][cfg][m] = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
                out["k1_us"][cfg][m] = f("gpu__time_duration.sum")
    return out


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    if kind == "k1-summary":
        obj = k1_summary(src, sys.argv[4], sys.argv[5])
    elif kind == "launches-agg":
        obj = launches_agg(src, sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else "")
    else:
        obj = report(src) if kind == "report" else launches(src)
    with open(dst, "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", dst, len(obj))
