"""Per-kernel SASS instruction mix of libmwcg_cuda.so (cuobjdump -sass).

    python tools/sass_mix.py [--lib PATH] [--out profiles/NAME.json]

Static counts (instructions in the kernel's code, not executed counts): how
many FP64-pipe instructions (DADD/DMUL/DFMA/DSETP) each fused kernel carries
against selects, integer/address work, memory and control.  Runs without a
GPU (the library is cross-compiled for sm_100a).
"""
import argparse
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODES = {0: "fp64", 1: "dw", 2: "qdw", 3: "tw", 4: "qtw"}
FP64 = ("DADD", "DMUL", "DFMA")
GROUPS = collections.OrderedDict([
    ("fp64_arith", FP64), ("fp64_cmp", ("DSETP",)), ("select", ("FSEL", "SEL")),
    ("pred_logic", ("PLOP3", "P2R", "R2P", "ISETP", "LOP3")),
    ("int_addr", ("IMAD", "IADD3", "IADD", "VIADD", "LEA", "SHF", "MOV", "CS2R", "S2R", "HFMA2", "UIADD3", "UMOV",
                  "ULEA", "USHF", "UIMAD", "ULOP3", "UISETP", "USEL", "PRMT", "R2UR", "IABS", "I2F", "F2I",
                  "MUFU", "DMNMX", "FMNMX", "IMNMX", "VIMNMX", "FADD", "FMUL", "FFMA", "UFLO", "FLO", "POPC",
                  "BREV", "SGXT", "I2FP", "F2F", "F2FP", "VOTE", "VOTEU", "REDUX", "UPOPC", "UPRMT", "UF2FP")),
    ("global_mem", ("LDG", "STG", "LDC", "LDCU", "ATOMG", "RED", "ATOM", "UBLKCP", "UBLKPF", "LD", "ST", "CCTL")),
    ("local_mem", ("LDL", "STL")), ("shared_mem", ("LDS", "STS", "LDSM", "SYNCS", "ATOMS")),
    ("shuffle", ("SHFL",)),
    ("control", ("BRA", "BSSY", "BSYNC", "EXIT", "BAR", "WARPSYNC", "NOP", "MEMBAR", "ERRBAR", "CGAERRBAR", "RET",
                 "CALL", "BREAK", "NANOSLEEP", "YIELD", "DEPBAR", "FENCE", "ACQBULK", "ELECT", "BMOV", "BPT",
                 "UCGABAR_ARV", "UCGABAR_WAIT", "ENDCOLLECTIVE", "PLOP3U", "KILL", "JMP", "BRX", "JMX", "UCLEA",
                 "UP2UR", "UR2UP", "UPLOP3", "UTMACCTL", "UTMACMDFLUSH", "LEPC", "ACQSHMINIT", "WARPGROUP")),
])


def demangle_hint(sym):
    """cg_spmv_pq<M, FUSED, CT> etc. from the mangled name (no c++filt needed)."""
    m = re.match(r"_ZN4mwcg(\d+)([A-Za-z0-9_]+)", sym)
    if not m:
        return sym, None
    name = m.group(2)[:int(m.group(1))]
    rest = m.group(2)[int(m.group(1)):]
    mode = re.match(r"ILi(\d)E", rest)
    tags = []
    if "NS_6DiaTagE" in rest:
        tags.append("dia")
    elif re.match(r"ILi\dELb[01]EsE", rest):
        tags.append("int16")
    elif re.match(r"ILi\dELb[01]EiE", rest):
        tags.append("int32")
    fused = re.match(r"ILi\dELb([01])E", rest)
    if fused and name in ("cg_spmv_pq", "cg_update", "cg_update_tma", "cg_init"):
        tags.append("fused" if fused.group(1) == "1" else "unfused")
    return name + ("[" + ",".join(tags) + "]" if tags else ""), (int(mode.group(1)) if mode else None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2510_13536_b200", "libmwcg_cuda.so"))
    ap.add_argument("--out", default="")
    ap.add_argument("--kernels", default="cg_spmv_pq,cg_update,cg_update_tma,cg_xpay,cg_xpay_tma,cg_init")
    a = ap.parse_args()
    txt = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
    want = set(a.kernels.split(","))
    rows, cur, cnt = [], None, None
    ins = re.compile(r"^\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d\s+)?([A-Z0-9_]+)")
    for line in txt.splitlines():
        f = re.search(r"Function : (\S+)", line)
        if f:
            if cur:
                rows.append((cur, cnt))
            cur, cnt = f.group(1), collections.Counter()
            continue
        m = ins.match(line)
        if m and cur:
            cnt[m.group(1)] += 1
    if cur:
        rows.append((cur, cnt))
    out = []
    for sym, c in rows:
        name, mode = demangle_hint(sym)
        base = name.split("[")[0]
        if base not in want or "unfused" in name or "int16" in name:
            continue
        total = sum(c.values())
        g = collections.OrderedDict()
        rest = collections.Counter(c)
        for gname, ops in GROUPS.items():
            g[gname] = sum(rest.pop(o, 0) for o in ops)
        g["other"] = sum(rest.values())
        row = {"kernel": name, "mode": MODES.get(mode), "instructions": total,
               "DADD": c["DADD"], "DMUL": c["DMUL"], "DFMA": c["DFMA"], "DSETP": c["DSETP"], "FSEL": c["FSEL"],
               "SEL": c["SEL"], "PLOP3": c["PLOP3"], "groups": g,
               "fp64_pipe_share": round((g["fp64_arith"] + g["fp64_cmp"]) / max(1, total), 3)}
        if rest:
            row["other_ops"] = dict(rest)
        out.append(row)
    out.sort(key=lambda r: (r["kernel"], str(r["mode"])))
    print(f"{'kernel':34s} {'mode':5s} {'instr':>6s} {'DADD':>5s} {'DMUL':>5s} {'DFMA':>5s} {'DSETP':>5s} "
          f"{'FSEL':>5s} {'SEL':>4s} {'PLOP3':>5s} {'int':>5s} {'mem':>4s} {'lmem':>4s} {'ctl':>4s} fp64%")
    for r in out:
        g = r["groups"]
        print(f"{r['kernel']:34s} {str(r['mode']):5s} {r['instructions']:6d} {r['DADD']:5d} {r['DMUL']:5d} "
              f"{r['DFMA']:5d} {r['DSETP']:5d} {r['FSEL']:5d} {r['SEL']:4d} {r['PLOP3']:5d} {g['int_addr']:5d} "
              f"{g['global_mem']:4d} {g['local_mem']:4d} {g['control']:4d} {100 * r['fp64_pipe_share']:5.1f}")
    if a.out:
        json.dump({"what": "static SASS instruction mix per fused kernel (cuobjdump -sass, sm_100a)",
                   "lib": os.path.relpath(a.lib, ROOT), "kernels": out}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    sys.exit(main())
