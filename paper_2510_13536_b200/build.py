"""Build libmwcg_cuda.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

    python -m paper_2510_13536_b200.build [--verbose]

Flags that matter for parity: -fmad=false (no FMA contraction: the reference
kernels are unfused and TwoProd must not fuse), IEEE div/sqrt (no fast math),
and -ffp-contract=off for the host-side sequential norm.
"""
import argparse
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libmwcg_cuda.so")
# debug build with device-side index checks on every matrix walk (-DMWCG_BOUNDS;
# csrc/common.cuh), loaded by tests/test_gpu_bounds.py through MWCG_LIB
LIB_BOUNDS = os.path.join(PKG, "libmwcg_cuda_bounds.so")
SOURCES = ["capi.cu", "sell.cu", "ops.cu", "cg.cu", "mm.cu", "problemgen.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-shared",
]


def nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def build(verbose=False, force=False, defines=(), out=None):
    lib = out or LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "mwcg_cuda.h"))
    if (not force and os.path.exists(lib)
            and os.path.getmtime(lib) >= max(os.path.getmtime(d) for d in deps)):
        return lib
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-I", CSRC, "-o", lib + ".tmp", *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


def build_all(verbose=False, force=False):
    """The product library and the bounds-checked debug build, compiled side by side."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(2) as ex:
        f1 = ex.submit(build, verbose, force)
        f2 = ex.submit(build, False, force, ("MWCG_BOUNDS",), LIB_BOUNDS)
        return f1.result(), f2.result()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--out", default=None)
    ap.add_argument("--all", action="store_true", help="also build the -DMWCG_BOUNDS debug library")
    a = ap.parse_args()
    if a.all:
        print(*build_all(verbose=a.verbose, force=a.force or a.verbose))
        sys.exit(0)
    print(build(verbose=a.verbose, force=a.force or a.verbose, defines=a.defines, out=a.out))
    sys.exit(0)
