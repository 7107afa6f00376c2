"""Build libbf.so (the C-ABI of include/bf.h) in-tree with nvcc for sm_100a.

    python -m paper_1611_00127_b200.build [--force]

Each .cu is compiled separately (in parallel) and linked into
paper_1611_00127_b200/libbf.so.  The setup translation units (split, S~, AMG setup)
are compiled with --fmad=false in addition to their explicit __dmul_rn/__dadd_rn
rounding (determinism contract).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
SO = os.path.join(PKG, "libbf.so")
# the checked variant (-DBF_CHECKED: device-side bounds / progress checks, matrix validation; see
# bf_internal.cuh) for the memory-safety runs; loaded instead of libbf.so when BF_LIB=checked
SO_CHECKED = os.path.join(PKG, "libbf_checked.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
           "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")] + ARCH
NOFMA = {"k_split.cu", "k_amg_setup.cu", "k_ilu.cu"}


def nvcc():
    for p in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if p and os.path.exists(p):
            return p
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps_mtime():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "bf.h"), __file__]
    return max(os.path.getmtime(f) for f in files)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    so = SO_CHECKED if checked else SO
    bdir = BUILD + ("_checked" if checked else "")
    if not force and os.path.exists(so) and os.path.getmtime(so) >= _deps_mtime():
        return so
    os.makedirs(bdir, exist_ok=True)
    nv = nvcc()

    def compile_one(f):
        obj = os.path.join(bdir, f[:-3] + ".o")
        flags = list(NVFLAGS) + (["-DBF_CHECKED"] if checked else [])
        if f in NOFMA:
            flags.append("--fmad=false")
        cmd = [nv, *flags, "-c", os.path.join(CSRC, f), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {f}:\n{r.stdout}\n{r.stderr}")
        return obj

    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = so + ".tmp%d" % os.getpid()
    cmd = [nv, "-shared", *ARCH, "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
