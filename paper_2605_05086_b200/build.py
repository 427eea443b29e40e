"""Build libchap.so (the CUDA path) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libchap.so")
SOURCES = ["chap.cu"]
HEADERS = ["common.cuh", "eval.cuh", "tabu.cuh", "host.h", "portfolio.cuh", "lp.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-shared", "--expt-relaxed-constexpr"]


def _deps():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "chap.h")]
    return max(os.path.getmtime(f) for f in files)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= _deps():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = os.environ.get("CHAP_NVCC_FLAGS", "").split()   # experiments (e.g. -DCHAP_GEN_MINB=4)
    cmd = [nvcc] + NVCC_FLAGS + extra + ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-o", SO + ".tmp"]
    cmd += [os.path.join(CSRC, s) for s in SOURCES]
    cmd += ["-ldl"]   # NCCL is dlopen'ed at run time (csrc/portfolio.cuh)
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
