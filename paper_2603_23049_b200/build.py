"""Build libpcr.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension machinery).

    python -m paper_2603_23049_b200.build [--verbose]

Objects go to build/ (git-ignored); the shared library lands next to this file so that it
travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "pcr")
LIB = os.path.join(PKG, "libpcr.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-Wall", "-I" + os.path.join(ROOT, "include")]
# experiment knobs only (e.g. PCR_NVCC_EXTRA="-DPCR_POLY_PAIRS=2"); the default build uses none
COMMON += os.environ.get("PCR_NVCC_EXTRA", "").split()

SOURCES = [
    "host/blake2b.cpp",
    "host/planner.cpp",
    "kernels/kv_copy.cu",
    os.environ.get("PCR_ATTN_SRC", "kernels/suffix_attn.cu"),   # experiment knob
    "runtime/nccl_dl.cpp",
    "runtime/ssd_io.cpp",
    "runtime/capi.cu",
]
HEADERS = ["host/blake2b.h", "host/planner.h", "kernels/kernels.h", "kernels/sm100_ptx.cuh", "runtime/nccl_dl.h", "runtime/ssd_io.h"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdr_time = max([_mtime(os.path.join(CSRC, h)) for h in HEADERS] +
                   [_mtime(os.path.join(ROOT, "include", "pcr.h")), _mtime(__file__)])
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace("/", "_") + ".o")
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), hdr_time):
            cmd = [NVCC, *ARCH, *COMMON, "-x", "cu" if src.endswith(".cu") else "c++", "-c", s, "-o", o]
            if src.endswith(".cu") and verbose:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        # shared cudart: the CUDA runtime the process already has (torch's) serves the library too
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", LIB, *objs, "-lpthread", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
