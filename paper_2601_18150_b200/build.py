"""Build libfp8q.so (the C-ABI of include/fp8q.h) in-tree with nvcc for sm_100a.

No fast-math: the quantizers rely on IEEE division/reciprocal/FMA with subnormals honoured
(DESIGN.md §5.1); -lineinfo so ncu's source page maps to the .cu files.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libfp8q.so")
SOURCES = ["capi.cu", "quant.cu", "gemm.cu", "gemm_skinny.cu", "producers.cu", "kv.cu", "mx.cu"]
HEADERS = ["ptx.cuh", "quant_kernels.h", "scale_tables.cuh", "packed.cuh", "group_quant.cuh", "pdl.cuh", "trace.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=true",
]


def _inputs():
    return ([os.path.join(CSRC, s) for s in SOURCES + HEADERS]
            + [os.path.join(ROOT, "include", "fp8q.h"), os.path.abspath(__file__)])


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _inputs())


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """trace=True: the dev timeline build libfp8q_trace.so (-DFP8Q_TRACE, csrc/trace.cuh), loaded
    only through FP8Q_LIB by tools/decode_timeline.py; the production library never has it."""
    lib = LIB.replace(".so", "_trace.so") if trace else LIB
    if not force and not trace and up_to_date():
        return LIB
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, *( ["-Xptxas", "-v"] if verbose else []), *(["-DFP8Q_TRACE"] if trace else []),
           "-I", os.path.join(ROOT, "include"),
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
