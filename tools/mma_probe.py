#!/usr/bin/env python3
"""Dev driver for tools/mma_probe.cu: cycles per k-block of the MMA issue sequence with resident
operands, per mode (see the .cu header), for one CTA pair and for a full-chip grid."""
import ctypes
import os
import subprocess

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libmmaprobe.so")
SRC = os.path.join(HERE, "mma_probe.cu")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                           "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "paper_2601_18150_b200", "csrc"), SRC,
                           "-o", SO])
lib = ctypes.CDLL(SO)
lib.mma_probe.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
NAMES = {0: "pair N256, 2 commits/kb (kernel)", 1: "pair N256, no commits", 2: "pair N256, 1 commit/kb",
         3: "pair N128, 2 commits/kb", 4: "pair N256, 2 commits/kb, 4-stage ring", 5: "1-CTA N256, 2 commits/kb",
         6: "1-CTA N16, 2 commits/kb", 7: "1-CTA N64, 2 commits/kb", 8: "1-CTA N128, 2 commits/kb", 9: "1-CTA N16 + 2 waits + fence/kb"}
out = torch.zeros(148, dtype=torch.int64, device="cuda")
nkb = 1024
for grid in (2, 148):
    for mode in range(10):
        out.zero_()
        for _ in range(2):
            rc = lib.mma_probe(mode, nkb, grid, out.data_ptr())
        v = out.cpu().numpy()
        v = v[v > 0]
        ideal = {3: 256, 6: 32, 7: 128, 8: 256, 9: 32}.get(mode, 512)
        print(f"grid {grid:3d} mode {mode} {NAMES[mode]:42s} rc={rc} cycles/kb med {np.median(v) / nkb:7.1f} "
              f"max {v.max() / nkb:7.1f}  (nominal {ideal})", flush=True)
