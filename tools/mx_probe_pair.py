#!/usr/bin/env python3
"""Dev experiment driver for tools/mx_probe_pair.cu (CTA-pair block-scaled MMA scale sources)."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libmxprobepair.so")
SRC = os.path.join(HERE, "mx_probe_pair.cu")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                           "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "paper_2601_18150_b200", "csrc"), SRC,
                           "-o", SO])


def idesc(a_sf=0, b_sf=0):
    return (b_sf << 4) | ((256 >> 3) << 17) | (1 << 23) | ((256 >> 4) << 24) | (a_sf << 29)


def words(fn):
    """[2 ctas][8 cols][128 lanes] words with byte j = fn(cta, col, lane, j)."""
    w = np.zeros((2, 8, 128), np.uint64)
    for c in range(2):
        for col in range(8):
            for l in range(128):
                v = 0
                for j in range(4):
                    v |= (fn(c, col, l, j) & 0xFF) << (8 * j)
                w[c, col, l] = v
    return w.astype(np.uint32)


def run(sfa, sfb, a_sf=0, b_sf=0):
    lib = ctypes.CDLL(SO)
    lib.mx_probe_pair.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]
    a = torch.from_numpy(sfa.reshape(-1).view(np.int32)).cuda()
    b = torch.from_numpy(sfb.reshape(-1).view(np.int32)).cuda()
    d = torch.zeros(256 * 256, dtype=torch.float32, device="cuda")
    rc = lib.mx_probe_pair(a.data_ptr(), b.data_ptr(), idesc(a_sf, b_sf), d.data_ptr())
    assert rc == 0, rc
    d = d.cpu().numpy().reshape(256, 256)
    with np.errstate(divide="ignore"):
        return np.round(np.log2(d / 32.0)).astype(np.int64) + 127


if "--build-only" in sys.argv:
    sys.exit(0)
ONE = 127
for src in (0, 1):
    sfa = words(lambda c, col, l, j, src=src: (10 + l) if c == src else 5)
    sfb = words(lambda c, col, l, j: ONE)
    e = run(sfa, sfb)
    print(f"A from CTA{src}: rows const over n: {bool(np.all(e == e[:, :1]))}")
    print("   code per row (0..255):", e[:, 0].tolist())
for src in (0, 1):
    for g in (0, 1):
        sfa = words(lambda c, col, l, j: ONE)
        sfb = words(lambda c, col, l, j, src=src, g=g: (10 + 32 * (col % 4) + (l % 32)) if (c == src and col // 4 == g) else 5)
        e = run(sfa, sfb)
        print(f"B from CTA{src} cols {4 * g}..{4 * g + 3}: const over m: {bool(np.all(e == e[:1, :]))}")
        print("   code per n, row 0:  ", e[0, :].tolist())
        print("   code per n, row 200:", e[200, :].tolist())
