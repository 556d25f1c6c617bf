#!/usr/bin/env python3
"""Dev experiment driver for tools/mx_probe.cu (block-scaled MMA scale-factor TMEM layout)."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libmxprobe.so")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "mx_probe.cu")):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                           "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "paper_2601_18150_b200", "csrc"),
                           os.path.join(HERE, "mx_probe.cu"), "-o", SO])
lib = ctypes.CDLL(SO)
lib.mx_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                         ctypes.c_uint32, ctypes.c_void_p]


def idesc(n, a_sf=0, b_sf=0, m=128):
    return (b_sf << 4) | ((n >> 3) << 17) | (1 << 23) | ((m >> 4) << 24) | (a_sf << 29)


def words(byte_fn, cols):
    """[cols][128 lanes] uint32 words, byte j of lane l of column c = byte_fn(c, l, j)."""
    w = np.zeros((cols, 128), np.uint32)
    for c in range(cols):
        for l in range(128):
            v = 0
            for j in range(4):
                v |= (byte_fn(c, l, j) & 0xFF) << (8 * j)
            w[c, l] = v
    return w


def run(sfa, sfb, n, a_sf, b_sf, a_off=0, b_off=0):
    a = torch.from_numpy(sfa.reshape(-1).astype(np.int64).astype(np.uint32).view(np.int32)).cuda()
    b = torch.from_numpy(sfb.reshape(-1).astype(np.int64).astype(np.uint32).view(np.int32)).cuda()
    d = torch.zeros(128 * 256, dtype=torch.float32, device="cuda")
    rc = lib.mx_probe(a.data_ptr(), b.data_ptr(), n, idesc(n, a_sf, b_sf), a_off, b_off, d.data_ptr())
    assert rc == 0, rc
    d = d.cpu().numpy().reshape(128, 256)[:, :n]
    with np.errstate(divide="ignore"):
        e = np.log2(d / 32.0)
    return d, e


def show(tag, e, axis_len):
    print(tag)
    ex = np.round(e).astype(np.int64)
    uniq = np.unique(ex)
    print("  distinct exponents:", uniq[:12], "... count", uniq.size)
    return ex




def main():
    if "--align" in sys.argv:
        for a_off in (2, 4, 8):
            sfa = words(lambda c, l, j: (20 + 32 * c + (l % 32)) if (l < 32 and j == 0) else 5, 8)
            sfb = words(lambda c, l, j: 127, 8)
            try:
                d, e = run(sfa, sfb, 128, 0, 0, a_off, 0)
                ex = np.round(e).astype(np.int64)[:, 0] + 127
                print("a_off", a_off, "ok codes", ex[:4].tolist(), "col", (ex[0] - 20) // 32, flush=True)
            except AssertionError as err:
                print("a_off", a_off, "error", err, flush=True)
                return
        return
    layout_probes()


def layout_probes():
    ONE = 127


    def lane_map(ex, base):
        return ex - (base - 127)


    # A: code(c, l) = 20 + 32 c + (l % 32) for lanes < 32; lanes >= 32 hold 200 + (l // 32) (quarter tag)
    for a_sf in (0, 1, 3):
        sfa = words(lambda c, l, j, a_sf=a_sf: ((20 + 32 * c + (l % 32)) if l < 32 else 250 - (l // 32)) if (j == a_sf and c < 4)
                    else 5, 8)
        sfb = words(lambda c, l, j: ONE, 8)
        d, e = run(sfa, sfb, 128, a_sf, 0)
        ex = np.round(e).astype(np.int64)[:, 0] + 127  # the SFA exponent byte each row used
        print(f"A sf_id={a_sf}: rows const across n: {bool(np.all(np.round(e) == np.round(e)[:, :1]))}")
        print("   code per row 0..127:", ex.tolist())
    # B: code(c, l) = 20 + 32 (c % 4) + (l % 32) for lanes < 32 in columns c < 4 (probe 1) / c >= 4 (probe 2)
    for b_sf in (0, 2):
        for half in (0, 1):
            sfa = words(lambda c, l, j: ONE, 8)
            sfb = words(lambda c, l, j, half=half, b_sf=b_sf: ((20 + 32 * (c % 4) + (l % 32)) if l < 32 else 250 - (l // 32))
                        if (j == b_sf and c // 4 == half) else 5, 8)
            d, e = run(sfa, sfb, 256, 0, b_sf)
            ex = np.round(e).astype(np.int64)[0, :] + 127
            print(f"B sf_id={b_sf} cols {4 * half}..{4 * half + 3}: const across m: {bool(np.all(np.round(e) == np.round(e)[:1, :]))}")
            print("   code per n 0..255:", ex.tolist())


if __name__ == "__main__" and "--build-only" not in sys.argv:
    main()
