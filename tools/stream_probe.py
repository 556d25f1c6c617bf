#!/usr/bin/env python3
"""Dev driver for tools/stream_probe.cu: GB/s of streaming an FP8 [N, K] weight into shared
memory by access pattern (2-D TMA boxes of the row-major matrix vs contiguous 16 KB blocks of a
block-tiled layout), grid and ring depth; 4 copies rotate so L2 never holds the weight."""
import ctypes
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libstreamprobe.so")
SRC = os.path.join(HERE, "stream_probe.cu")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                           "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "paper_2601_18150_b200", "csrc"), SRC,
                           "-o", SO])
lib = ctypes.CDLL(SO)
lib.stream_probe.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_longlong,
                             ctypes.c_int, ctypes.c_void_p]
NAMES = {0: "2-D TMA box 128x128B (row-major)", 1: "16 KB bulk copy (block-tiled)", 2: "2-D TMA box 128x256B"}
for (n, k) in ((24576, 4096), (6144, 4096), (4096, 12288)):
    ws = [torch.randint(0, 255, (n, k), dtype=torch.uint8, device="cuda") for _ in range(4)]
    st = torch.cuda.current_stream().cuda_stream
    for grid in (148, 96):
        for mode in (0, 1, 2):
            for stages in ((4, 6) if mode == 2 else (4, 8, 12)):
                for w in ws:
                    assert lib.stream_probe(mode, stages, w.data_ptr(), n, k, grid, st) == 0
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 20
                e0.record()
                for i in range(reps):
                    lib.stream_probe(mode, stages, ws[i % 4].data_ptr(), n, k, grid, st)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / reps
                print(f"[{n},{k}] grid {grid:3d} {NAMES[mode]:36s} stages {stages:2d}: {us:7.2f} us  "
                      f"{n * k / us / 1e3:7.1f} GB/s", flush=True)
