#!/usr/bin/env python3
"""Dev: library context for the prefill GEMM -- cuBLASLt FP8 through torch._scaled_mm on the
Qwen3-8B prefill shapes, (a) per-tensor scales (no per-block promotion at all: the ceiling of an
FP8 GEMM on this part) and (b) DeepSeek-style blockwise scales (1x128 activations, 128x128
weights) if this torch/cuBLAS exposes them, beside fp8_block_gemm.  CUDA events, back-to-back
launches on a warm box, BF16 output.  Not a test and not a bench line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_18150_b200 import fp8q  # noqa: E402

dev = torch.device("cuda")
M = 8192
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (24576, 4096), "down": (4096, 12288)}


def timeit(fn, iters=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / iters


g = torch.Generator(device=dev)
g.manual_seed(0)
for name, (n, k) in SHAPES.items():
    w = (torch.randn((n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    x = torch.randn((M, k), generator=g, device=dev).to(torch.bfloat16)
    wq, ws = fp8q.quantize_weight_blockwise(w)
    xq, xs = fp8q.quantize_act_per_token_group(x)
    y = torch.empty((M, n), dtype=torch.bfloat16, device=dev)
    flop = 2 * M * n * k
    rec = {"shape": [M, n, k], "name": name}
    t = timeit(lambda: fp8q.fp8_block_gemm(xq, xs, wq, ws, out=y))
    rec["ours_tflops"] = round(flop / t / 1e9, 1)
    a8 = xq.view(torch.float8_e4m3fn)
    b8 = wq.view(torch.float8_e4m3fn)
    one = torch.ones((), device=dev)
    try:
        t = timeit(lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16))
        rec["cublas_pertensor_tflops"] = round(flop / t / 1e9, 1)
    except Exception as e:  # noqa: BLE001
        rec["cublas_pertensor"] = f"unavailable: {type(e).__name__}: {str(e)[:120]}"
    # blockwise: scale_a [M, K/128] (1x128), scale_b [N/128, K/128] (128x128)
    sa = torch.ones((M, k // 128), device=dev, dtype=torch.float32)
    sb = torch.ones((n // 128, k // 128), device=dev, dtype=torch.float32)
    for label, (A, B) in {"blockwise": (sa, sb), "blockwise_t": (sa.t().contiguous().t(), sb)}.items():
        try:
            t = timeit(lambda: torch._scaled_mm(a8, b8.t(), scale_a=A, scale_b=B, out_dtype=torch.bfloat16))
            rec[f"cublas_{label}_tflops"] = round(flop / t / 1e9, 1)
        except Exception as e:  # noqa: BLE001
            rec[f"cublas_{label}"] = f"unavailable: {type(e).__name__}: {str(e)[:160]}"
    print(json.dumps(rec), flush=True)
