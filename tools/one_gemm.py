#!/usr/bin/env python3
"""Launch one kernel shape a few times (target for `ncu -k regex:... -s W -c N`).
usage: one_gemm.py gemm M N K | wq N K | wqlayer | aq M K | rms M K | silu M I | kv T cols | mxgemm M N K | grouped T name [skew]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2601_18150_b200 import fp8q  # noqa: E402

what = sys.argv[1]
reps = int(os.environ.get("REPS", "5"))
dev = torch.device("cuda")
g = torch.Generator(device=dev)
g.manual_seed(0)
if what == "gemm":
    m, n, k = map(int, sys.argv[2:5])
    w = (torch.randn((n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    x = torch.randn((m, k), generator=g, device=dev).to(torch.bfloat16)
    wq, ws = fp8q.quantize_weight_blockwise(w)
    xq, xs = fp8q.quantize_act_per_token_group(x)
    y = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
    for _ in range(reps):
        fp8q.fp8_block_gemm(xq, xs, wq, ws, out=y)
elif what == "wq":
    n, k = map(int, sys.argv[2:4])
    w = (torch.randn((n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    for _ in range(reps):
        fp8q.quantize_weight_blockwise(w)
elif what == "wqlayer":  # one Qwen3-8B layer's 4 weights in one batched launch (the sync step)
    items = []
    for n, k in synth.QWEN3_8B_LINEARS.values():
        w = (torch.randn((n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
        items.append((w, torch.empty((n, k), dtype=torch.uint8, device=dev),
                      torch.empty(((n + 127) // 128, (k + 127) // 128), dtype=torch.float32, device=dev)))
    for _ in range(reps):
        fp8q.quantize_weight_blockwise_batched(items)
elif what == "aq":
    m, k = map(int, sys.argv[2:4])
    x = torch.randn((m, k), generator=g, device=dev).to(torch.bfloat16)
    for _ in range(reps):
        fp8q.quantize_act_per_token_group(x)
elif what == "rms":
    m, k = map(int, sys.argv[2:4])
    x = torch.randn((m, k), generator=g, device=dev).to(torch.bfloat16)
    gam = torch.ones(k, dtype=torch.bfloat16, device=dev)
    for _ in range(reps):
        fp8q.rmsnorm_quantize_act_per_token_group(x, gam, 1e-6)
elif what == "silu":
    m, i = map(int, sys.argv[2:4])
    x = torch.randn((m, 2 * i), generator=g, device=dev).to(torch.bfloat16)
    for _ in range(reps):
        fp8q.silu_mul_quantize_act_per_token_group(x)
elif what == "mxgemm":
    m, n, k = map(int, sys.argv[2:5])
    w = (torch.randn((n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    x = torch.randn((m, k), generator=g, device=dev).to(torch.bfloat16)
    wq, ws = fp8q.mx_quantize(w)
    xq, xs = fp8q.mx_quantize(x)
    y = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
    for _ in range(reps):
        fp8q.fp8_mx_gemm(xq, xs, wq, ws, out=y)
elif what == "kv":
    t, cols = map(int, sys.argv[2:4])
    x = torch.randn((t, cols), generator=g, device=dev).to(torch.bfloat16)
    amax = torch.zeros(1, dtype=torch.int32, device=dev)
    cache = torch.empty((t, cols), dtype=torch.uint8, device=dev)
    for _ in range(reps):
        fp8q.kv_amax_update(x, amax)
        fp8q.kv_quantize_append(x, fp8q.kv_scale_from_amax(amax), cache)
elif what == "grouped":
    T = int(sys.argv[2])
    E, n, k = synth.QWEN3_30B_EXPERTS[sys.argv[3]]
    skew = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
    sizes = synth.moe_group_sizes(T, seed=0, skew=skew)
    off = torch.from_numpy(synth.offsets_from_sizes(sizes)).to(dev)
    rows = int(sizes.sum())
    w = (torch.randn((E * n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    wq, ws = fp8q.quantize_weight_blockwise(w)
    x = torch.randn((rows, k), generator=g, device=dev).to(torch.bfloat16)
    xq, xs = fp8q.quantize_act_per_token_group(x)
    for _ in range(reps):
        fp8q.fp8_block_gemm_grouped(xq, xs, wq.view(E, n, k), ws.view(E, n // 128, k // 128), off)
torch.cuda.synchronize()
