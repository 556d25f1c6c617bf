#!/usr/bin/env python3
"""Dev: what the 2:1 read:write streaming pattern of the quantizers can reach on this B200.
Times (CUDA events, L2 flushed by a 512 MB write between iterations) torch's own streaming
kernels -- bf16 copy (1:1) and the bf16 -> float8_e4m3fn cast (2:1, the quantizers' byte
pattern without the amax/scale work) -- beside our activation and weight quantizers at the
same shapes.  Prints GB/s of algorithmic bytes and the fraction of MEASURED_PEAKS hbm_gbs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_18150_b200 import fp8q  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # noqa: BLE001
    PEAK = 6540.0
dev = torch.device("cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # keep the GPU busy while the host enqueues (tensor-map encode, output allocation), so
        # the interval measures the kernel, not the binding's host overhead
        torch.cuda._sleep(400_000)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def line(name, us, nbytes):
    gbs = nbytes / us / 1e3
    print(f"{name:40s} {us:8.2f} us {gbs:8.1f} GB/s {gbs / PEAK:6.1%}")


for (m, k) in [(8192, 4096), (8192, 12288), (24576, 4096), (32768, 12288)]:
    x = torch.randn((m, k), device=dev).to(torch.bfloat16)
    e = m * k
    y = torch.empty_like(x)
    line(f"torch copy bf16 [{m},{k}]", timeit(lambda: y.copy_(x)), 4 * e)
    z = torch.empty((m, k), dtype=torch.float8_e4m3fn, device=dev)
    line(f"torch cast bf16->e4m3 [{m},{k}]", timeit(lambda: z.copy_(x)), 3 * e)
    line(f"act quant [{m},{k}]", timeit(lambda: fp8q.quantize_act_per_token_group(x)), e * 3.03125)
    line(f"weight quant [{m},{k}]", timeit(lambda: fp8q.quantize_weight_blockwise(x)), e * (3 + 4 / 16384))
    del x, y, z
