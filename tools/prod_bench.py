"""Dev timing of the NEXT-2 producer-fused quantizers at the bench shapes (CUDA events, L2
flushed by a write + read of 256 MB before each launch, median of 20)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2601_18150_b200 import fp8q

HBM = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6540.0
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t_ms(fn, iters=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_(); flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(400_000)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


g = torch.Generator(device="cuda"); g.manual_seed(0)
M = 8192
x = torch.randn((M, 4096), generator=g, device="cuda").to(torch.bfloat16)
gam = torch.ones(4096, dtype=torch.bfloat16, device="cuda")
q = torch.empty((M, 4096), dtype=torch.uint8, device="cuda")
s = torch.empty((32, M), dtype=torch.float32, device="cuda")
t = t_ms(lambda: fp8q.rmsnorm_quantize_act_per_token_group(x, gam, 1e-6, q, s))
by = M * 4096 * (3 + 4 / 128)
print(json.dumps({"kernel": "rmsnorm_quantize", "shape": [M, 4096], "us": round(t * 1e3, 1),
                  "GBps": round(by / t / 1e6, 1), "frac_hbm": round(by / t / 1e6 / HBM, 4)}))
gu = torch.randn((M, 2 * 12288), generator=g, device="cuda").to(torch.bfloat16)
q2 = torch.empty((M, 12288), dtype=torch.uint8, device="cuda")
s2 = torch.empty((96, M), dtype=torch.float32, device="cuda")
t = t_ms(lambda: fp8q.silu_mul_quantize_act_per_token_group(gu, q2, s2))
by = M * 12288 * (5 + 4 / 128)
print(json.dumps({"kernel": "silu_mul_quantize", "shape": [M, 12288], "us": round(t * 1e3, 1),
                  "GBps": round(by / t / 1e6, 1), "frac_hbm": round(by / t / 1e6 / HBM, 4)}))
