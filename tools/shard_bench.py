"""Dev: column-parallel shard GEMM shapes (bench.py tp_shards) timed alone, cold L2 -- for
kernel-choice A/Bs (FP8Q_GEMM_KIND)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2601_18150_b200 import fp8q

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
g = torch.Generator(device="cuda"); g.manual_seed(0)
M = 8192
acts = {}
for k in (2048, 4096, 12288):
    x = torch.randn((M, k), generator=g, device="cuda").to(torch.bfloat16)
    acts[k] = fp8q.quantize_act_per_token_group(x)
shapes = [(768, 4096), (512, 4096), (3072, 4096), (512, 12288), (1536, 4096), (1024, 4096), (2048, 12288),
          (640, 2048), (256, 4096), (1280, 2048)]
for n, k in shapes:
    w = (torch.randn((n, k), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    wq, ws = fp8q.quantize_weight_blockwise(w)
    xq, xs = acts[k]
    y = torch.empty((M, n), dtype=torch.bfloat16, device="cuda")
    fn = lambda: fp8q.fp8_block_gemm(xq, xs, wq, ws, out=y)
    for _ in range(3): fn()
    ts = []
    for _ in range(15):
        flush.zero_(); flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(400_000); a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.median(ts))
    print(json.dumps({"shape": [M, n, k], "us": round(t * 1e3, 1), "TFLOPs": round(2 * M * n * k / t / 1e9, 1)}), flush=True)
