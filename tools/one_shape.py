"""Dev: graph-timed back-to-back fp8_block_gemm launches of one shape (weights rotated over
copies larger than L2), e.g. `python tools/one_shape.py 256 24576 4096`; FP8Q_LIB=path loads
another build of the library (A/B of two builds on one box)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_18150_b200 import fp8q
from tools.kernel_bench import graph_time

shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(256, 24576, 4096)]
g = torch.Generator(device="cuda"); g.manual_seed(0)
for m, n, k in shapes:
    x = torch.randn((m, k), generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn((n, k), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    xq, xs = fp8q.quantize_act_per_token_group(x)
    wq, ws = fp8q.quantize_weight_blockwise(w)
    y = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    t = graph_time(lambda wc: fp8q.fp8_block_gemm(xq, xs, wc, ws, out=y), wq)
    print(json.dumps({"shape": [m, n, k], "us": round(t * 1e3, 2), "TFLOPs": round(2 * m * n * k / (t * 1e-3) / 1e12, 1),
                      "lib": os.environ.get("FP8Q_LIB", "default"),
                      "split": os.environ.get("FP8Q_TAIL_SPLIT", "1")}), flush=True)
