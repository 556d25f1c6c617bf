"""Dev probe: fused decode activation quantization (fp8_linear_dynamic, XQ) vs the two-step path
and the oracle on a few shapes; times one launch of each."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16, rel_frobenius

for (m, n, k) in [(1, 1024, 384), (1, 6144, 4096), (16, 1024, 384), (1, 24576, 4096)]:
    wb = synth.qwen3_weight(n, k, 1)
    wq, ws = fp8q.quantize_weight_blockwise(to_dev_bf16(wb))
    xb = synth.qwen3_activation(m, k, 2)
    x = to_dev_bf16(xb)
    y = fp8q.fp8_linear_dynamic(x, wq, ws, out_dtype=torch.float32)
    xq, xs = fp8q.quantize_act_per_token_group(x)
    r = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=torch.float32)
    torch.cuda.synchronize()
    oa, osa = oracle.quantize_act_per_token_group(xb)
    ow, osw = oracle.quantize_weight_blockwise(wb)
    ref = oracle.gemm_rows(oa, osa, ow, osw)
    def t(fn):
        for _ in range(3): fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(400000); a.record(); fn(); b.record(); b.synchronize(); return a.elapsed_time(b) * 1e3
    print(json.dumps({"shape": [m, n, k], "xq_vs_oracle": rel_frobenius(y.cpu().numpy(), ref),
                      "twostep_vs_oracle": rel_frobenius(r.cpu().numpy(), ref),
                      "xq_us": round(t(lambda: fp8q.fp8_linear_dynamic(x, wq, ws)), 1),
                      "gemm_us": round(t(lambda: fp8q.fp8_block_gemm(xq, xs, wq, ws)), 1)}), flush=True)
