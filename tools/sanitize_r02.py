"""Dev: small launches of every round-2 kernel path for compute-sanitizer (memcheck /
racecheck / synccheck): batched act quant, exact producers, prefill pair + one-CTA GEMM,
grouped GEMM, decode kernel (stream-K, ordered stream-K, cluster split-K)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16

dev = torch.device("cuda")
xs = [to_dev_bf16(synth.qwen3_activation(m, k, 1)) for m, k in [(37, 384), (5, 2176), (64, 4096)]]
outs = [(torch.empty(x.shape, dtype=torch.uint8, device=dev),
         torch.empty((x.shape[1] // 128, fp8q.act_scales_ld(x.shape[0])), dtype=torch.float32, device=dev)) for x in xs]
fp8q.quantize_act_per_token_group_batched([(x, c, s) for x, (c, s) in zip(xs, outs)])
g = to_dev_bf16(synth.f32_to_bf16_bits(np.ones(1024, np.float32)))
fp8q.rmsnorm_quantize_act_per_token_group(to_dev_bf16(synth.qwen3_activation(33, 1024, 2)), g, 1e-6)
fp8q.silu_mul_quantize_act_per_token_group(to_dev_bf16(synth.qwen3_activation(17, 2 * 768, 3)))
w = to_dev_bf16(synth.qwen3_weight(1024, 1024, 4))
wq, wsc = fp8q.quantize_weight_blockwise(w)
for m in (512, 300):  # pair kernel, one-CTA kernel
    a, sa = fp8q.quantize_act_per_token_group(to_dev_bf16(synth.qwen3_activation(m, 1024, 5)))
    fp8q.fp8_block_gemm(a, sa, wq, wsc)
w2 = to_dev_bf16(synth.qwen3_weight(4096, 1024, 7))
wq2, ws2 = fp8q.quantize_weight_blockwise(w2)
w3 = to_dev_bf16(synth.qwen3_weight(128 * 150, 1024, 10))  # 150 tiles: ordered stream-K
wq3, ws3 = fp8q.quantize_weight_blockwise(w3)
for m in (1, 5, 8, 40):  # decode: stream-K / cluster split-K / ordered stream-K
    x = to_dev_bf16(synth.qwen3_activation(m, 1024, 6))
    fp8q.fp8_linear_dynamic(x, wq, wsc)
    fp8q.fp8_linear_dynamic(x, wq2, ws2)
    fp8q.fp8_linear_dynamic(x, wq3, ws3)
E, n, k = 4, 256, 512
we = to_dev_bf16(synth.qwen3_weight(E * n, k, 8))
weq, wes = fp8q.quantize_weight_blockwise(we)
sizes = np.array([70, 0, 130, 33])
off = torch.from_numpy(synth.offsets_from_sizes(sizes)).to(dev)
a, sa = fp8q.quantize_act_per_token_group(to_dev_bf16(synth.qwen3_activation(int(sizes.sum()), k, 9)))
fp8q.fp8_block_gemm_grouped(a, sa, weq.view(E, n, k), wes.view(E, n // 128, k // 128), off)
torch.cuda.synchronize()
print("sanitize ok")
