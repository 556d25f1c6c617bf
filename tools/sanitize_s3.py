"""Dev: small launches of the session-3 staged quantizer kernels for compute-sanitizer
(memcheck / racecheck / synccheck): the weight kernel forced onto its TMA-staged path
(FP8Q_WEIGHT_KERNEL=bulk, set below before the library loads) on a ragged batch, and the
activation kernel's 8-row-unit path on ragged token counts / group counts."""
import os, sys
os.environ.setdefault("FP8Q_WEIGHT_KERNEL", "bulk")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16

dev = torch.device("cuda")
ws = [to_dev_bf16(synth.qwen3_weight(n, k, 20 + i)) for i, (n, k) in enumerate([(300, 208), (128, 4096), (1000, 384)])]
items = [(w, torch.empty(w.shape, dtype=torch.uint8, device=dev),
          torch.empty(((w.shape[0] + 127) // 128, (w.shape[1] + 127) // 128), dtype=torch.float32, device=dev))
         for w in ws]
fp8q.quantize_weight_blockwise_batched(items)
xs = [to_dev_bf16(synth.qwen3_activation(m, k, 30 + i)) for i, (m, k) in enumerate([(300, 384), (257, 2176), (513, 4096)])]
outs = [(torch.empty(x.shape, dtype=torch.uint8, device=dev),
         torch.empty((x.shape[1] // 128, fp8q.act_scales_ld(x.shape[0])), dtype=torch.float32, device=dev)) for x in xs]
fp8q.quantize_act_per_token_group_batched([(x, c, s) for x, (c, s) in zip(xs, outs)])
torch.cuda.synchronize()
print("sanitize s3 ok")
