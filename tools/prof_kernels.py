"""Dev: one launch of each hot kernel at the bench shapes, for `ncu --set full` captures
(-k regex filters the kernel): the layer's batched activation quantization, the four prefill
GEMMs, the layer requant, the MoE fc2 grouped GEMM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2601_18150_b200 import fp8q
from paper_2601_18150_b200.sync import TensorSpec, WeightSyncEngine

dev = torch.device("cuda")
g = torch.Generator(device=dev); g.manual_seed(0)
M = 8192
lay = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 24576, 4096), ("down", 4096, 12288)]
w = {n: (torch.randn((nn, k), generator=g, device=dev) * 0.02).to(torch.bfloat16) for n, nn, k in lay}
x = {n: torch.randn((M, k), generator=g, device=dev).to(torch.bfloat16) for n, _, k in lay}
eng = WeightSyncEngine([TensorSpec(n, nn, k) for n, nn, k in lay], dev)
eng.sync_step(1, w)
xq = {n: torch.empty((M, k), dtype=torch.uint8, device=dev) for n, _, k in lay}
xs = {n: torch.empty((k // 128, M), dtype=torch.float32, device=dev) for n, _, k in lay}
fp8q.quantize_act_per_token_group_batched([(x[n], xq[n], xs[n]) for n, _, _ in lay])
y = {n: torch.empty((M, nn), dtype=torch.bfloat16, device=dev) for n, nn, _ in lay}
for n, _, _ in lay:
    fp8q.fp8_block_gemm(xq[n], xs[n], eng.codes[n], eng.scales[n], out=y[n])
E, n2, k2 = synth.QWEN3_30B_EXPERTS["down"]
we = (torch.randn((E * n2, k2), generator=g, device=dev) * 0.02).to(torch.bfloat16)
wq, ws = fp8q.quantize_weight_blockwise(we)
sizes = synth.moe_group_sizes(8192, seed=0)
off = torch.from_numpy(synth.offsets_from_sizes(sizes)).to(dev)
rows = int(sizes.sum())
xe = torch.randn((rows, k2), generator=g, device=dev).to(torch.bfloat16)
aq, asc = fp8q.quantize_act_per_token_group(xe)
ye = torch.empty((rows, n2), dtype=torch.bfloat16, device=dev)
fp8q.fp8_block_gemm_grouped(aq, asc, wq.view(E, n2, k2), ws.view(E, n2 // 128, k2 // 128), off, out=ye)
torch.cuda.synchronize()
print("ok")
