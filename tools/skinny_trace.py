#!/usr/bin/env python3
"""Dev tool: CTA 0's timeline (SM clock cycles) for one decode-kernel (gemm_skinny.cu) launch.
Per k-block: 0 producer issue, 1 MMA sees stage full, 2 promotion sees partial, 3 promotion
done.  Row 0 also: 4 kernel entry, 5 after setup, 6 exit.  usage: skinny_trace.py M N K"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_18150_b200 import fp8q  # noqa: E402

m, n, k = (int(a) for a in sys.argv[1:4])
dev = torch.device("cuda")
g = torch.Generator(device=dev)
g.manual_seed(0)
w = (torch.randn((n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
x = torch.randn((m, k), generator=g, device=dev).to(torch.bfloat16)
wq, ws = fp8q.quantize_weight_blockwise(w)
xq, xs = fp8q.quantize_act_per_token_group(x)
lib = fp8q.load_library()
lib.fp8q_debug_set_gemm_trace.argtypes = [ctypes.c_void_p]
tr = torch.zeros(96 * 12 + 1024, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    fp8q.fp8_block_gemm(xq, xs, wq, ws)
wq2 = wq.clone()
flush.view(torch.int64).sum()
torch.cuda._sleep(400_000)
if "--pair" in sys.argv:  # a first GEMM (untraced) right before the traced one: PDL overlap
    fp8q.fp8_block_gemm(xq, xs, wq2, ws)
lib.fp8q_debug_set_gemm_trace(tr.data_ptr())
fp8q.fp8_block_gemm(xq, xs, wq, ws)
torch.cuda.synchronize()
lib.fp8q_debug_set_gemm_trace(None)
allt = tr.cpu().numpy().view(np.uint32).astype(np.int64)
t = allt[:1152].reshape(96, 12)
cta = allt[1152:].reshape(256, 4)
live = np.nonzero(cta[:, 1])[0]
t0 = cta[live, 0].min()
ent, ext = (cta[live, 0] - t0) % (1 << 32), (cta[live, 1] - t0) % (1 << 32)
print(f"CTAs {len(live)}: entry ns min/med/max {ent.min()}/{int(np.median(ent))}/{ent.max()}  "
      f"exit ns min/med/max {ext.min()}/{int(np.median(ext))}/{ext.max()}")
print("exit histogram (us):", np.histogram(ext / 1000, bins=8)[0].tolist(), np.round(np.histogram(ext / 1000, bins=8)[1], 1).tolist())
first, sdone = (cta[live, 2] - t0) % (1 << 32), (cta[live, 3] - t0) % (1 << 32)
print(f"first partial ns min/med/max {first.min()}/{int(np.median(first))}/{first.max()}  "
      f"stream done ns min/med/max {sdone.min()}/{int(np.median(sdone))}/{sdone.max()}")
slow = np.argsort(ext)[-6:]
for i in slow:
    print(f"  slow CTA {live[i]:3d}: entry {ent[i]} first {first[i]} stream_done {sdone[i]} exit {ext[i]}")
base = t[0, 4]
rel = (t - base) % (1 << 32)
print(f"entry 0  setup_done {rel[0, 5]}  dependency_wait_done {rel[0, 7]}  exit {rel[0, 6]}")
print("it   issue   full   tfull   done   full-issue  tfull-full  done-tfull")
last = int(np.max(np.nonzero(t[:, 0])[0])) if np.any(t[:, 0]) else -1
for i in range(last + 1):
    r = rel[i]
    print(f"{i:3d} {r[0]:7d} {r[1]:7d} {r[2]:7d} {r[3]:7d}  {r[1] - r[0]:8d} {r[2] - r[1]:8d} {r[3] - r[2]:8d}")
