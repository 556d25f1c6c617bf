#!/usr/bin/env python3
"""Dev tool: print CTA 0's pipeline timeline (SM clock) for one fp8_block_gemm launch.
Events per k-block: 0 producer issue, 1 MMA sees TMEM buffer free, 2 MMA issue (smem full),
3 promotion sees partial ready, 4 promotion tile entry (first k-block of a tile only), 5 promotion done, 6/7 store begin/end."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_18150_b200 import fp8q  # noqa: E402

m, n, k = (int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (8192, 6144, 4096)
dev = torch.device("cuda")
g = torch.Generator(device=dev)
g.manual_seed(0)
w = (torch.randn((n, k), generator=g, device=dev) * 0.02).to(torch.bfloat16)
x = torch.randn((m, k), generator=g, device=dev).to(torch.bfloat16)
wq, ws = fp8q.quantize_weight_blockwise(w)
xq, xs = fp8q.quantize_act_per_token_group(x)
lib = fp8q.load_library()
lib.fp8q_debug_set_gemm_trace.argtypes = [ctypes.c_void_p]
tr = torch.zeros(96 * 12, dtype=torch.int32, device=dev)
for _ in range(3):
    fp8q.fp8_block_gemm(xq, xs, wq, ws)
lib.fp8q_debug_set_gemm_trace(tr.data_ptr())
fp8q.fp8_block_gemm(xq, xs, wq, ws)
torch.cuda.synchronize()
lib.fp8q_debug_set_gemm_trace(None)
t = tr.cpu().numpy().view(np.uint32).reshape(96, 12).astype(np.int64)
base = t[0, 0]
t = (t - base) % (1 << 32)
names = ["prod", "mma_tfree", "mma_issue", "epi_ready", "epi_entry", "epi_done", "st_begin", "st_end", "st_waited", "st_written", "st_fenced"]
print("kb  " + " ".join(f"{n_:>10s}" for n_ in names) + "   d_issue  rdy-iss  rel-rdy  done-rdy")
prev = None
for i in range(96):
    row = t[i, :11]
    d_issue = row[2] - prev if prev is not None else 0
    prev = row[2]
    print(f"{i:3d} " + " ".join(f"{v:10d}" for v in row)
          + f"  {d_issue:8d} {row[3] - row[2]:8d} {row[4] - row[3]:8d} {row[5] - row[3]:8d}")

if os.environ.get("FP8Q_GEMM_DEBUG", "0") == "1":
    # release path (dev mode 1): 3 first warp sees partial, 9 last warp sees it, 8/10 first/last
    # warp released, 11 issuer starts waiting for the buffer of k-block i, 1 issuer sees it free
    print("kb  ready_w0 ready_wlast  rel_w0 rel_wlast  mma_prewait(i+2)  tfree(i+2)   [relative to ready_w0]")
    for i in range(8, 20):
        r = t[i]
        n2 = t[i + 2]
        print(f"{i:3d} {0:8d} {r[9] - r[3]:11d} {r[8] - r[3]:8d} {r[10] - r[3]:9d} {n2[11] - r[3]:17d} {n2[1] - r[3]:11d}")
