mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -k dev_kinds > gpurun_out/kinds.log 2>&1; echo kinds=$?
tail -2 gpurun_out/kinds.log
python - <<'PY'
import torch, sys
sys.path.insert(0, ".")
from paper_2601_18150_b200 import fp8q
dev = torch.device("cuda")
for (m, n, k) in [(65536, 2048, 768), (65536, 1536, 2048), (8192, 24576, 768)]:
    w = (torch.randn((n, k), device=dev) * 0.02).to(torch.bfloat16)
    x = torch.randn((m, k), device=dev).to(torch.bfloat16)
    wq, ws = fp8q.quantize_weight_blockwise(w)
    xq, xs = fp8q.quantize_act_per_token_group(x)
    y = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
    for _ in range(3): fp8q.fp8_block_gemm(xq, xs, wq, ws, out=y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): fp8q.fp8_block_gemm(xq, xs, wq, ws, out=y)
    b.record(); b.synchronize()
    t = a.elapsed_time(b) / 10
    print("dense", (m, n, k), f"{t*1e3:.1f} us", f"{2*m*n*k/t/1e9:.0f} TFLOP/s")
PY
