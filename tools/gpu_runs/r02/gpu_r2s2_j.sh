# run J: paired weight-tile issue A/B for the decode kernel + ncu of one decode GEMM (clock-control none)
timeout 300 python tools/kernel_bench.py --what none --decode --graph --flush read > gpurun_out/j_base.txt 2>&1
FP8Q_SKINNY_PAIRW=1 timeout 300 python tools/kernel_bench.py --what none --decode --graph --flush read > gpurun_out/j_pairw.txt 2>&1
FP8Q_SKINNY_PAIRW=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x -k "skinny or decode" 2>&1 | tail -3 > gpurun_out/j_tests.txt
timeout 600 ncu --set full --clock-control none -k regex:skinny -c 2 -o gpurun_out/j_dec python -c "
import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16
for n,k in [(24576,4096),(4096,12288)]:
    w = to_dev_bf16(synth.qwen3_weight(n, k, 1)); wq, ws = fp8q.quantize_weight_blockwise(w)
    x = to_dev_bf16(synth.qwen3_activation(1, k, 2)); xq, xs = fp8q.quantize_act_per_token_group(x)
    y = fp8q.fp8_block_gemm(xq, xs, wq, ws); torch.cuda.synchronize()
" > gpurun_out/j_ncu.txt 2>&1
