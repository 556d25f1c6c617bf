# run G: XQ debug -- correctness vs oracle per path, sanitizer, ncu of one fused launch
timeout 300 python tools/xq_probe.py > gpurun_out/g_probe.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python -c "
import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16
w = to_dev_bf16(synth.qwen3_weight(1024, 384, 1)); wq, ws = fp8q.quantize_weight_blockwise(w)
x = to_dev_bf16(synth.qwen3_activation(1, 384, 2)); y = fp8q.fp8_linear_dynamic(x, wq, ws); torch.cuda.synchronize(); print('ok')
" > gpurun_out/g_race.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python -c "
import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16
w = to_dev_bf16(synth.qwen3_weight(1024, 384, 1)); wq, ws = fp8q.quantize_weight_blockwise(w)
x = to_dev_bf16(synth.qwen3_activation(1, 384, 2)); y = fp8q.fp8_linear_dynamic(x, wq, ws); torch.cuda.synchronize(); print('ok')
" > gpurun_out/g_sync.txt 2>&1
timeout 600 ncu --set full -k regex:skinny -c 1 -o gpurun_out/g_xq python -c "
import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16
w = to_dev_bf16(synth.qwen3_weight(6144, 4096, 1)); wq, ws = fp8q.quantize_weight_blockwise(w)
x = to_dev_bf16(synth.qwen3_activation(1, 4096, 2)); y = fp8q.fp8_linear_dynamic(x, wq, ws); torch.cuda.synchronize()
" > gpurun_out/g_ncu.txt 2>&1
