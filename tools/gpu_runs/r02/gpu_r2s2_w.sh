# run W: why the 192 KB operand ring fails to launch (error string), one shape
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2601_18150_b200 import fp8q
x=torch.randn(8192,4096,device='cuda').to(torch.bfloat16); w=(torch.randn(6144,4096,device='cuda')*0.02).to(torch.bfloat16)
xq,xs=fp8q.quantize_act_per_token_group(x); wq,ws=fp8q.quantize_weight_blockwise(w)
try:
    fp8q.fp8_block_gemm(xq,xs,wq,ws); torch.cuda.synchronize(); print('pair ok')
except Exception as e: print('pair', e)
x2=x[:300].contiguous(); a,b=fp8q.quantize_act_per_token_group(x2)
try:
    fp8q.fp8_block_gemm(a,b,wq,ws); torch.cuda.synchronize(); print('one-cta ok')
except Exception as e: print('one-cta', e)
print(torch.cuda.get_device_properties(0))
" > gpurun_out/w_err.txt 2>&1
