"""Column-parallel shard GEMMs (north_star: "The GEMM is reported ... as column-parallel
shards"): the N/P slices of the Qwen3 weights at prefill M (few 256 x 256 tiles, ragged N,
short K) -- parity against the oracle on sampled rows, bitwise determinism, BF16 = RNE(F32)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import rel_frobenius, to_dev_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k", [(8192, 768, 4096), (8192, 256, 4096), (8192, 640, 2048), (2048, 512, 4096),
                                   (4096, 384, 1024)])
def test_shard_gemm(m, n, k):
    wb = synth.qwen3_weight(n, k, 3)
    xb = synth.qwen3_activation(m, k, 4)
    wq, ws = fp8q.quantize_weight_blockwise(to_dev_bf16(wb))
    xq, xs = fp8q.quantize_act_per_token_group(to_dev_bf16(xb))
    y = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=torch.float32)
    y2 = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=torch.float32)
    yb = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32), y2.view(torch.int32))  # deterministic
    assert torch.equal(yb.view(torch.int16), y.to(torch.bfloat16).view(torch.int16))
    rows = np.unique(np.r_[0, m - 1, np.random.default_rng(m + n).integers(0, m, 24)])
    oa, osa = oracle.quantize_act_per_token_group(xb[rows])
    ow, osw = oracle.quantize_weight_blockwise(wb)
    ref = oracle.gemm_rows(oa, osa, ow, osw)
    assert rel_frobenius(y[torch.from_numpy(rows).cuda()].cpu().numpy(), ref) <= 1e-5
