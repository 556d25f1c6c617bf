"""fp8_linear_dynamic: one W8A8 linear with the activations quantized
dynamically inside the call (at m <= 16 by the decode GEMM itself, in shared memory; otherwise
the quantizer and the GEMM chained by programmatic dependent launch, the codes in the caller's
workspace).  Bar: BIT-identical to the separate
quantize_act_per_token_group + fp8_block_gemm calls (which the other suites pin to the oracle);
plus a direct oracle check (oracle quantizer, fp64 GEMM) on the outputs."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import rel_frobenius, to_dev_bf16

pytestmark = pytest.mark.gpu


def _weight(n, k, seed):
    wb = synth.qwen3_weight(n, k, seed)
    wq, ws = fp8q.quantize_weight_blockwise(to_dev_bf16(wb))
    return wb, wq, ws


@pytest.mark.parametrize("m", [1, 2, 5, 16, 17, 31, 32, 33, 64, 65, 128, 300])
@pytest.mark.parametrize("n,k", [(6144, 4096), (4096, 12288), (1024, 384), (520, 256)])
def test_linear_dynamic_equals_two_step(m, n, k):
    _, wq, ws = _weight(n, k, 7)
    xb = synth.qwen3_activation(m, k, seed=m + k)
    x = to_dev_bf16(xb)
    for dt in (torch.float32, torch.bfloat16):
        y = fp8q.fp8_linear_dynamic(x, wq, ws, out_dtype=dt)
        xq, xs = fp8q.quantize_act_per_token_group(x)
        ref = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=dt)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16 if dt == torch.bfloat16 else torch.int32),
                           ref.view(torch.int16 if dt == torch.bfloat16 else torch.int32)), (m, n, k, dt)


@pytest.mark.parametrize("m,n,k", [(8192, 6144, 4096), (2048, 512, 12288)])
def test_linear_dynamic_equals_two_step_tail_split(m, n, k):
    # prefill shapes whose CTA-pair GEMM splits its tail-wave tiles along K (gemm.cu plan_split):
    # the linear's workspace carries the split partials too, and both paths take the same plan
    lib = fp8q.load_library()
    assert lib.fp8_block_gemm_workspace_size(m, n, k) > 0
    _, wq, ws = _weight(n, k, 9)
    x = to_dev_bf16(synth.qwen3_activation(m, k, seed=5))
    y = fp8q.fp8_linear_dynamic(x, wq, ws)
    xq, xs = fp8q.quantize_act_per_token_group(x)
    ref = fp8q.fp8_block_gemm(xq, xs, wq, ws)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("m", [1, 7, 16])
@pytest.mark.parametrize("n,k,launches", [(24576, 4096, 1), (4096, 4096, 1), (256, 16384, 1), (3072, 2048, 1),
                                          (24576, 8192, 2)])
def test_linear_dynamic_fused_decode_modes(m, n, k, launches):
    # m <= 16: the decode GEMM quantizes its own activations where its CTAs' k-blocks fit the
    # shared-memory slots -- ordered stream-K whose ranges cross tiles (gate_up: every k-block),
    # cluster split-K (o_proj: cs = 4; 2 tiles of K = 16384: cs = 8, 16 k-blocks per CTA) -- and
    # falls back to two launches where they do not (stream-K over 64 k-blocks); every mode
    # bit-identical to the separate calls
    _, wq, ws = _weight(n, k, 13)
    x = to_dev_bf16(synth.qwen3_activation(m, k, seed=3 * m + 1))
    for dt in (torch.float32, torch.bfloat16):
        before = fp8q.kernel_launches()
        y = fp8q.fp8_linear_dynamic(x, wq, ws, out_dtype=dt)
        assert fp8q.kernel_launches() - before == launches, (m, n, k)
        xq, xs = fp8q.quantize_act_per_token_group(x)
        ref = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=dt)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16 if dt == torch.bfloat16 else torch.int32),
                           ref.view(torch.int16 if dt == torch.bfloat16 else torch.int32)), (m, n, k, dt)


@pytest.mark.parametrize("m", [1, 8, 40])
def test_linear_dynamic_against_oracle(m):
    n, k = 768, 1024
    wb, wq, ws = _weight(n, k, 3)
    xb = synth.qwen3_activation(m, k, seed=11)
    y = fp8q.fp8_linear_dynamic(to_dev_bf16(xb), wq, ws, out_dtype=torch.float32)
    torch.cuda.synchronize()
    oa, osa = oracle.quantize_act_per_token_group(xb)
    ow, osw = oracle.quantize_weight_blockwise(wb)
    ref = oracle.gemm_rows(oa, osa, ow, osw)
    assert rel_frobenius(y.cpu().numpy(), ref) <= 1e-5


def test_linear_dynamic_ragged_strided_and_flag():
    n, k = 384, 640
    _, wq, ws = _weight(n, k, 5)
    big = torch.zeros((9, k + 64), dtype=torch.bfloat16, device="cuda")
    big[:, :k] = to_dev_bf16(synth.qwen3_activation(9, k, seed=2))
    x = big[:, :k]  # row stride k + 64
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    y = fp8q.fp8_linear_dynamic(x, wq, ws, out_dtype=torch.float32, nonfinite_flag=flag)
    xq, xs = fp8q.quantize_act_per_token_group(x.contiguous())
    ref = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32), ref.view(torch.int32))
    assert int(flag.item()) == 0
    big[3, 17] = float("inf")
    fp8q.fp8_linear_dynamic(x, wq, ws, nonfinite_flag=flag)
    torch.cuda.synchronize()
    assert int(flag.item()) == 1


def test_linear_dynamic_extremes():
    # full-range activation bits (tiny groups on the division path, huge values) through the
    # fused quantizer: still identical to the two-step path
    n, k = 256, 512
    _, wq, ws = _weight(n, k, 9)
    xb = synth.uniform_bits((12, k), 4, lo=0x0001, hi=0x4700)
    xb[::3] |= 0x8000
    xb[5, :128] = 0
    xb[6, 128:256] = 0x0001
    x = to_dev_bf16(xb)
    y = fp8q.fp8_linear_dynamic(x, wq, ws, out_dtype=torch.float32)
    xq, xs = fp8q.quantize_act_per_token_group(x)
    ref = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32), ref.view(torch.int32))
