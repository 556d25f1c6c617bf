"""GPU parity of the NEXT-4 MXFP8 variant against its oracle (readings X1-X3): the quantizer
bit-exact (codes and E8M0 scale bytes, native layout mapped back to [rows, k/32]), and the
block-scaled tcgen05 GEMM against the fp64 reference (rel. Frobenius <= 1e-5 on F32 output,
bitwise on an exact scale-probe case; BF16 = RNE of F32)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import rel_frobenius, to_dev_bf16, to_host_u8

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,k,kind", [(1, 128, "act"), (37, 4096, "act"), (300, 384, "weight"), (256, 2048, "wide"),
                                          (129, 768, "act")])
def test_mx_quantize_bit_exact(rows, k, kind):
    if kind == "act":
        bits = synth.qwen3_activation(rows, k, 1)
    elif kind == "weight":
        bits = synth.qwen3_weight(rows, k, 2)
    else:
        bits = synth.uniform_bits((rows, k), 3, lo=0x0001, hi=0x7F00)
    codes, sf = fp8q.mx_quantize(to_dev_bf16(bits))
    torch.cuda.synchronize()
    oc, osf = oracle.mx_quantize(bits)
    assert np.array_equal(fp8q.mx_scales_logical(sf, rows, k), osf)
    assert np.array_equal(to_host_u8(codes), oc)


def _mx_operands(m, n, k, seed):
    xa = synth.qwen3_activation(m, k, seed)
    xw = synth.qwen3_weight(n, k, seed + 1)
    a, sa = fp8q.mx_quantize(to_dev_bf16(xa))
    b, sb = fp8q.mx_quantize(to_dev_bf16(xw))
    torch.cuda.synchronize()
    return a, sa, b, sb


@pytest.mark.parametrize("m,n,k", [(128, 256, 128), (37, 512, 1024), (300, 768, 512), (1000, 256, 4096)])
def test_mx_gemm_vs_oracle(m, n, k):
    a, sa, b, sb = _mx_operands(m, n, k, 5)
    y = fp8q.fp8_mx_gemm(a, sa, b, sb, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rows = np.arange(m) if m <= 64 else np.unique(np.r_[0, m - 1, np.random.default_rng(m).integers(0, m, 30)])
    ref = oracle.mx_gemm_rows(to_host_u8(a), fp8q.mx_scales_logical(sa, m, k), to_host_u8(b),
                              fp8q.mx_scales_logical(sb, n, k), rows)
    got = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert rel_frobenius(got, ref) <= 1e-5
    yb = fp8q.fp8_mx_gemm(a, sa, b, sb, out_dtype=torch.bfloat16)
    assert torch.equal(yb.view(torch.int16), y.to(torch.bfloat16).view(torch.int16))


def test_mx_gemm_scale_probe_bitwise():
    # every 1x32 block is the constant +-448 * 2^e: codes 0x7E/0xFE, scale bytes e + 127, so
    # D[m,n] = sum over blocks of +-32 * 448^2 * 2^(ea + eb): exact in fp32 for a small spread
    m, n, k = 128, 256, 512
    rng = np.random.default_rng(7)
    ea = rng.integers(-3, 4, size=(m, k // 32))
    eb = rng.integers(-3, 4, size=(n, k // 32))
    sa_ = rng.choice([-1, 1], size=(m, k // 32))
    sb_ = rng.choice([-1, 1], size=(n, k // 32))
    xa = np.repeat(sa_ * 448.0 * np.exp2(ea), 32, axis=1).astype(np.float32)
    xb = np.repeat(sb_ * 448.0 * np.exp2(eb), 32, axis=1).astype(np.float32)
    a, sa = fp8q.mx_quantize(to_dev_bf16(synth.f32_to_bf16_bits(xa)))
    b, sb = fp8q.mx_quantize(to_dev_bf16(synth.f32_to_bf16_bits(xb)))
    y = fp8q.fp8_mx_gemm(a, sa, b, sb, out_dtype=torch.float32).cpu().numpy().astype(np.float64)
    want = np.einsum("mj,nj->mn", sa_ * np.exp2(ea), sb_ * np.exp2(eb)) * 32 * 448.0 * 448.0
    assert np.array_equal(y, want)


def test_mx_gemm_full_size_sampled():
    # Qwen3-8B qkv at M = 8192 (the bench shape), sampled rows against the oracle
    m, n, k = 8192, 6144, 4096
    a, sa, b, sb = _mx_operands(m, n, k, 9)
    y = fp8q.fp8_mx_gemm(a, sa, b, sb, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rows = np.unique(np.r_[0, 127, 128, m - 1, np.random.default_rng(3).integers(0, m, 6)])
    ref = oracle.mx_gemm_rows(to_host_u8(a[torch.from_numpy(rows).cuda()]),
                              fp8q.mx_scales_logical(sa, m, k)[rows], to_host_u8(b),
                              fp8q.mx_scales_logical(sb, n, k))
    assert rel_frobenius(y[torch.from_numpy(rows).cuda()].cpu().numpy(), ref) <= 1e-5
