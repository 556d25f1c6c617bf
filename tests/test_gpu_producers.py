"""GPU parity of the NEXT-2 producer-fused quantizers against the oracle.

Definition (oracle/producers.py, readings N1/N2): Qwen3's RMSNorm / SiLU(gate)*up
as HF evaluates them (binary32, two BF16 roundings), every step correctly rounded, the sum of
squares exact and silu correctly rounded from its real value; then the per-token-group
quantizer.  Bar: y, codes and scales BIT-EXACT against the oracle's
definition -- element by element, no tolerance.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import act_scales_logical, to_dev_bf16, to_host_u8

pytestmark = pytest.mark.gpu


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def _check_exact(y_dev, codes_dev, scales_dev, y_or, m, k):
    y = _bits(y_dev)
    nd = np.count_nonzero(y != y_or)
    assert nd == 0, f"{nd} BF16 outputs differ from the oracle"
    oc, os_ = oracle.quantize_act_per_token_group(y_or)
    assert np.array_equal(act_scales_logical(scales_dev, m).view(np.uint32), os_.view(np.uint32))
    assert np.array_equal(to_host_u8(codes_dev), oc)


def _rms(xb, gb, eps):
    m, k = xb.shape
    x, g = to_dev_bf16(xb), to_dev_bf16(gb)
    y = torch.empty((m, k), dtype=torch.bfloat16, device="cuda")
    codes, scales = fp8q.rmsnorm_quantize_act_per_token_group(x, g, eps, y_out=y)
    c2, s2 = fp8q.rmsnorm_quantize_act_per_token_group(x, g, eps)  # no y output: same bytes
    torch.cuda.synchronize()
    assert torch.equal(c2, codes) and torch.equal(s2[:, :m], scales[:, :m])
    return y, codes, scales


@pytest.mark.parametrize("m,k,seed", [(4, 4096, 0), (37, 2048, 1), (1, 4096, 2), (5, 768, 3), (3, 128, 4),
                                      (2048, 4096, 5), (129, 384, 6), (64, 3072, 7), (16, 1280, 8)])
def test_rmsnorm_quantize(m, k, seed):
    xb = synth.qwen3_activation(m, k, seed)
    gb = synth.f32_to_bf16_bits((1.0 + 0.2 * np.random.default_rng(seed).standard_normal(k)).astype(np.float32))
    eps = 1e-6
    y, codes, scales = _rms(xb, gb, eps)
    _check_exact(y, codes, scales, oracle.rmsnorm_bf16(xb, gb, eps), m, k)


def test_rmsnorm_full_range_rows():
    # random finite BF16 over the whole range: wide dynamic range (the binary64 sum is inexact),
    # subnormal mean squares, overflowing products -- the exact-sum path and IEEE edge cases
    k = 1024
    xb = synth.uniform_bits((64, k), 11, lo=0x0001, hi=0x5F00)  # |x| < 2^63: squares stay finite
    xb[::2] |= 0x8000
    xb[5] = synth.uniform_bits((1, k), 12, lo=0x0001, hi=0x0100)[0]  # tiny row: subnormal mean square
    gb = synth.f32_to_bf16_bits((1.0 + 0.2 * np.random.default_rng(1).standard_normal(k)).astype(np.float32))
    y, codes, scales = _rms(xb, gb, 1e-6)
    _check_exact(y, codes, scales, oracle.rmsnorm_bf16(xb, gb, 1e-6), 64, k)


def test_rmsnorm_mean_of_squares_ties():
    # rows whose mean of squares is EXACTLY a binary32 midpoint (1 + 2^-24, ties to even), or
    # lies 2^-120-ish above one (the binary64 sum loses it): the kernel must take its exact path
    k = 256
    rows = []
    for extra in (None, 2.0 ** -60, 2.0 ** -30):
        row = np.zeros(k, np.float32)
        row[:240] = 1.0
        row[240:244] = 2.0
        row[244:248] = 2.0 ** -9
        if extra is not None:
            row[250] = extra
        rows.append(row)
    for sc in (2.0 ** -40, 2.0 ** 20, 3.0):  # scaled copies (3: not a power of two, no tie)
        rows.append(rows[0] * sc)
    xb = synth.f32_to_bf16_bits(np.stack(rows))
    gb = synth.f32_to_bf16_bits(np.linspace(0.5, 2.0, k).astype(np.float32))
    for eps in (0.0, 1e-6):
        y, codes, scales = _rms(xb, gb, eps)
        _check_exact(y, codes, scales, oracle.rmsnorm_bf16(xb, gb, eps), len(rows), k)


def test_rmsnorm_full_size_sampled():
    # the bench-sized input (8192 x 4096): every row's y bit-exact on a sample of rows, and the
    # kernel's codes/scales equal the oracle quantizer of the oracle y on those rows
    m, k = 8192, 4096
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    x = torch.randn((m, k), generator=g, device="cuda").to(torch.bfloat16)
    x[:, ::613] *= 50
    gamma = (1 + 0.1 * torch.randn(k, generator=g, device="cuda")).to(torch.bfloat16)
    y = torch.empty((m, k), dtype=torch.bfloat16, device="cuda")
    codes, scales = fp8q.rmsnorm_quantize_act_per_token_group(x, gamma, 1e-6, y_out=y)
    torch.cuda.synchronize()
    rows = torch.arange(0, m, 97)
    xb = _bits(x[rows])
    gb = _bits(gamma)
    y_or = oracle.rmsnorm_bf16(xb, gb, 1e-6)
    assert np.array_equal(_bits(y[rows]), y_or)
    oc, os_ = oracle.quantize_act_per_token_group(y_or)
    assert np.array_equal(to_host_u8(codes[rows]), oc)
    assert np.array_equal(scales[:, rows].cpu().numpy().T.view(np.uint32), os_.view(np.uint32))


@pytest.mark.parametrize("m,inter,seed", [(4, 1536, 0), (37, 768, 1), (64, 12288, 2), (1, 128, 3), (300, 2048, 4),
                                          (7, 384, 5)])
def test_silu_mul_quantize(m, inter, seed):
    gub = synth.qwen3_activation(m, 2 * inter, seed)
    gu = to_dev_bf16(gub)
    y = torch.empty((m, inter), dtype=torch.bfloat16, device="cuda")
    codes, scales = fp8q.silu_mul_quantize_act_per_token_group(gu, y_out=y)
    torch.cuda.synchronize()
    _check_exact(y, codes, scales, oracle.silu_mul_bf16(gub), m, inter)
    c2, _ = fp8q.silu_mul_quantize_act_per_token_group(gu)
    assert torch.equal(c2, codes)


def test_silu_every_gate_value():
    # exhaustive: all 65,280 finite BF16 gate values g with up = 1 -> y = RN_BF16(silu(g)), and
    # with up = 2^-3 / 3.0 (the product's binary32 rounding and BF16 re-rounding)
    bits = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    bits = bits[(bits & 0x7F80) != 0x7F80]
    n = bits.size
    inter = 128 * 60
    rows = -(-n // inter)
    gate = np.zeros(rows * inter, np.uint16)
    gate[:n] = bits
    gate = gate.reshape(rows, inter)
    for u in (1.0, 0.125, 3.0):
        up = np.full((rows, inter), synth.f32_to_bf16_bits(np.float32(u)), np.uint16)
        gub = np.concatenate([gate, up], axis=1)
        y = torch.empty((rows, inter), dtype=torch.bfloat16, device="cuda")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        codes, scales = fp8q.silu_mul_quantize_act_per_token_group(to_dev_bf16(gub), y_out=y, nonfinite_flag=flag)
        torch.cuda.synchronize()
        y_or = oracle.silu_mul_bf16(gub)
        got = _bits(y)
        nd = np.count_nonzero(got != y_or)
        assert nd == 0, (u, nd, [(hex(a), hex(b), hex(c)) for a, b, c in
                                 zip(gate.ravel()[(got != y_or).ravel()][:5], got[got != y_or][:5],
                                     y_or[got != y_or][:5])])
        if u == 1.0:
            assert np.array_equal(got.ravel()[:n], oracle.silu_bf16_table()[bits])
        # the quantizer flags a group iff it holds a non-finite y (u = 3: s * u overflows)
        assert int(flag.item()) == int(np.any((y_or & 0x7F80) == 0x7F80))


def test_producer_validation():
    x = torch.zeros((4, 8192), dtype=torch.bfloat16, device="cuda")
    g = torch.ones(8192, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(fp8q.Fp8qError, match="SHAPE"):
        fp8q.rmsnorm_quantize_act_per_token_group(x, g, 1e-6)  # k > 4096
    with pytest.raises(fp8q.Fp8qError, match="SHAPE"):
        fp8q.silu_mul_quantize_act_per_token_group(torch.zeros((2, 200), dtype=torch.bfloat16, device="cuda"))
