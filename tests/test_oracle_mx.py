"""Pins for the NEXT-4 MXFP8 oracle (readings X1-X3 in DESIGN.md §3):
power-of-two (E8M0) scales on 1x32 blocks, the smallest 2^e with 448 * 2^e >= amax.

Pins (none re-types the oracle): exact rational/frexp arithmetic for the exponent over every
positive finite BF16 amax; an independent numpy/torch implementation of the block quantizer
(numpy amax, exact power-of-two division, torch float8_e4m3fn cast); closed forms (amax exactly
448 * 2^e -> code 0x7E, zero block -> scale byte 127); the no-saturation property; and a numpy
fp64 matmul of the dequantized operands for the GEMM reference.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth


def indep_exponent(amax: float) -> int:
    if amax == 0.0:
        return 0
    # smallest e with 448 * 2^e >= amax, by frexp: amax = f 2^p, f in [0.5, 1)
    f, p = math.frexp(amax / 448.0)  # amax / 448 in binary64 is exact enough to compare below
    e = p - 1 if f == 0.5 else p
    while 448.0 * 2.0 ** (e - 1) >= amax:  # exact comparisons in binary64 (BF16 amax)
        e -= 1
    while 448.0 * 2.0 ** e < amax:
        e += 1
    return max(e, -127)


def test_mx_exponent_all_bf16_amax():
    bits = np.arange(1, 0x7F80, dtype=np.uint32).astype(np.uint16)
    vals = synth.bf16_bits_to_f32(bits)
    for b, v in zip(bits[::7], vals[::7]):
        assert oracle.mx_exponent(float(v)) == indep_exponent(float(v)), hex(int(b))
    assert oracle.mx_exponent(0.0) == 0
    assert oracle.mx_exponent(448.0) == 0 and oracle.mx_exponent(449.0) == 1 and oracle.mx_exponent(224.0) == -1


def indep_mx_quantize(bits: np.ndarray):
    x = synth.bf16_bits_to_f32(bits).astype(np.float64)
    rows, cols = x.shape
    nb = -(-cols // 32)
    codes = np.empty((rows, cols), np.uint8)
    sf = np.empty((rows, nb), np.uint8)
    for r in range(rows):
        for b in range(nb):
            blk = x[r, 32 * b:32 * b + 32]
            e = indep_exponent(float(np.max(np.abs(blk))))
            sf[r, b] = e + 127
            q = torch.from_numpy((blk / 2.0 ** e).astype(np.float32))
            assert float(q.abs().max()) <= 448.0  # X2: no element saturates
            codes[r, 32 * b:32 * b + 32] = q.to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    return codes, sf


@pytest.mark.parametrize("rows,cols,kind", [(3, 256, "act"), (5, 200, "weight"), (2, 4096, "act"), (4, 96, "wide")])
def test_mx_quantize_matches_library(rows, cols, kind):
    if kind == "act":
        bits = synth.qwen3_activation(rows, cols, 3)
    elif kind == "weight":
        bits = synth.qwen3_weight(rows, cols, 4)
    else:
        bits = synth.uniform_bits((rows, cols), 5, lo=0x0001, hi=0x7F00)
    c, s = oracle.mx_quantize(bits)
    ci, si = indep_mx_quantize(bits)
    assert np.array_equal(s, si)
    assert np.array_equal(c, ci)


def test_mx_closed_forms():
    x = np.zeros((2, 64), np.float32)
    x[0, :32] = 448.0 * 4.0
    x[0, 5] = -448.0 * 4.0
    x[1, 40] = 3.0
    c, s = oracle.mx_quantize(synth.f32_to_bf16_bits(x))
    assert s[0, 0] == 127 + 2 and c[0, 0] == 0x7E and c[0, 5] == 0xFE
    assert s[0, 1] == 127 and np.all(c[0, 32:] == 0)  # zero block -> scale byte 127 (2^0)
    assert s[1, 1] == 127 + oracle.mx_exponent(3.0) and s[1, 0] == 127


def test_mx_gemm_reference_matches_numpy():
    a, sfa = oracle.mx_quantize(synth.qwen3_activation(4, 256, 1))
    b, sfb = oracle.mx_quantize(synth.qwen3_weight(16, 256, 2))
    dec = torch.arange(256, dtype=torch.int32).to(torch.uint8).view(torch.float8_e4m3fn).double().numpy()
    av = dec[a] * np.repeat(np.exp2(sfa.astype(np.float64) - 127), 32, axis=1)
    bv = dec[b] * np.repeat(np.exp2(sfb.astype(np.float64) - 127), 32, axis=1)
    ref = av @ bv.T
    got = oracle.mx_gemm_rows(a, sfa, b, sfb)
    assert np.allclose(got, ref, rtol=1e-13, atol=0)
