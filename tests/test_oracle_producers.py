"""Pins for the NEXT-2 producer oracles: binary64 -> BF16 rounding,
RMSNorm and SiLU(gate)*up, each rounded to BF16 before the per-token-group quantizer (the
unfused pipeline's definition).

Pins: an independent Python implementation of round-to-nearest-even to 8 significant bits
(built on Python's correctly rounded round()), exhaustive BF16 round trips and midpoints,
numpy binary64 RMSNorm / SiLU, and closed forms (constant row -> gamma, one-hot row -> sqrt(K)
gamma, silu(0) = 0, scale invariance of RMSNorm).
"""
import math

import numpy as np
import pytest

import oracle
import synth


def py_round_bf16(d: float) -> int:
    """Independent RNE of a binary64 to BF16 bits (normal range), via Python's round()."""
    if d == 0.0:
        return 0x8000 if math.copysign(1.0, d) < 0 else 0
    m, e = math.frexp(abs(d))          # |d| = m 2^e, m in [0.5, 1)
    r = round(m * 256.0)               # exact product; round() is half-to-even
    v = math.ldexp(r, e - 8)
    bits = int(np.float32(v).view(np.uint32)) >> 16
    return bits | (0x8000 if d < 0 else 0)


def test_f64_to_bf16_roundtrip_and_midpoints():
    # every finite BF16 value round-trips; every midpoint goes to the even neighbour
    for b in range(0x0080, 0x7F80, 7):  # normal BF16 values
        v = float(synth.bf16_bits_to_f32(np.uint16(b)))
        assert oracle.f64_to_bf16(v) == b and oracle.f64_to_bf16(-v) == b | 0x8000
        nxt = float(synth.bf16_bits_to_f32(np.uint16(b + 1)))
        mid = (v + nxt) / 2
        assert oracle.f64_to_bf16(mid) == (b if b % 2 == 0 else b + 1)
        assert oracle.f64_to_bf16(math.nextafter(mid, 0)) == b
        assert oracle.f64_to_bf16(math.nextafter(mid, math.inf)) == b + 1
    assert oracle.f64_to_bf16(0.0) == 0 and oracle.f64_to_bf16(-0.0) == 0x8000


def test_f64_to_bf16_matches_independent_rounding():
    rng = np.random.default_rng(0)
    for d in rng.standard_normal(20000) * np.exp2(rng.integers(-60, 60, 20000)):
        assert oracle.f64_to_bf16(float(d)) == py_round_bf16(float(d))


@pytest.mark.parametrize("m,k,eps", [(4, 4096, 1e-6), (3, 2048, 1e-5), (2, 768, 1e-6)])
def test_rmsnorm_matches_numpy_fp64(m, k, eps):
    x = synth.qwen3_activation(m, k, seed=k)
    g = synth.f32_to_bf16_bits((1.0 + 0.1 * np.random.default_rng(k).standard_normal(k)).astype(np.float32))
    y = oracle.rmsnorm_bf16(x, g, eps)
    xf = synth.bf16_bits_to_f32(x).astype(np.float64)
    gf = synth.bf16_bits_to_f32(g).astype(np.float64)
    inv = 1.0 / np.sqrt((xf * xf).sum(axis=1, keepdims=True) / k + float(np.float32(eps)))
    ref = xf * inv * gf
    want = np.array([[py_round_bf16(float(v)) for v in row] for row in ref], dtype=np.uint16)
    # numpy's pairwise summation order differs from the oracle's sequential sum: the binary64
    # results agree to ~1e-15 relative, so at most a vanishing number of BF16 ties may differ
    assert np.count_nonzero(y != want) <= max(1, y.size // 10000)


def test_rmsnorm_closed_forms():
    k = 4096
    g = synth.f32_to_bf16_bits((1.0 + np.arange(k) % 7 * 0.125).astype(np.float32))
    x = np.zeros((3, k), np.float32)
    x[0, :] = 3.0                      # constant row -> y = gamma
    x[1, :] = -0.5                     # negative constant -> -gamma
    x[2, 123] = 2.0                    # one-hot -> y_j = sqrt(K) gamma_j = 64 gamma_j
    y = oracle.rmsnorm_bf16(synth.f32_to_bf16_bits(x), g, 0.0)
    assert np.array_equal(y[0], g)
    assert np.array_equal(y[1], g | np.uint16(0x8000))
    gf = synth.bf16_bits_to_f32(g)
    assert synth.bf16_bits_to_f32(y[2, 123]) == 64.0 * gf[123]
    assert np.count_nonzero(y[2]) == 1
    # scale invariance (eps = 0): x and 4x normalise to the same BF16 values
    xr = synth.qwen3_activation(2, k, seed=3)
    x4 = synth.f32_to_bf16_bits(synth.bf16_bits_to_f32(xr) * 4.0)
    assert np.array_equal(oracle.rmsnorm_bf16(xr, g, 0.0), oracle.rmsnorm_bf16(x4, g, 0.0))


def test_silu_mul_matches_numpy_and_closed_forms():
    m, inter = 3, 512
    gu = synth.qwen3_activation(m, 2 * inter, seed=9)
    y = oracle.silu_mul_bf16(gu)
    f = synth.bf16_bits_to_f32(gu).astype(np.float64)
    g, u = f[:, :inter], f[:, inter:]
    ref = g / (1.0 + np.exp(-g)) * u
    want = np.array([[py_round_bf16(float(v)) for v in row] for row in ref], dtype=np.uint16)
    assert np.count_nonzero(y != want) <= 1
    z = np.zeros((1, 8), np.float32)
    z[0, :4] = [0.0, 40.0, -40.0, 1.0]
    z[0, 4:] = [5.0, 3.0, 2.0, 1.0]
    yz = synth.bf16_bits_to_f32(oracle.silu_mul_bf16(synth.f32_to_bf16_bits(z)))[0]
    assert yz[0] == 0.0                           # silu(0) * u = 0
    assert yz[1] == 120.0                         # silu(40) = 40 in binary64 -> 40 * 3
    assert -1e-15 < yz[2] <= 0.0                  # silu(-40) ~ -1.7e-16 * 2
    assert yz[3] == float(synth.bf16_bits_to_f32(np.uint16(py_round_bf16(1.0 / (1.0 + math.exp(-1.0))))))


def test_producer_quantize_composition():
    # the fused definitions are exactly "producer in BF16, then O3-O6"
    x = synth.qwen3_activation(5, 2048, seed=1)
    g = synth.f32_to_bf16_bits(np.ones(2048, np.float32))
    y, codes, scales = oracle.rmsnorm_quantize(x, g, 1e-6)
    c2, s2 = oracle.quantize_act_per_token_group(y)
    assert np.array_equal(codes, c2) and np.array_equal(scales, s2)
