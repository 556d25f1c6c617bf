"""Pins for oracle O3-O6 (block amax, scale, element map, layouts).

PAPER.md:54-58 (§2.1.1, Eq. (1)): W_hat = round(W / scale), scale from the block's
maximum absolute value, B = 128x128; activations dynamic, 1x128.
Readings Q2-Q8, Q10-Q12.  Pins used here (none re-types the oracle):
  * exact rational arithmetic (fractions) for RN32(amax/448) over ALL 32,639 BF16 amax
    values and for RN32(x/s) on sampled pairs;
  * an independent implementation from library routines (numpy amax + numpy binary32
    division + torch's clamped float8 cast) on random, ragged and extreme-range inputs;
  * closed forms: zero block, amax = 448, 448*I, block probes with scale exactly 2^e;
  * invariants: power-of-two equivariance, the half-ULP error bound.
"""
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import synth


def rn32_exact(q: Fraction) -> np.float32:
    """The binary32 nearest to the rational q, ties to even (by exhaustive neighbour test)."""
    guess = np.float32(float(q))  # within an ulp or so; fix up exactly below
    best = None
    cands = [guess]
    for _ in range(2):
        cands = cands + [np.nextafter(c, np.float32(np.inf)) for c in cands] + \
            [np.nextafter(c, np.float32(-np.inf)) for c in cands]
    cands = sorted(set(float(c) for c in cands if np.isfinite(c)))
    for c in cands:
        d = abs(Fraction(c) - q)
        if best is None or d < best[0]:
            best = (d, [c])
        elif d == best[0]:
            best[1].append(c)
    if len(best[1]) == 1:
        return np.float32(best[1][0])
    even = [c for c in best[1] if (np.float32(c).view(np.uint32) & 1) == 0]
    assert len(even) == 1
    return np.float32(even[0])


def indep_quantize_blocks(bits: np.ndarray, br: int, bc: int):
    """Independent library implementation of O3-O5 (numpy + torch), for cross-checking."""
    x = synth.bf16_bits_to_f32(bits)
    n, k = x.shape
    nb, kb = -(-n // br), -(-k // bc)
    scales = np.empty((nb, kb), dtype=np.float32)
    codes = np.empty((n, k), dtype=np.uint8)
    for i in range(nb):
        for j in range(kb):
            blk = x[i * br:(i + 1) * br, j * bc:(j + 1) * bc]
            amax = np.float32(np.max(np.abs(blk))) if blk.size else np.float32(0)
            s = np.float32(1.0) if amax == 0 else np.float32(amax) / np.float32(448.0)
            scales[i, j] = s
            q = (blk / s).astype(np.float32)
            t = torch.from_numpy(q).clamp(-448.0, 448.0)
            codes[i * br:(i + 1) * br, j * bc:(j + 1) * bc] = t.to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    return codes, scales


def test_scale_map_all_bf16_amax_exact_rational():
    # O4 over every positive finite BF16 amax (32,639 values), incl. subnormal results.
    amax_bits = np.arange(synth.AMAX_BITS_MIN, synth.AMAX_BITS_MAX + 1, dtype=np.uint16)
    amax = synth.bf16_bits_to_f32(amax_bits)
    # oracle scales via a 1-row weight matrix per amax (one block each)
    w = np.zeros((amax.size, 128), dtype=np.uint16)
    w[:, 0] = amax_bits
    # each row is its own block only if we quantize row by row; use activation groups instead
    _, s_act = oracle.quantize_act_per_token_group(w)
    s_act = s_act[:, 0]
    n_sub = 0
    for a, s in zip(amax, s_act):
        want = rn32_exact(Fraction(float(a)) / 448)
        assert s.view(np.uint32) == want.view(np.uint32), (a, s, want)
        n_sub += int(s < np.finfo(np.float32).tiny)
    assert n_sub == 1247  # 1,247 amax values give subnormal scales
    # the same map through the scalar entry point and through 128x128 weight blocks
    for a in amax[::997]:
        assert oracle.block_scale(a) == rn32_exact(Fraction(float(a)) / 448)


def test_zero_block_and_negative_zero():
    w = np.zeros((130, 260), dtype=np.uint16)
    w[129, 259] = 0x8000  # -0
    codes, scales = oracle.quantize_weight_blockwise(w)
    assert np.all(scales == 1.0)  # SPEC.md:111 (reading Q5)
    assert codes[129, 259] == 0x80 and np.count_nonzero(codes) == 1  # reading Q6


def test_amax_448_scale_one():
    # amax = 448 -> scale 1, the max element encodes to the max-finite code
    w = synth.f32_to_bf16_bits(np.float32([[448.0, -448.0, 1.0, 0.5]]))
    codes, scales = oracle.quantize_weight_blockwise(w)
    assert scales[0, 0] == 1.0
    assert list(codes[0]) == [0x7E, 0xFE, 0x38, 0x30]


def test_bf16_analogue_of_spec_8_96_example():
    # SPEC.md:113 uses 8.96 (not BF16-representable); nearest BF16 is 8.9375.
    a = np.float32(8.9375)
    w = synth.f32_to_bf16_bits(np.float32([[8.9375, 1.0]]))
    codes, scales = oracle.quantize_weight_blockwise(w)
    assert scales[0, 0] == rn32_exact(Fraction(8.9375) / 448)
    assert codes[0, 0] == 0x7E
    assert abs(448.0 * float(scales[0, 0]) - float(a)) <= float(a) * 2.0 ** -24


def test_448_identity():
    # 448*I with one block covering all -> diagonal 0x7E, off-diagonal 0x00
    w = synth.f32_to_bf16_bits(np.eye(128, dtype=np.float32) * 448.0)
    codes, scales = oracle.quantize_weight_blockwise(w)
    assert scales.shape == (1, 1) and scales[0, 0] == 1.0
    assert np.array_equal(codes, np.eye(128, dtype=np.uint8) * 0x7E)


@pytest.mark.parametrize("n,k", [(256, 256), (300, 200), (128, 1), (1, 128), (129, 383)])
def test_block_probe_exact_scales(n, k):
    bits, e = synth.block_probe_bits(n, k, seed=n + k)
    codes, scales = oracle.quantize_weight_blockwise(bits)
    assert np.array_equal(scales, np.exp2(e).astype(np.float32))
    sign = (bits >> 15).astype(bool)
    assert np.all(codes[~sign] == 0x7E) and np.all(codes[sign] == 0xFE)


@pytest.mark.parametrize("seed,n,k,kind", [(0, 256, 256, "normal"), (1, 300, 200, "normal"),
                                           (2, 257, 384, "uniform"), (3, 131, 136, "uniform")])
def test_weight_matches_independent_library_implementation(seed, n, k, kind):
    bits = synth.qwen3_weight(n, k, seed) if kind == "normal" else synth.uniform_bits((n, k), seed)
    codes, scales = oracle.quantize_weight_blockwise(bits)
    c2, s2 = indep_quantize_blocks(bits, 128, 128)
    assert np.array_equal(scales.view(np.uint32), s2.view(np.uint32))
    assert np.array_equal(codes, c2)


@pytest.mark.parametrize("seed,m,k,kind", [(0, 4, 256, "normal"), (1, 37, 1024, "normal"),
                                           (2, 64, 384, "uniform")])
def test_act_matches_independent_library_implementation(seed, m, k, kind):
    bits = synth.qwen3_activation(m, k, seed) if kind == "normal" else synth.uniform_bits((m, k), seed)
    codes, scales = oracle.quantize_act_per_token_group(bits)
    c2, s2 = indep_quantize_blocks(bits, 1, 128)
    assert np.array_equal(scales.view(np.uint32), s2.view(np.uint32))
    assert np.array_equal(codes, c2)


def test_act_zero_row_and_one_hot():
    x = np.zeros((3, 256), dtype=np.uint16)
    x[1] = synth.f32_to_bf16_bits(np.where(np.arange(256) == 77, 3.25, 0.0).astype(np.float32))
    x[2] = synth.f32_to_bf16_bits(np.arange(1, 257, dtype=np.float32))  # SPEC.md:133 [1..T]
    codes, scales = oracle.quantize_act_per_token_group(x)
    assert np.all(scales[0] == 1.0) and not codes[0].any()
    assert codes[1, 77] == 0x7E and np.count_nonzero(codes[1]) == 1
    assert scales[1, 1] == 1.0
    table = torch.arange(256, dtype=torch.int32).to(torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    deq = table[codes[2]] * np.repeat(scales[2], 128)
    ref = synth.bf16_bits_to_f32(x[2]).astype(np.float64)
    assert np.all(np.abs(deq - ref) <= 2.0 ** -4 * ref + 1e-6)


def test_power_of_two_equivariance():
    # quantize(2^k W) -> identical codes, scales x 2^k (normal range)
    bits = synth.qwen3_weight(256, 384, seed=5)
    x = synth.bf16_bits_to_f32(bits)
    c0, s0 = oracle.quantize_weight_blockwise(bits)
    for p in (-8, -1, 1, 8, 20):
        cp, sp = oracle.quantize_weight_blockwise(synth.f32_to_bf16_bits(x * np.float32(2.0 ** p)))
        assert np.array_equal(cp, c0)
        assert np.array_equal(sp, s0 * np.float32(2.0 ** p))


def test_error_bound_and_element_rational_check():
    # SURVEY §8(c) O3-O6 bound: r = |x/s|; |dec(q) s - x| <= (2^(floor(log2 r)-4) + 2^-24 r) s
    # for r >= 2^-6, else <= (2^-10 + 2^-24 r) s.  Plus: RN32(x/s) via exact rationals.
    bits = synth.uniform_bits((256, 256), seed=11, lo=0x2000, hi=0x6000)
    codes, scales = oracle.quantize_weight_blockwise(bits)
    x = synth.bf16_bits_to_f32(bits).astype(np.float64)
    s = np.repeat(np.repeat(scales.astype(np.float64), 128, 0), 128, 1)
    table = torch.arange(256, dtype=torch.int32).to(torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    deq = table[codes] * s
    r = np.abs(x / s)
    with np.errstate(divide="ignore"):
        tight = np.where(r >= 2.0 ** -6, 2.0 ** (np.floor(np.log2(np.maximum(r, 1e-300))) - 4), 2.0 ** -10)
    assert np.all(np.abs(deq - x) <= (tight + 2.0 ** -24 * r) * s)
    rng = np.random.default_rng(3)
    for idx in rng.integers(0, bits.size, 300):
        i, j = divmod(int(idx), 256)
        sv = scales[i // 128, j // 128]
        qv = rn32_exact(Fraction(float(synth.bf16_bits_to_f32(bits[i, j]))) / Fraction(float(sv)))
        assert oracle.quantize_element(synth.bf16_bits_to_f32(bits[i, j]), sv) == codes[i, j]
        assert oracle.e4m3_encode(qv) == codes[i, j]


def test_nonfinite_rejected():
    w = np.zeros((4, 128), dtype=np.uint16)
    w[2, 5] = 0x7F80  # +inf
    with pytest.raises(oracle.OracleError):
        oracle.quantize_weight_blockwise(w)
    w[2, 5] = 0x7FC1  # NaN
    with pytest.raises(oracle.OracleError):
        oracle.quantize_act_per_token_group(w)


def test_fused_equals_separate_projections():
    # reading Q14: q/k/v (and gate/up) boundaries are 128-aligned, so quantizing the fused
    # matrix equals quantizing the parts (8B qkv = q 4096 + k 1024 + v 1024 rows; scaled down).
    q, k, v = (synth.qwen3_weight(r, 256, seed=s) for r, s in ((512, 1), (128, 2), (128, 3)))
    cf, sf = oracle.quantize_weight_blockwise(np.concatenate([q, k, v]))
    parts = [oracle.quantize_weight_blockwise(t) for t in (q, k, v)]
    assert np.array_equal(cf, np.concatenate([p[0] for p in parts]))
    assert np.array_equal(sf, np.concatenate([p[1] for p in parts]))
