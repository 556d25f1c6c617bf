"""Pins for the NEXT-2 producer oracle (readings N1, N2;
oracle/producers.py): Qwen3's RMSNorm and SiLU(gate)*up as the BF16 activations the
quantizer consumes, every binary32 step correctly rounded, sums exact.

Pins (none retypes the oracle's formula):
  * the rational -> binary32 / BF16 rounding against numpy's IEEE double -> float cast, an
    independent round()-based rounding, torch's float -> bfloat16 cast, and exact midpoints;
  * the exact sum of squares against Fraction brute force and math.fsum (correctly rounded);
  * the reciprocal square root against 50-digit decimal sqrt and closed forms;
  * RMSNorm closed forms (constant / one-hot rows, power-of-two scale invariance) and torch's
    float32 Qwen3RMSNorm (library ops) up to its own rounding noise;
  * the SiLU table against numpy binary64 (exp) rounded independently, torch's bfloat16 silu,
    and closed forms at 0, +-1, the smallest subnormal (a rounding tie broken by sigmoid > 1/2)
    and large |g|.
"""
import decimal
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import producers as P


def py_round_bf16(d: float) -> int:
    """Independent RNE of a binary64 to BF16 bits (normal range), via Python's round()."""
    if d == 0.0:
        return 0x8000 if math.copysign(1.0, d) < 0 else 0
    m, e = math.frexp(abs(d))          # |d| = m 2^e, m in [0.5, 1)
    r = round(m * 256.0)               # exact product; round() is half-to-even
    v = math.ldexp(r, e - 8)
    bits = int(np.float32(v).view(np.uint32)) >> 16
    return bits | (0x8000 if d < 0 else 0)


# ---------------------------------------------------------------- rounding helpers
def test_f64_to_bf16_roundtrip_and_midpoints():
    # the C helper: every BF16 value round-trips; every midpoint goes to the even neighbour
    for b in range(0x0080, 0x7F80, 7):
        v = float(synth.bf16_bits_to_f32(np.uint16(b)))
        assert oracle.f64_to_bf16(v) == b and oracle.f64_to_bf16(-v) == b | 0x8000
        nxt = float(synth.bf16_bits_to_f32(np.uint16(b + 1)))
        mid = (v + nxt) / 2
        assert oracle.f64_to_bf16(mid) == (b if b % 2 == 0 else b + 1)
        assert oracle.f64_to_bf16(math.nextafter(mid, 0)) == b
        assert oracle.f64_to_bf16(math.nextafter(mid, math.inf)) == b + 1
    assert oracle.f64_to_bf16(0.0) == 0 and oracle.f64_to_bf16(-0.0) == 0x8000


def test_rational_to_f32_matches_ieee_cast():
    # numpy's double -> float cast is IEEE round-to-nearest-even (one rounding): over the whole
    # range incl. subnormal outputs and overflow
    rng = np.random.default_rng(1)
    d = rng.standard_normal(4000) * np.exp2(rng.integers(-160, 130, 4000).astype(np.float64))
    with np.errstate(over="ignore"):
        want = d.astype(np.float32)
    for x, w in zip(d, want):
        got = P.rational_to_f32(Fraction(float(x)))
        assert got.view(np.uint32) == w.view(np.uint32), x
    # exact midpoints between neighbouring floats: ties to the even significand
    for b in rng.integers(0x00000001, 0x7F7FFFFF, 500, dtype=np.int64):
        lo = np.uint32(b).view(np.float32)
        hi = np.uint32(b + 1).view(np.float32)
        mid = (Fraction(float(lo)) + Fraction(float(hi))) / 2
        want = lo if b % 2 == 0 else hi
        assert P.rational_to_f32(mid) == want and P.rational_to_f32(-mid) == -want


def test_rational_to_bf16_matches_independent_rounding():
    rng = np.random.default_rng(2)
    d = rng.standard_normal(3000) * np.exp2(rng.integers(-120, 120, 3000).astype(np.float64))
    for d in d[np.abs(d) >= 2.0 ** -126]:  # py_round_bf16 covers the normal range
        assert P.rational_to_bf16_bits(Fraction(float(d))) == py_round_bf16(float(d))
    # BF16 subnormals: quantum 2^-133; the half-quantum rounds to 0 (even), 3 half-quanta to 2
    q = Fraction(1, 2 ** 133)
    assert P.rational_to_bf16_bits(q / 2) == 0 and P.rational_to_bf16_bits(-q / 2, True) == 0x8000
    assert P.rational_to_bf16_bits(q * 3 / 2) == 2
    assert P.rational_to_bf16_bits(q / 2 + Fraction(1, 2 ** 300)) == 1
    # overflow: the largest BF16 (0x7F7F) and the midpoint above it (rounds to infinity)
    mx = Fraction(float(synth.bf16_bits_to_f32(np.uint16(0x7F7F))))
    assert P.rational_to_bf16_bits(mx) == 0x7F7F
    assert P.rational_to_bf16_bits(mx * (1 + Fraction(1, 256))) == 0x7F80


def test_f32_to_bf16_matches_torch_cast():
    rng = np.random.default_rng(3)
    bits = rng.integers(0, 0xFF800000, 200000, dtype=np.uint64).astype(np.uint32)
    bits = bits[(bits & 0x7F800000) != 0x7F800000]  # finite
    f = bits.view(np.float32)
    want = torch.from_numpy(f.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(P.f32_to_bf16_bits(f), want)


# ---------------------------------------------------------------- sum of squares, rsqrt
def test_sum_squares_exact_against_fractions_and_fsum():
    for seed in range(6):
        row = synth.uniform_bits((1, 64), seed)[0]  # finite BF16 over the whole range
        row[::7] |= 0x8000
        exact = sum(Fraction(float(v)) ** 2 for v in synth.bf16_bits_to_f32(row))
        s = P.sum_squares_exact(row)
        assert s == exact
        sq = [float(v) ** 2 for v in synth.bf16_bits_to_f32(row).astype(np.float64)]  # exact in binary64
        assert float(s) == math.fsum(sq)  # both correctly rounded
    assert P.sum_squares_exact(np.zeros(8, np.uint16)) == 0
    assert P.sum_squares_exact(np.array([0x3F80, 0xBF80, 0x4000], np.uint16)) == 6  # 1 + 1 + 4


def _rsqrt_decimal(v: np.float32) -> np.float32:
    with decimal.localcontext() as ctx:
        ctx.prec = 50
        r = 1 / decimal.Decimal(float(v)).sqrt()
    return P.rational_to_f32(Fraction(r))  # 50 digits: far from any binary32 midpoint


def test_rsqrt_f32_correctly_rounded():
    rng = np.random.default_rng(4)
    vs = (rng.random(3000) * np.exp2(rng.integers(-140, 120, 3000).astype(np.float64))).astype(np.float32)
    for v in vs[vs > 0]:
        assert P.rsqrt_f32(v) == _rsqrt_decimal(v), v
    for v, r in [(4.0, 0.5), (1.0, 1.0), (0.25, 2.0), (2.0 ** -126, 2.0 ** 63), (2.0 ** 100, 2.0 ** -50)]:
        assert P.rsqrt_f32(np.float32(v)) == np.float32(r)
    assert P.rsqrt_f32(np.float32(np.inf)) == 0.0


# ---------------------------------------------------------------- RMSNorm
def test_rmsnorm_closed_forms():
    k = 4096
    g = synth.f32_to_bf16_bits((1.0 + np.arange(k) % 7 * 0.125).astype(np.float32))
    x = np.zeros((3, k), np.float32)
    x[0, :] = 4.0                      # constant power-of-two row (eps = 0): t = 1, y = gamma
    x[1, :] = -0.5                     # negative constant -> -gamma
    x[2, 123] = 2.0                    # one-hot: ms = 4/4096 = 2^-10, r = 32, t = 64, y = 64 gamma
    y = oracle.rmsnorm_bf16(synth.f32_to_bf16_bits(x), g, 0.0)
    assert np.array_equal(y[0], g)
    assert np.array_equal(y[1], g | np.uint16(0x8000))
    gf = synth.bf16_bits_to_f32(g)
    assert synth.bf16_bits_to_f32(y[2, 123]) == 64.0 * gf[123]
    assert np.count_nonzero(y[2] & 0x7FFF) == 1
    # power-of-two scale invariance (eps = 0): x and 4x normalise to the same BF16 values
    xr = synth.qwen3_activation(2, k, seed=3)
    x4 = synth.f32_to_bf16_bits(synth.bf16_bits_to_f32(xr) * 4.0)
    assert np.array_equal(oracle.rmsnorm_bf16(xr, g, 0.0), oracle.rmsnorm_bf16(x4, g, 0.0))


def test_rmsnorm_mean_of_squares_tie():
    # a row whose mean of squares is EXACTLY a binary32 midpoint (1 + 2^-24): 240 ones, four 2s,
    # four 2^-9 (K = 256) -> ms rounds to even (1.0), so r = 1, t = x; one tiny extra square
    # (2^-120) puts it above the midpoint -> ms = 1 + 2^-23, r = RN32(1/sqrt(1 + 2^-23)) < 1.
    k = 256
    row = np.zeros(k, np.float32)
    row[:240] = 1.0
    row[240:244] = 2.0
    row[244:248] = 2.0 ** -9
    g = synth.f32_to_bf16_bits(np.ones(k, np.float32))
    xb = synth.f32_to_bf16_bits(row[None, :])
    assert P.sum_squares_exact(xb[0]) / k == 1 + Fraction(1, 2 ** 24)
    y = oracle.rmsnorm_bf16(xb, g, 0.0)
    assert np.array_equal(y[0], xb[0])
    row2 = row.copy()
    row2[250] = 2.0 ** -60
    xb2 = synth.f32_to_bf16_bits(row2[None, :])
    ms = P.rational_to_f32(P.sum_squares_exact(xb2[0]) / k)
    assert ms == np.float32(1 + 2.0 ** -23)
    assert P.rsqrt_f32(ms) == np.float32(1 - 2.0 ** -24)
    y2 = oracle.rmsnorm_bf16(xb2, g, 0.0)
    # t = RN_BF16(RN32(2 (1 - 2^-24))) = 2: the BF16 outputs are unchanged by the rounding
    assert np.array_equal(y2[0, :248], xb2[0, :248])


@pytest.mark.parametrize("m,k,eps", [(6, 4096, 1e-6), (4, 2048, 1e-5), (3, 768, 1e-6)])
def test_rmsnorm_matches_torch_float32_qwen3(m, k, eps):
    # Qwen3RMSNorm as torch computes it on the CPU in float32 (library reduction order and
    # rsqrt): our definition differs only where torch's float32 rounding noise crosses a BF16
    # rounding boundary -- a vanishing fraction of elements
    x = synth.qwen3_activation(m, k, seed=k)
    g = synth.f32_to_bf16_bits((1.0 + 0.1 * np.random.default_rng(k).standard_normal(k)).astype(np.float32))
    y = oracle.rmsnorm_bf16(x, g, eps)
    xt = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).float()
    gt = torch.from_numpy(g.view(np.int16)).view(torch.bfloat16)
    var = xt.pow(2).mean(-1, keepdim=True)
    ref = gt * (xt * torch.rsqrt(var + eps)).to(torch.bfloat16)
    want = ref.view(torch.int16).numpy().view(np.uint16)
    assert np.count_nonzero(y != want) <= max(2, y.size // 2000)


# ---------------------------------------------------------------- SiLU
def test_silu_table_against_binary64_and_closed_forms():
    tab = oracle.silu_bf16_table()
    bits = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    finite = (bits & 0x7F80) != 0x7F80
    g = synth.bf16_bits_to_f32(bits).astype(np.float64)
    with np.errstate(over="ignore"):
        s64 = g / (1.0 + np.exp(-g))  # numpy binary64: ~1e-16 relative
    s64[np.isnan(s64)] = -0.0  # g -> -inf in exp: silu -> -0
    idx = np.nonzero(finite)[0]
    want = np.array([py_round_bf16(float(v)) if abs(v) >= 2.0 ** -126 or v == 0 else -1 for v in s64[idx]])
    normal = want >= 0
    assert np.array_equal(tab[idx][normal], want[normal].astype(np.uint16))
    assert np.all(tab[~finite] == 0x7FC0)
    # closed forms
    assert tab[0x0000] == 0x0000 and tab[0x8000] == 0x8000
    assert tab[0x3F80] == py_round_bf16(1.0 / (1.0 + math.exp(-1.0)))          # 0.7310585... -> 0x3F3B
    assert tab[0xBF80] == py_round_bf16(-math.exp(-1.0) / (1.0 + math.exp(-1.0)))
    assert tab[0x0001] == 0x0001   # g = 2^-133: g/2 is the 0 | 2^-133 midpoint, sigmoid > 1/2 rounds up
    assert tab[0x8001] == 0x8000   # g = -2^-133: |silu| < 2^-134 -> -0
    assert tab[0x4396] == 0x4396   # g = 300: silu = g (1 - 1e-130) -> g
    assert tab[0xC396] == 0x8000   # g = -300 -> -0


def test_silu_table_against_torch_bf16_silu():
    # torch evaluates silu of a bfloat16 tensor in float32 and rounds once: it can differ
    # from the correctly rounded value only within float32 noise of a BF16 midpoint
    # (|g| < 2^-120 is left out: there silu(g) ~ g/2 lands in the BF16 subnormal range, where
    # g/2 is an exact rounding tie that the real sigmoid > 1/2 breaks upwards, while torch's
    # binary32 sigmoid rounds to exactly 0.5 and the tie goes to even)
    bits = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    bits = bits[((bits & 0x7F80) != 0x7F80) & ((bits & 0x7F80) >= (7 << 7))]
    t = torch.nn.functional.silu(torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16))
    got = oracle.silu_bf16_table()[bits]
    assert np.count_nonzero(t.view(torch.int16).numpy().view(np.uint16) != got) <= 32


def test_silu_mul_closed_forms_and_composition():
    gu = synth.qwen3_activation(3, 1024, seed=9)
    y = oracle.silu_mul_bf16(gu)
    s = oracle.silu_bf16_table()[gu[:, :512]]
    ones = np.concatenate([gu[:, :512], np.full((3, 512), 0x3F80, np.uint16)], axis=1)
    assert np.array_equal(oracle.silu_mul_bf16(ones), s)                      # u = 1 -> y = s
    twos = np.concatenate([gu[:, :512], np.full((3, 512), 0x4000, np.uint16)], axis=1)
    assert np.array_equal(synth.bf16_bits_to_f32(oracle.silu_mul_bf16(twos)),
                          2 * synth.bf16_bits_to_f32(s))                      # u = 2 -> 2 s (exact)
    sf = synth.bf16_bits_to_f32(s).astype(np.float64)
    uf = synth.bf16_bits_to_f32(gu[:, 512:]).astype(np.float64)
    want = np.array([[py_round_bf16(float(v)) for v in row] for row in sf * uf], dtype=np.uint16)
    assert np.array_equal(y, want)  # s * u is exact in binary64: one rounding


def test_producer_quantize_composition():
    # the fused definitions are exactly "producer in BF16, then O3-O6"
    x = synth.qwen3_activation(5, 2048, seed=1)
    g = synth.f32_to_bf16_bits(np.ones(2048, np.float32))
    y, codes, scales = oracle.rmsnorm_quantize(x, g, 1e-6)
    c2, s2 = oracle.quantize_act_per_token_group(y)
    assert np.array_equal(codes, c2) and np.array_equal(scales, s2)
    gu = synth.qwen3_activation(4, 1024, seed=2)
    y, codes, scales = oracle.silu_mul_quantize(gu)
    c2, s2 = oracle.quantize_act_per_token_group(y)
    assert np.array_equal(codes, c2) and np.array_equal(scales, s2)
