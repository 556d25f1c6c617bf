"""Oracle for the NEXT-2 producers: the BF16 activations the rollout
forward feeds to the quantized linear layers ("activation quantization is
performed dynamically" on the layer inputs) -- Qwen3's RMSNorm (input of q/k/v and gate/up)
and SiLU(gate) * up (input of down_proj).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain Python integers / fractions /
decimal and numpy IEEE binary32 element operations; no code shared with the product.

Definitions (DESIGN.md §3 readings N1, N2): Hugging Face's Qwen3 modules evaluate both
producers in binary32 and round to BF16 twice (Qwen3RMSNorm: `x * rsqrt(var + eps)` in fp32,
`.to(bf16)`, then `weight * (.)` in BF16; Qwen3MLP: `act_fn(gate_proj(x)) * up_proj(x)` on
BF16 tensors).  Written out with every binary32 operation correctly rounded and every value
the paper's pipeline rounds to BF16 rounded once, to nearest even:

  RMSNorm   ms  = RN32( (sum_i x_i^2) / K )           the sum of squares EXACT (real)
            r   = RN32( 1 / sqrt( RN32(ms + eps) ) )   correctly rounded reciprocal sqrt
            t_j = RN_BF16( RN32(x_j * r) )
            y_j = RN_BF16( RN32(gamma_j * t_j) )
  SiLU-mul  s_j = RN_BF16( g_j / (1 + e^(-g_j)) )     correctly rounded from the real value
            y_j = RN_BF16( RN32(s_j * u_j) )

Each step is a plain definition: an exact real value, rounded.  The oracle computes the
exact values with Python integers (sum of squares of BF16 values: integers times powers of
two), exact rational comparisons (the reciprocal square root) and 60-digit decimal arithmetic
with a checked error margin (exp), and the binary32 products with numpy float32 (IEEE).
"""
from __future__ import annotations

import decimal
import math
from fractions import Fraction

import numpy as np

_BF16_SUB_Q = -133  # exponent of the BF16 subnormal quantum (2^-133)
_F32_SUB_Q = -149


def _round_rational(num: int, den: int, mant_bits: int, emin_q: int, emax: int) -> tuple[int, int, bool]:
    """RNE of the positive rational num/den to a binary float with `mant_bits` significant
    bits, subnormal quantum 2^emin_q and largest finite binade 2^emax.  Returns (q, e, inf)
    with the result q * 2^e (q < 2^mant_bits or == 2^mant_bits after a carry)."""
    assert num > 0 and den > 0
    e = num.bit_length() - den.bit_length()  # 2^e <= num/den < 2^(e+2)
    if (num << max(0, -e)) < (den << max(0, e)):
        e -= 1
    # now 2^e <= num/den < 2^(e+1)
    qe = max(e - (mant_bits - 1), emin_q)
    n, d = (num << -qe, den) if qe <= 0 else (num, den << qe)
    q, r = divmod(n, d)
    if 2 * r > d or (2 * r == d and q & 1):
        q += 1
    inf = (q << qe) >= (1 << (emax + 1)) if qe >= 0 else q >= (1 << (emax + 1 - qe))
    return q, qe, inf


def rational_to_f32(x: Fraction) -> np.float32:
    """RN32 of an exact rational (round to nearest even, IEEE binary32: subnormals, overflow
    to infinity)."""
    if x == 0:
        return np.float32(0.0)
    q, e, inf = _round_rational(abs(x.numerator), x.denominator, 24, _F32_SUB_Q, 127)
    v = np.float32(np.inf) if inf else np.float32(math.ldexp(q, e))  # exact: q <= 2^24
    return -v if x < 0 else v


def rational_to_bf16_bits(x: Fraction, negative_zero: bool = False) -> int:
    """RN_BF16 of an exact rational, as BF16 bits (ties to even, overflow to infinity)."""
    if x == 0:
        return 0x8000 if negative_zero else 0
    q, e, inf = _round_rational(abs(x.numerator), x.denominator, 8, _BF16_SUB_Q, 127)
    if inf:
        bits = 0x7F80
    else:
        bits = int(np.float32(math.ldexp(q, e)).view(np.uint32)) >> 16  # exact: 8 bits
    return bits | (0x8000 if x < 0 else 0)


def f32_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """RN_BF16 of binary32 values (ties to even; NaN -> 0x7FC0), elementwise."""
    u = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(np.asarray(f, dtype=np.float32))
    r[nan] = 0x7FC0
    return r


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _bf16_int_parts(bits: np.ndarray):
    """|x| = m * 2^ex with integer m (BF16: 8 significant bits; subnormals m < 128)."""
    b = bits.astype(np.int64) & 0x7FFF
    E = b >> 7
    mant = b & 0x7F
    m = np.where(E == 0, mant, mant | 0x80)
    ex = np.where(E == 0, -133, E - 134)
    return m, ex, E


_SQ_SHIFT = 266  # x^2 = m^2 * 2^(2 ex) with 2 ex >= -266


def sum_squares_exact(row_bits: np.ndarray) -> Fraction:
    """sum_i x_i^2 of a BF16 row, exactly: every square is the integer m^2 times 2^(2 ex), so
    the sum is an integer (summed per exponent, then combined) times 2^-266."""
    m, ex, E = _bf16_int_parts(np.asarray(row_bits))
    if np.any(E == 0xFF):
        raise ValueError("non-finite input")
    live = m > 0
    pos = (2 * ex + _SQ_SHIFT)[live]
    cnt = np.bincount(pos, weights=(m[live] * m[live]).astype(np.float64))  # each bin < 2^53: exact
    total = 0
    for p in np.nonzero(cnt)[0]:
        total += int(cnt[p]) << int(p)
    return Fraction(total, 1 << _SQ_SHIFT)


def rsqrt_f32(v: np.float32) -> np.float32:
    """RN32(1 / sqrt(v)) for a positive finite binary32 v, correctly rounded: a binary64
    candidate checked (and moved) against the exact midpoint conditions mid^2 * v <> 1."""
    v = np.float32(v)
    if v == np.float32(np.inf):
        return np.float32(0.0)
    if v == 0:
        return np.float32(np.inf)
    vf = Fraction(float(v))
    c = np.float32(1.0 / math.sqrt(float(v)))
    for _ in range(4):
        a = Fraction(float(c))
        lo = Fraction(float(np.nextafter(c, np.float32(0.0))))
        hi = Fraction(float(np.nextafter(c, np.float32(np.inf))))
        mlo, mhi = (a + lo) / 2, (a + hi) / 2
        if mlo * mlo * vf > 1:          # 1/sqrt(v) < mlo: the lower neighbour is nearer
            c = np.nextafter(c, np.float32(0.0))
        elif mhi * mhi * vf < 1:        # 1/sqrt(v) > mhi
            c = np.nextafter(c, np.float32(np.inf))
        else:
            if mlo * mlo * vf == 1 or mhi * mhi * vf == 1:  # exact tie: to even
                nb = np.nextafter(c, np.float32(0.0 if mlo * mlo * vf == 1 else np.inf))
                if int(c.view(np.uint32)) & 1:
                    c = nb
            return c
    raise AssertionError("rsqrt candidate did not converge")


def rmsnorm_bf16(x_bits: np.ndarray, gamma_bits: np.ndarray, eps: float) -> np.ndarray:
    """N2 RMSNorm (module docstring) of BF16 rows [m, k] with BF16 gamma [k]; eps is taken as
    the binary32 value the C-ABI receives."""
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    m, k = x_bits.shape
    g = bf16_bits_to_f32(np.asarray(gamma_bits, dtype=np.uint16))
    eps32 = np.float32(eps)
    y = np.empty((m, k), dtype=np.uint16)
    for i in range(m):
        ms = rational_to_f32(sum_squares_exact(x_bits[i]) / k)
        r = rsqrt_f32(np.float32(ms + eps32))
        with np.errstate(over="ignore", under="ignore", invalid="ignore"):
            t = f32_to_bf16_bits(bf16_bits_to_f32(x_bits[i]) * r)
            y[i] = f32_to_bf16_bits(g * bf16_bits_to_f32(t))
    return y


# ---------------------------------------------------------------- SiLU
_SILU_TABLE = None


def _silu_bf16_of(bits: int) -> int:
    """RN_BF16(g / (1 + e^-g)) for one BF16 g, correctly rounded (60-digit decimal with an
    asserted margin to the nearest BF16 rounding boundary)."""
    E = (bits >> 7) & 0xFF
    neg = bool(bits & 0x8000)
    if E == 0xFF:
        return 0x7FC0  # non-finite input: NaN (the quantizer flags it)
    g = Fraction(float(np.uint32(bits << 16).view(np.float32)))
    if g == 0:
        return bits  # silu(+-0) = +-0
    if g > 200:  # e^-g < 1e-86: g (1 - e^-g + ...) is within 1e-86 of g, a BF16 value
        return bits
    if g < -200:  # |silu| < 200 e^-200 < 2^-134 (half the smallest BF16 subnormal)
        return 0x8000
    with decimal.localcontext() as ctx:
        ctx.prec = 60
        ctx.Emin = -999999
        gd = decimal.Decimal(g.numerator) / decimal.Decimal(g.denominator)  # exact: a dyadic
        s = gd / (1 + (-gd).exp())
        sf = Fraction(s)
    # the 60-digit value is within 1e-57 relative of the real one; its rounding is decided
    # unless it lies that close to a BF16 rounding boundary (asserted never to happen)
    out = rational_to_bf16_bits(sf, negative_zero=neg)
    margin = abs(sf) * Fraction(1, 10 ** 55)
    assert rational_to_bf16_bits(sf - margin, neg) == out == rational_to_bf16_bits(sf + margin, neg), bits
    return out


def silu_bf16_table() -> np.ndarray:
    """s(g) = RN_BF16(silu(g)) for all 65,536 BF16 bit patterns g (computed once per process)."""
    global _SILU_TABLE
    if _SILU_TABLE is None:
        _SILU_TABLE = np.array([_silu_bf16_of(b) for b in range(1 << 16)], dtype=np.uint16)
    return _SILU_TABLE


def silu_mul_bf16(gate_up_bits: np.ndarray) -> np.ndarray:
    """N2 SiLU-mul (module docstring) of gate_up = [gate | up] (each [m, I]) -> BF16 [m, I]."""
    gu = np.ascontiguousarray(gate_up_bits, dtype=np.uint16)
    m, k2 = gu.shape
    inter = k2 // 2
    s = silu_bf16_table()[gu[:, :inter]]
    with np.errstate(over="ignore", under="ignore", invalid="ignore"):
        return f32_to_bf16_bits(bf16_bits_to_f32(s) * bf16_bits_to_f32(gu[:, inter:]))
