"""Pins for oracle O1 (decode) and O2 (encode) -- PAPER.md:54 (§2.1.1 E4M3).

Each check is against something other than the oracle itself: the paper/spec constants
(tests/golden/e4m3_constants.txt), torch's independent float8_e4m3fn codec (a library
routine), exact midpoints built from that library table, and the half-ULP bound.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "e4m3_constants.txt")


def torch_decode_table() -> np.ndarray:
    codes = torch.arange(256, dtype=torch.int32).to(torch.uint8)
    return codes.view(torch.float8_e4m3fn).to(torch.float64).numpy()


def torch_encode_sat(x: np.ndarray) -> np.ndarray:
    """torch's RNE cast, made saturating by clamping to +-448 first (SURVEY finding 9)."""
    t = torch.from_numpy(np.asarray(x, dtype=np.float32))
    t = torch.where(torch.isnan(t), t, t.clamp(-448.0, 448.0))
    return t.to(torch.float8_e4m3fn).view(torch.uint8).numpy()


def _golden_rows():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            kind, a, b, *_ = line.split()
            rows.append((kind, a, b))
    return rows


@pytest.mark.parametrize("kind,a,b", _golden_rows())
def test_golden_constants(kind, a, b):
    if kind == "decode":
        got = oracle.e4m3_decode(int(a, 16))
        if b == "nan":
            assert math.isnan(got)
        else:
            assert got == float(b) and math.copysign(1, got) == math.copysign(1, float(b))
    else:
        assert oracle.e4m3_encode(float(a)) == int(b, 16)


def test_decode_matches_library_all_256():
    ours = oracle.e4m3_decode_table()
    ref = torch_decode_table()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert nan.sum() == 2 and nan[0x7F] and nan[0xFF]
    assert np.array_equal(ours[~nan], ref[~nan])
    assert np.array_equal(np.signbit(ours[~nan]), np.signbit(ref[~nan]))  # -0 at 0x80
    finite = ref[~nan]
    assert len(finite) == 254 and len(np.unique(finite)) == 253  # +-0 share a value


def test_encode_roundtrip_all_finite_codes():
    # encode(decode(p)) == p for every non-NaN pattern (+-0 to themselves)
    table = torch_decode_table()
    for c in range(256):
        if c in (0x7F, 0xFF):
            continue
        assert oracle.e4m3_encode(table[c]) == c


def test_encode_nan():
    assert oracle.e4m3_encode(float("nan")) in (0x7F, 0xFF)


def _positive_values():
    t = torch_decode_table()
    return t[:0x7F]  # codes 0x00..0x7E ascending


def test_encode_all_midpoints_ties_to_even_and_neighbours():
    # x exactly halfway -> the pattern with even mantissa.  The 126 positive
    # midpoints are exact in fp32; one ulp either side must go to the nearer neighbour.
    v = _positive_values()
    for lo in range(126):
        mid = np.float32((v[lo] + v[lo + 1]) / 2)
        assert float(mid) == (v[lo] + v[lo + 1]) / 2
        even = lo if lo % 2 == 0 else lo + 1
        assert oracle.e4m3_encode(mid) == even
        assert oracle.e4m3_encode(-mid) == 0x80 | even
        below = np.nextafter(mid, np.float32(0))
        above = np.nextafter(mid, np.float32(np.inf))
        assert oracle.e4m3_encode(below) == lo
        assert oracle.e4m3_encode(above) == lo + 1


def _encode_many(x: np.ndarray) -> np.ndarray:
    return np.array([oracle.e4m3_encode(float(v)) for v in x], dtype=np.uint8)


def test_encode_matches_clamped_library_cast_strided_sweep():
    # A strided sweep over all 2^32 fp32 bit patterns (both signs, subnormals, huge) against
    # torch's independent RNE cast (clamped to +-448 => saturating).
    bits = np.arange(0, 1 << 32, 20011, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[~np.isnan(x)]
    assert np.array_equal(_encode_many(x), torch_encode_sat(x))


def test_encode_matches_library_near_every_midpoint():
    v = _positive_values()
    mids = ((v[:-1] + v[1:]) / 2).astype(np.float32)
    xs = []
    for m in mids:
        a = m
        for _ in range(4):
            a = np.nextafter(a, np.float32(0))
        for _ in range(9):
            xs.append(a)
            a = np.nextafter(a, np.float32(np.inf))
    xs = np.array(xs, dtype=np.float32)
    xs = np.concatenate([xs, -xs, v.astype(np.float32), np.float32([447.9, 448.0, 463.9, 464.0, 1e30])])
    assert np.array_equal(_encode_many(xs), torch_encode_sat(xs))


def test_half_ulp_error_bound():
    # for |x| in [2^-6, 448]: |decode(encode(x)) - x| <= 2^-4 * 2^floor(log2|x|)
    rng = np.random.default_rng(1)
    x = (2.0 ** rng.uniform(-6, math.log2(448), 20000)).astype(np.float32)
    x *= np.where(rng.integers(0, 2, x.size) == 1, -1, 1).astype(np.float32)
    table = torch_decode_table()
    codes = _encode_many(x)
    err = np.abs(table[codes] - x.astype(np.float64))
    bound = 2.0 ** -4 * 2.0 ** np.floor(np.log2(np.abs(x.astype(np.float64))))
    assert np.all(err <= bound)
    # idempotence
    assert np.array_equal(_encode_many(table[codes].astype(np.float32)), codes)
