"""Pins for the NEXT-3 FP8 KV-cache oracle (§2.3.1: per-step QKV scale
recalibration; SPEC.md:262-297 kvquant; readings K1-K4 in DESIGN.md §3).

Pins (none re-types the oracle's arithmetic):
  * an independent library implementation: numpy amax, numpy binary32 division, torch's
    float8_e4m3fn cast (RNE) of the clamped quotient, numpy saturation count;
  * closed forms: the calibration amax element encodes to 0x7E (0xFE), 10x amax saturates to
    0x7E and is counted, an all-zero calibration gives scale 1;
  * invariants: power-of-two equivariance (x 2^k -> scale 2^k, same codes), set monotonicity
    of trainer-side calibration (superset -> scale >=), inference-side = trainer-side on the
    same data, slot mapping = row permutation, and the half-ULP round-trip bound.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

# Qwen3-8B: 8 KV heads x head_dim 128 per token
KV_COLS = 8 * 128


def indep_quantize(bits: np.ndarray, s: np.float32):
    x = synth.bf16_bits_to_f32(bits)
    q = (x / np.float32(s)).astype(np.float32)
    sat = int(np.count_nonzero(np.abs(q) >= np.float32(464.0)))
    codes = torch.from_numpy(q).clamp(-448.0, 448.0).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    return codes, sat


@pytest.mark.parametrize("rows,seed", [(1, 0), (37, 1), (256, 2)])
def test_kv_matches_library_implementation(rows, seed):
    calib = synth.qwen3_activation(rows, KV_COLS, seed)
    amax = oracle.kv_amax(calib)
    assert amax == np.max(np.abs(synth.bf16_bits_to_f32(calib)))
    s = oracle.kv_scale(amax)
    assert s == np.float32(amax) / np.float32(448.0)
    # append a different batch, partly beyond the calibrated range (x3 -> saturates)
    new = synth.qwen3_activation(rows, KV_COLS, seed + 100)
    big = synth.f32_to_bf16_bits(synth.bf16_bits_to_f32(new) * np.float32(3.0))
    for x in (new, big):
        cache = np.zeros((rows, KV_COLS), np.uint8)
        sat = oracle.kv_quantize_append(x, s, cache)
        codes, sat_ref = indep_quantize(x, s)
        assert np.array_equal(cache, codes)
        assert sat == sat_ref
    assert sat > 0  # the x3 batch really exercised saturation


def test_kv_closed_forms():
    x = np.zeros((2, 256), np.float32)
    x[0, 17] = -3.0
    x[1, 200] = 1.5
    bits = synth.f32_to_bf16_bits(x)
    s = oracle.kv_scale(oracle.kv_amax(bits))
    assert s == np.float32(3.0) / np.float32(448.0)
    cache = np.zeros((2, 256), np.uint8)
    assert oracle.kv_quantize_append(bits, s, cache) == 0
    assert cache[0, 17] == 0xFE  # -amax -> -448
    assert cache[1, 0] == 0x00 and cache[0, 0] == 0x00
    # 10x the calibrated amax saturates to +-448 and is counted
    y = synth.f32_to_bf16_bits(np.array([[30.0, -30.0, 3.0, 0.0]], np.float32))
    c2 = np.zeros((1, 4), np.uint8)
    assert oracle.kv_quantize_append(y, s, c2) == 2
    assert list(c2[0]) == [0x7E, 0xFE, 0x7E, 0x00]
    # zero calibration -> scale 1 (SPEC.md:94,111 reading Q5)
    assert oracle.kv_scale(oracle.kv_amax(np.zeros((3, 128), np.uint16))) == np.float32(1.0)
    # -0 keeps its sign (Q6)
    c3 = np.zeros((1, 1), np.uint8)
    oracle.kv_quantize_append(np.array([[0x8000]], np.uint16), s, c3)
    assert c3[0, 0] == 0x80


def test_kv_saturation_threshold_is_464():
    # quotients just below / at 464 (the midpoint between 448 and 480) with s = 1
    q = np.array([[462.0, 464.0, 466.0, -464.0, 448.0, 456.0]], np.float32)
    bits = synth.f32_to_bf16_bits(q)  # all exactly representable in BF16
    assert np.array_equal(synth.bf16_bits_to_f32(bits), q)
    c = np.zeros((1, 6), np.uint8)
    assert oracle.kv_quantize_append(bits, np.float32(1.0), c) == 3  # 464, 466, -464
    assert list(c[0]) == [0x7E] * 3 + [0xFE, 0x7E, 0x7E]


def test_kv_power_of_two_equivariance():
    x = synth.qwen3_activation(16, KV_COLS, 5)
    s = oracle.kv_scale(oracle.kv_amax(x))
    c0 = np.zeros((16, KV_COLS), np.uint8)
    oracle.kv_quantize_append(x, s, c0)
    for k in (-3, 5):
        xk = synth.f32_to_bf16_bits(synth.bf16_bits_to_f32(x) * np.float32(2.0 ** k))
        sk = oracle.kv_scale(oracle.kv_amax(xk))
        assert sk == s * np.float32(2.0 ** k)
        ck = np.zeros_like(c0)
        oracle.kv_quantize_append(xk, sk, ck)
        assert np.array_equal(ck, c0)


def test_kv_calibration_monotone_and_sides_agree():
    batches = [synth.qwen3_activation(8, KV_COLS, 10 + i) for i in range(4)]
    full = oracle.kv_calibrate(batches)
    for i in range(4):
        assert oracle.kv_calibrate(batches[: i + 1]) <= full
        assert oracle.kv_calibrate([batches[i]]) <= full
    # inference side (one calibration forward) == trainer side on that same data
    assert oracle.kv_calibrate([batches[2]]) == oracle.kv_scale(oracle.kv_amax(batches[2]))


def test_kv_slot_mapping_is_row_permutation():
    x = synth.qwen3_activation(6, 256, 7)
    s = oracle.kv_scale(oracle.kv_amax(x))
    ident = np.zeros((6, 256), np.uint8)
    oracle.kv_quantize_append(x, s, ident)
    slots = np.array([9, 0, 4, 11, 2, 7], np.int32)
    cache = np.full((12, 256), 0xAA, np.uint8)
    oracle.kv_quantize_append(x, s, cache, slots)
    assert np.array_equal(cache[slots], ident)
    untouched = np.setdiff1d(np.arange(12), slots)
    assert np.all(cache[untouched] == 0xAA)


def test_kv_round_trip_bound():
    # non-saturated elements: |dec(code) s - x| <= (2^(floor(log2 r) - 4) + 2^-24 r) s, r = |x/s|
    # (r >= 2^-6; below: 2^-10 s + ...), the element map's half-ULP bound
    x = synth.qwen3_activation(32, KV_COLS, 8)
    s = oracle.kv_scale(oracle.kv_amax(x))
    cache = np.zeros((32, KV_COLS), np.uint8)
    oracle.kv_quantize_append(x, s, cache)
    dec = torch.from_numpy(cache).view(torch.float8_e4m3fn).double().numpy()
    xv = synth.bf16_bits_to_f32(x).astype(np.float64)
    r = np.abs(xv / float(s))
    half_ulp = np.where(r >= 2.0 ** -6, np.exp2(np.floor(np.log2(np.maximum(r, 2.0 ** -6))) - 4), 2.0 ** -10)
    assert np.all(np.abs(dec * float(s) - xv) <= (half_ulp + 2.0 ** -24 * r) * float(s) * (1 + 1e-12))
    assert math.isfinite(float(s))


def test_kv_rejects_nonfinite():
    with pytest.raises(oracle.OracleError):
        oracle.kv_amax(np.array([[0x3F80, 0x7F80]], np.uint16))
