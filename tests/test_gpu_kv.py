"""GPU parity of the NEXT-3 FP8 KV cache (§2.3.1; readings K1-K4) against
the oracle: calibration amax and scale bit-exact, appended codes bit-exact, saturation counts
exact, slot mapping, and the inference-side protocol (reset -> calibrating forward -> frozen
scale for the rest of the step)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16, to_host_u8

pytestmark = pytest.mark.gpu
KV_COLS = 8 * 128  # Qwen3-8B: 8 KV heads x head_dim 128


def _dev_amax_scale(batches):
    amax = torch.zeros(1, dtype=torch.int32, device="cuda")
    for b in batches:
        fp8q.kv_amax_update(to_dev_bf16(b), amax)
    scale = fp8q.kv_scale_from_amax(amax)
    torch.cuda.synchronize()
    return int(amax.item()), scale


@pytest.mark.parametrize("rows,cols", [(1, KV_COLS), (37, KV_COLS), (8192, KV_COLS), (5, 200), (3, 12)])
def test_kv_calibration_matches_oracle(rows, cols):
    batches = [synth.qwen3_activation(rows, cols, s) for s in range(3)]
    amax_bits, scale = _dev_amax_scale(batches)
    want = oracle.kv_calibrate(batches)
    got_amax = np.uint32(amax_bits << 16).view(np.float32)
    assert got_amax == max(float(oracle.kv_amax(b)) for b in batches)
    assert scale.cpu().numpy().view(np.uint32)[0] == np.float32(want).view(np.uint32)


def test_kv_scale_zero_and_many():
    bits = np.array([0, 0x3F80, 0x0001, 0x7F7F, 0x0B80, 0x0B7F], np.int32)
    got = fp8q.kv_scale_from_amax(torch.from_numpy(bits).cuda()).cpu().numpy()
    for b, g in zip(bits, got):
        want = oracle.kv_scale(float(synth.bf16_bits_to_f32(np.uint16(b))))
        assert np.float32(g).view(np.uint32) == np.float32(want).view(np.uint32), hex(b)


@pytest.mark.parametrize("rows,cols,slotted", [(1, KV_COLS, False), (64, KV_COLS, True), (513, KV_COLS, True),
                                               (8192, KV_COLS, False), (7, 200, True), (4, 24, False),
                                               (3, 12, True)])
def test_kv_append_matches_oracle(rows, cols, slotted):
    calib = synth.qwen3_activation(rows, cols, 1)
    scale = oracle.kv_scale(oracle.kv_amax(calib))
    x = synth.f32_to_bf16_bits(synth.bf16_bits_to_f32(synth.qwen3_activation(rows, cols, 2)) * np.float32(2.5))
    num_slots = 2 * rows + 3
    slots = np.random.default_rng(rows).permutation(num_slots)[:rows].astype(np.int32) if slotted else None
    ref = np.full((num_slots, cols), 0xAA, np.uint8)
    sat_ref = oracle.kv_quantize_append(x, scale, ref, slots)
    cache = torch.full((num_slots, cols), 0xAA, dtype=torch.uint8, device="cuda")
    sat = torch.zeros(1, dtype=torch.int32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    fp8q.kv_quantize_append(to_dev_bf16(x), torch.tensor([scale], device="cuda"), cache,
                            torch.from_numpy(slots).cuda() if slotted else None, sat, flag)
    torch.cuda.synchronize()
    assert np.array_equal(to_host_u8(cache), ref)
    assert int(sat.item()) == sat_ref and sat_ref > 0
    assert int(flag.item()) == 0


@pytest.mark.parametrize("scale_bits", [0x3E300000, 0x07124925, 0x07124924, 0x00000123, 0x7C000000, 0x3F800000])
def test_kv_append_exhaustive_bf16(scale_bits):
    # every finite BF16 value (both signs) through the append kernel, for scales on both sides
    # of the Markstein fast-path threshold RN32(2^-104/448) = 0x07124925, a subnormal scale, a
    # huge scale and 1.0: codes and saturation count bit-exact against the oracle
    allb = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    allb = allb[(allb & 0x7FFF) < 0x7F80]
    pad = (-allb.size) % KV_COLS
    x = np.concatenate([allb, np.zeros(pad, np.uint16)]).reshape(-1, KV_COLS)
    s = np.uint32(scale_bits).view(np.float32)
    ref = np.zeros(x.shape, np.uint8)
    sat_ref = oracle.kv_quantize_append(x, s, ref)
    cache = torch.zeros(x.shape, dtype=torch.uint8, device="cuda")
    sat = torch.zeros(1, dtype=torch.int32, device="cuda")
    fp8q.kv_quantize_append(to_dev_bf16(x), torch.tensor([s], device="cuda"), cache, None, sat)
    torch.cuda.synchronize()
    got = to_host_u8(cache)
    bad = np.nonzero(got != ref)
    assert bad[0].size == 0, (hex(int(x[bad][0])), hex(int(got[bad][0])), hex(int(ref[bad][0])))
    assert int(sat.item()) == sat_ref


def test_kv_flags():
    x = synth.qwen3_activation(4, KV_COLS, 3)
    x[2, 5] = 0x7FC0  # NaN
    cache = torch.zeros((4, KV_COLS), dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    slots = torch.tensor([0, 1, 9, 3], dtype=torch.int32, device="cuda")  # 9 is out of range
    fp8q.kv_quantize_append(to_dev_bf16(x), torch.tensor([0.5], device="cuda"), cache, slots, None, flag)
    amax = torch.zeros(1, dtype=torch.int32, device="cuda")
    f2 = torch.zeros(1, dtype=torch.int32, device="cuda")
    fp8q.kv_amax_update(to_dev_bf16(x), amax, f2)
    torch.cuda.synchronize()
    assert int(flag.item()) == 3  # bit 0: NaN in x, bit 1: slot out of range
    assert int(f2.item()) == 1
    assert np.all(to_host_u8(cache)[2] == 0)  # the row of slot 9 went nowhere


def test_kv_inference_side_protocol():
    # step t: reset (zero amax) -> the first forward calibrates -> scale frozen for decode appends
    prefill = synth.qwen3_activation(256, KV_COLS, 11)
    decode = [synth.qwen3_activation(16, KV_COLS, 20 + i) for i in range(3)]
    amax = torch.zeros(1, dtype=torch.int32, device="cuda")
    cache = torch.zeros((256 + 48, KV_COLS), dtype=torch.uint8, device="cuda")
    sat = torch.zeros(1, dtype=torch.int32, device="cuda")
    fp8q.kv_amax_update(to_dev_bf16(prefill), amax)
    scale = fp8q.kv_scale_from_amax(amax)
    fp8q.kv_quantize_append(to_dev_bf16(prefill), scale, cache[:256], None, sat)
    for i, d in enumerate(decode):
        sl = torch.arange(256 + 16 * i, 256 + 16 * (i + 1), dtype=torch.int32, device="cuda")
        fp8q.kv_quantize_append(to_dev_bf16(d), scale, cache, sl, sat)
    torch.cuda.synchronize()
    s = oracle.kv_scale(oracle.kv_amax(prefill))
    ref = np.zeros((256 + 48, KV_COLS), np.uint8)
    n = oracle.kv_quantize_append(prefill, s, ref)
    for i, d in enumerate(decode):
        n += oracle.kv_quantize_append(d, s, ref, np.arange(256 + 16 * i, 256 + 16 * (i + 1), dtype=np.int32))
    assert np.array_equal(to_host_u8(cache), ref)
    assert int(sat.item()) == n
    # the calibration forward itself never saturates (its amax element encodes to +-448)
    c0 = np.zeros((256, KV_COLS), np.uint8)
    assert oracle.kv_quantize_append(prefill, s, c0) == 0
