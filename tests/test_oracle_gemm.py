"""Pins for oracle O7 (fp64 GEMM reference) and O8 (grouped GEMM).

SPEC.md:135-143 (qgemm_w8a8), north_star (rel. Frobenius <= 1e-3 vs the fp64 product of
the dequantized operands), SURVEY §8(c) O7/O8.  Pins: numpy's fp64 matmul of operands
decoded by torch's float8 table (an independent library routine, so a transposed
operand, a wrong scale index or a dropped term fails), the exact scale-probe closed form,
the SPEC's identity and 1x1 examples, and grouped == per-group dense.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

TABLE = torch.arange(256, dtype=torch.int32).to(torch.uint8).view(torch.float8_e4m3fn).to(torch.float64).numpy()


def dequant_act(codes, scales_logical):
    return TABLE[codes] * np.repeat(scales_logical.astype(np.float64), 128, axis=1)


def dequant_w(codes, scales):
    n, k = codes.shape
    s = np.repeat(np.repeat(scales.astype(np.float64), 128, 0), 128, 1)[:n, :k]
    return TABLE[codes] * s


@pytest.mark.parametrize("m,n,k,seed", [(4, 256, 256, 0), (37, 200, 384, 1), (128, 384, 128, 2), (1, 8, 256, 3)])
def test_gemm_matches_numpy_fp64(m, n, k, seed):
    a, sa = oracle.quantize_act_per_token_group(synth.qwen3_activation(m, k, seed))
    b, sb = oracle.quantize_weight_blockwise(synth.qwen3_weight(n, k, seed))
    y = oracle.gemm_rows(a, sa, b, sb)
    ref = dequant_act(a, sa) @ dequant_w(b, sb).T
    assert y.shape == (m, n)
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-300 + 1e-12 * np.abs(ref).max())
    rows = np.array([m - 1, 0], dtype=np.int64)
    np.testing.assert_array_equal(oracle.gemm_rows(a, sa, b, sb, rows), y[rows])


def test_gemm_scale_probe_exact():
    # every group/block is the constant +-448*2^e: codes 0x7E/0xFE, scales exactly 2^e, each
    # 128-deep partial is +-128*448^2 = +-49*2^19*... exactly, so Y has a closed form.
    m, n, k = 8, 256, 512
    rng = np.random.default_rng(0)
    ea = rng.integers(-3, 4, size=(m, k // 128))
    ew = rng.integers(-3, 4, size=(n // 128, k // 128))
    sgn_a = rng.choice([-1, 1], size=(m, k // 128))
    sgn_w = rng.choice([-1, 1], size=(n // 128, k // 128))
    xa = np.repeat(sgn_a * 448.0 * np.exp2(ea), 128, axis=1).astype(np.float32)
    xw = np.repeat(np.repeat(sgn_w * 448.0 * np.exp2(ew), 128, 0), 128, 1).astype(np.float32)
    a, sa = oracle.quantize_act_per_token_group(synth.f32_to_bf16_bits(xa))
    b, sb = oracle.quantize_weight_blockwise(synth.f32_to_bf16_bits(xw))
    assert np.array_equal(sa, np.exp2(ea).astype(np.float32))
    assert np.array_equal(sb, np.exp2(ew).astype(np.float32))
    y = oracle.gemm_rows(a, sa, b, sb)
    want = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            want[i, j] = sum(int(sgn_a[i, kb] * sgn_w[j // 128, kb]) * 128 * 448.0 * 448.0 *
                             2.0 ** int(ea[i, kb] + ew[j // 128, kb]) for kb in range(k // 128))
    assert np.array_equal(y, want)


def test_gemm_identity_and_1x1_examples():
    # SPEC.md:141 identity x identity; SPEC.md:143 1x1: A=[3], W=[[2]] -> deq(3)*deq(2)
    eye = synth.f32_to_bf16_bits(np.eye(128, dtype=np.float32))
    a, sa = oracle.quantize_act_per_token_group(eye)
    b, sb = oracle.quantize_weight_blockwise(eye)
    y = oracle.gemm_rows(a, sa, b, sb)
    d = (448.0 * float(sa[0, 0])) * (448.0 * float(sb[0, 0]))
    assert np.array_equal(y, np.eye(128) * d)
    xa = np.zeros((1, 128), np.float32); xa[0, 0] = 3.0
    xw = np.zeros((1, 128), np.float32); xw[0, 0] = 2.0
    a, sa = oracle.quantize_act_per_token_group(synth.f32_to_bf16_bits(xa))
    b, sb = oracle.quantize_weight_blockwise(synth.f32_to_bf16_bits(xw))
    y = oracle.gemm_rows(a, sa, b, sb)
    assert y[0, 0] == (448.0 * float(sa[0, 0])) * (448.0 * float(sb[0, 0]))
    assert abs(y[0, 0] - 6.0) <= 6.0 * 2.0 ** -22


def test_grouped_equals_per_group_dense():
    G, n, k = 5, 256, 256
    sizes = np.array([3, 0, 130, 1, 20])
    off = synth.offsets_from_sizes(sizes)
    m = int(off[-1])
    a, sa = oracle.quantize_act_per_token_group(synth.qwen3_activation(m, k, 4))
    bs = [oracle.quantize_weight_blockwise(synth.qwen3_weight(n, k, 10 + g)) for g in range(G)]
    b = np.stack([t[0] for t in bs]); sb = np.stack([t[1] for t in bs])
    y = oracle.gemm_grouped_rows(a, sa, b, sb, off)
    for g in range(G):
        r0, r1 = off[g], off[g + 1]
        ref = dequant_act(a[r0:r1], sa[r0:r1]) @ dequant_w(b[g], sb[g]).T
        np.testing.assert_allclose(y[r0:r1], ref, rtol=1e-12, atol=1e-12 * (np.abs(ref).max() if ref.size else 1))


def test_shape_mismatch_rejected():
    a = np.zeros((2, 256), np.uint8); sa = np.ones((2, 2), np.float32)
    b = np.zeros((3, 128), np.uint8); sb = np.ones((1, 1), np.float32)
    with pytest.raises(oracle.OracleError):
        oracle.gemm_rows(a, sa, b, sb)
