"""Full-size parity (SURVEY §8(c) O2 pin (iv) and O7 "large shapes"):

* the hardware E4M3 encode (`cvt.rn.satfinite.e4m3x2.f32`, step a3, through the quantizers'
  own helper) on ALL 2^32 fp32 bit patterns against the oracle's O2, bitwise;
* the prefill GEMM (C2: all four Qwen3-8B shapes at M = 8192) on EVERY output element: the
  kernel's F32 output against an fp64 matmul of the operands dequantized through the
  oracle-validated E4M3 table and the oracle's scales (the operands themselves come from the
  oracle quantizers), overall and per 128 x 128 output tile, plus BF16 = RNE(F32) bitwise at
  full size;
* the grouped expert GEMM (C4) at the real Qwen3-30B-A3B shapes, T = 8192 tokens routed top-8
  (65,536 rows), uniform and Zipf-skewed routing, fc2 [128][2048, 768] and fc1 [128][1536, 2048],
  every output element against the per-group fp64 product, and sampled rows against the CPU
  oracle itself.
The fp64 matmul is a library step on oracle-produced operands, not product code."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import act_scales_mn_from_logical, rel_frobenius

pytestmark = pytest.mark.gpu


def test_e4m3_encode_all_fp32_patterns():
    chunk = 1 << 28
    mism = 0
    for c in range((1 << 32) // chunk):
        base = c * chunk
        bits = torch.arange(base, base + chunk, dtype=torch.int64, device="cuda")
        bits = torch.where(bits >= 1 << 31, bits - (1 << 32), bits).to(torch.int32)
        x = bits.view(torch.float32)
        got = fp8q.e4m3_encode_f32(x).cpu().numpy()
        xh = (np.arange(base, base + chunk, dtype=np.uint64).astype(np.uint32)).view(np.float32)
        want = oracle.e4m3_encode_array(xh)
        nan = np.isnan(xh)
        # NaN input: any NaN code (S.1111.111); the quantizers reject NaN input anyway (Q8)
        assert np.all((got[nan] & 0x7F) == 0x7F), c
        bad = (got != want) & ~nan
        mism += int(bad.sum())
        assert mism == 0, (c, np.nonzero(bad)[0][:8] + base)
        del bits, x


def _dec_table():
    t = oracle.e4m3_decode_table()
    t = np.where(np.isnan(t), 0.0, t)  # NaN codes never occur in quantizer output
    return torch.from_numpy(t).cuda()


def _dequant_act(codes, sa, tab):
    a = tab[torch.from_numpy(codes).cuda().long()]
    s = torch.from_numpy(sa.astype(np.float64)).cuda().repeat_interleave(128, dim=1)
    return a * s


def _dequant_weight(codes, sb, tab):
    n, k = codes.shape
    b = tab[torch.from_numpy(codes).cuda().long()]
    s = torch.from_numpy(sb.astype(np.float64)).cuda().repeat_interleave(128, 0)[:n].repeat_interleave(128, 1)[:, :k]
    return b * s


def _tile_errors(y, ref, t=128):
    m, n = ref.shape
    d = (y.double() - ref)
    num = d.square()[: m // t * t, : n // t * t].reshape(m // t, t, n // t, t).sum(dim=(1, 3))
    den = ref.square()[: m // t * t, : n // t * t].reshape(m // t, t, n // t, t).sum(dim=(1, 3))
    return (num / den).sqrt()


@pytest.mark.parametrize("name", ["qkv", "o", "gate_up", "down"])
def test_gemm_prefill_full_output_fp64(name):
    n, k = synth.QWEN3_8B_LINEARS[name]
    m = 8192
    a, sa = oracle.quantize_act_per_token_group(synth.qwen3_activation(m, k, 3))
    b, sb = oracle.quantize_weight_blockwise(synth.qwen3_weight(n, k, 3))
    tab = _dec_table()
    ref = _dequant_act(a, sa, tab) @ _dequant_weight(b, sb, tab).T
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dsa = act_scales_mn_from_logical(sa, fp8q.act_scales_ld(m))
    dsb = torch.from_numpy(sb).cuda()
    y = fp8q.fp8_block_gemm(da, dsa, db, dsb, out_dtype=torch.float32)
    torch.cuda.synchronize()
    err = float(((y.double() - ref).norm() / ref.norm()).item())
    assert err <= 1e-3 and err <= 1e-5, err
    tiles = _tile_errors(y, ref)
    assert float(tiles.max()) <= 1e-5, (float(tiles.max()), torch.nonzero(tiles == tiles.max())[:4].tolist())
    # the production BF16 path at full size: RNE of the F32 result, bitwise
    yb = fp8q.fp8_block_gemm(da, dsa, db, dsb, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(yb.view(torch.int16), y.to(torch.bfloat16).view(torch.int16))


@pytest.mark.parametrize("expert,skew", [("down", 0.0), ("down", 1.2), ("gate_up", 0.0), ("gate_up", 1.2)])
def test_grouped_qwen3_30b_full_shape_t8192(expert, skew):
    E, n, k = synth.QWEN3_30B_EXPERTS[expert]
    sizes = synth.moe_group_sizes(8192, seed=1, skew=skew)
    off = synth.offsets_from_sizes(sizes)
    m = int(off[-1])
    assert m == 8192 * 8
    a, sa = oracle.quantize_act_per_token_group(synth.qwen3_activation(m, k, 11))
    wb = synth.qwen3_weight(E * n, k, 12)
    b, sb = oracle.quantize_weight_blockwise(wb)  # expert blocks never straddle experts (n % 128 == 0)
    b3 = b.reshape(E, n, k)
    sb3 = sb.reshape(E, n // 128, k // 128)
    da = torch.from_numpy(a).cuda()
    dsa = act_scales_mn_from_logical(sa, fp8q.act_scales_ld(m))
    y = fp8q.fp8_block_gemm_grouped(da, dsa, torch.from_numpy(b3).cuda(), torch.from_numpy(sb3).cuda(),
                                    torch.from_numpy(off).cuda(), out_dtype=torch.float32)
    yb = fp8q.fp8_block_gemm_grouped(da, dsa, torch.from_numpy(b3).cuda(), torch.from_numpy(sb3).cuda(),
                                     torch.from_numpy(off).cuda(), out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    tab = _dec_table()
    A = _dequant_act(a, sa, tab)
    num = den = 0.0
    worst = 0.0
    for g in range(E):
        r0, r1 = int(off[g]), int(off[g + 1])
        if r1 == r0:
            continue
        Bg = _dequant_weight(b3[g], sb3[g], tab)
        ref = A[r0:r1] @ Bg.T
        d = float((y[r0:r1].double() - ref).square().sum())
        r = float(ref.square().sum())
        num += d
        den += r
        worst = max(worst, (d / r) ** 0.5)
    err = (num / den) ** 0.5
    assert err <= 1e-5, err
    assert worst <= 1e-5, worst
    assert torch.equal(yb.view(torch.int16), y.to(torch.bfloat16).view(torch.int16))
    # sampled rows against the CPU oracle itself (first / last row of some experts + random)
    rows = np.unique(np.concatenate([off[1:-1][::16] - 1, off[:-1][::16], np.random.default_rng(3).integers(0, m, 16)]))
    rows = rows[(rows >= 0) & (rows < m)]
    ref_rows = oracle.gemm_grouped_rows(a, sa, b3, sb3, off, rows)
    assert rel_frobenius(y[torch.from_numpy(rows).cuda()].cpu().numpy(), ref_rows) <= 1e-5
