"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no amax, no scale, no E4M3 encode, no
GEMM): only input generators, which is the one thing ``oracle/`` and the product path
may share (DESIGN.md §4 "input recipe").  Everything is produced on the HOST from a
seeded ``torch.Generator`` / ``numpy`` RNG, as BF16 bit patterns (numpy ``uint16``);
callers copy the same bytes to the device.

Shapes follow SURVEY.md Appendix C (Qwen3-8B, Qwen3-30B-A3B) and BASELINE.json.
"""
from __future__ import annotations

import math

import numpy as np
import torch

# nn.Linear weight shapes [N = out, K = in]
QWEN3_8B_LINEARS = {
    "qkv": (6144, 4096),
    "o": (4096, 4096),
    "gate_up": (24576, 4096),
    "down": (4096, 12288),
}
QWEN3_8B_LAYERS = 36
QWEN3_30B_ATTN = {"qkv": (5120, 2048), "o": (2048, 4096)}
QWEN3_30B_EXPERTS = {"gate_up": (128, 1536, 2048), "down": (128, 2048, 768)}
QWEN3_30B_LAYERS = 48
QWEN3_30B_NUM_EXPERTS = 128
QWEN3_30B_TOPK = 8


def f32_to_bf16_bits(x: torch.Tensor | np.ndarray) -> np.ndarray:
    """float32 -> BF16 (torch's round-to-nearest-even cast) -> uint16 bit patterns."""
    t = torch.as_tensor(x, dtype=torch.float32)
    return t.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact widening of BF16 bit patterns to float32 (for building test inputs)."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def qwen3_weight(n: int, k: int, seed: int = 0, std: float = 0.02) -> np.ndarray:
    """W ~ N(0, std^2) with a per-row LogNormal(0, 0.5) gain so block amax varies
    (SURVEY.md §8(d) C2).  Returns BF16 bits [n, k]."""
    g = _gen(seed)
    w = torch.randn((n, k), generator=g, dtype=torch.float32) * std
    gain = torch.exp(torch.randn((n, 1), generator=g, dtype=torch.float32) * 0.5)
    return f32_to_bf16_bits(w * gain)


def qwen3_activation(m: int, k: int, seed: int = 0, outlier_frac: float = 0.005,
                     outlier_gain: float = 50.0) -> np.ndarray:
    """X ~ N(0, 1) with a fraction of outlier channels scaled x50 (LLM massive
    activations).  Returns BF16 bits [m, k]."""
    g = _gen(seed + 1_000_003)
    x = torch.randn((m, k), generator=g, dtype=torch.float32)
    n_out = max(1, int(round(outlier_frac * k))) if k else 0
    if n_out:
        ch = torch.randperm(k, generator=g)[:n_out]
        x[:, ch] *= outlier_gain
    return f32_to_bf16_bits(x)


def uniform_bits(shape, seed: int = 0, lo: int = 0, hi: int = 0x7F80) -> np.ndarray:
    """Random finite BF16 bit patterns with random sign (covers subnormals, tiny and huge
    magnitudes: the whole finite BF16 range).  Bits in [lo, hi) before the sign."""
    rng = np.random.default_rng(seed)
    mag = rng.integers(lo, hi, size=shape, dtype=np.uint32).astype(np.uint16)
    sign = (rng.integers(0, 2, size=shape, dtype=np.uint32).astype(np.uint16) << 15)
    return mag | sign


def block_probe_bits(n: int, k: int, seed: int = 0, emin: int = -6, emax: int = 6,
                     rows_per: int = 128, cols_per: int = 128) -> tuple[np.ndarray, np.ndarray]:
    """Block-probe matrix: block (i, j) (rows_per x cols_per) is filled with
    +-448 * 2^e_ij, e_ij distinct-ish small integers, random signs.  Every block's amax is
    448 * 2^e_ij, so its scale is exactly 2^e_ij and every code is 0x7E / 0xFE: the
    scale grid itself reveals which block was read.  Returns (bits [n,k], e [nb, kb])."""
    rng = np.random.default_rng(seed)
    nb, kb = -(-n // rows_per), -(-k // cols_per)
    e = rng.integers(emin, emax + 1, size=(nb, kb))
    vals = np.repeat(np.repeat(448.0 * np.exp2(e.astype(np.float64)), rows_per, 0), cols_per, 1)[:n, :k]
    sign = np.where(rng.integers(0, 2, size=(n, k)) == 1, -1.0, 1.0)
    return f32_to_bf16_bits((vals * sign).astype(np.float32)), e


# ----------------------------------------------------------------- exhaustive element map
# All 32,639 positive finite BF16 amax values A (bits 0x0001..0x7F7F) paired with every
# BF16 x in {0} U (0, A] (bits 0..A): 532,701,119 pairs (SURVEY.md §0 finding 2).
AMAX_BITS_MIN, AMAX_BITS_MAX = 0x0001, 0x7F7F


def exhaustive_pairs_count() -> int:
    a = np.arange(AMAX_BITS_MIN, AMAX_BITS_MAX + 1, dtype=np.int64)
    return int((a + 1).sum())


def _exhaustive_plan(unit: int) -> tuple[np.ndarray, np.ndarray]:
    """Split each amax A's x-range [0, A] into units of (unit - 1) values; each unit is
    one block (weights, unit = 16384) or one row (activations, unit = 128) holding A at
    position 0 followed by its slice of x bits.  Returns (amax_bits, start_bits) per unit."""
    a = np.arange(AMAX_BITS_MIN, AMAX_BITS_MAX + 1, dtype=np.int64)
    per = unit - 1
    nunits = (a + 1 + per - 1) // per
    amax = np.repeat(a, nunits)
    first = np.repeat(np.cumsum(nunits) - nunits, nunits)
    start = (np.arange(amax.size) - first) * per
    return amax, start


def _exhaustive_fill(amax: np.ndarray, start: np.ndarray, unit: int, negate: bool) -> np.ndarray:
    pos = np.arange(unit - 1, dtype=np.int64)[None, :]
    x = start[:, None] + pos
    x = np.where(x <= amax[:, None], x, 0)  # pad the last unit with zeros (x = 0 is in the map)
    out = np.concatenate([amax[:, None], x], axis=1).astype(np.uint16)
    if negate:
        out |= np.uint16(0x8000)
    return out


def exhaustive_weight_num_blocks() -> int:
    return int(_exhaustive_plan(128 * 128)[0].size)


def exhaustive_weight_chunks(blocks_per_chunk: int = 4096, negate: bool = False):
    """Yield BF16 bit matrices [nblk*128, 128]: a column of 128x128 blocks, each holding
    one amax A (at element (0,0)) and a contiguous slice of the x in [0, A]."""
    amax, start = _exhaustive_plan(128 * 128)
    for b0 in range(0, amax.size, blocks_per_chunk):
        blk = _exhaustive_fill(amax[b0:b0 + blocks_per_chunk], start[b0:b0 + blocks_per_chunk],
                               128 * 128, negate)
        yield blk.reshape(-1, 128, 128).reshape(-1, 128)


def exhaustive_act_num_rows() -> int:
    return int(_exhaustive_plan(128)[0].size)


def exhaustive_act_chunks(rows_per_chunk: int = 1 << 18, k: int = 128 * 8, negate: bool = False):
    """Yield BF16 bit matrices [rows, k]: each 128-channel group holds one amax A at its
    first channel followed by a slice of the x in [0, A]."""
    amax, start = _exhaustive_plan(128)
    gpr = k // 128
    per_chunk = rows_per_chunk * gpr
    for u0 in range(0, amax.size, per_chunk):
        grp = _exhaustive_fill(amax[u0:u0 + per_chunk], start[u0:u0 + per_chunk], 128, negate)
        pad = (-grp.shape[0]) % gpr
        if pad:
            grp = np.concatenate([grp, np.zeros((pad, 128), dtype=np.uint16)], axis=0)
        yield grp.reshape(-1, k)


# ----------------------------------------------------------------- MoE routing (C4)
def moe_group_sizes(tokens: int, num_experts: int = QWEN3_30B_NUM_EXPERTS,
                    topk: int = QWEN3_30B_TOPK, seed: int = 0, skew: float = 0.0) -> np.ndarray:
    """Rows per expert for `tokens` tokens routed top-k over seeded N(0,1) logits.
    skew > 0 adds a Gumbel + Zipf(skew) prior (SURVEY.md §8(d) C4 'skewed')."""
    g = _gen(seed + 7_777)
    logits = torch.randn((tokens, num_experts), generator=g)
    if skew > 0:
        ranks = torch.randperm(num_experts, generator=g).to(torch.float32) + 1.0
        prior = -skew * torch.log(ranks)
        gumbel = -torch.log(-torch.log(torch.rand((tokens, num_experts), generator=g).clamp_min(1e-20)))
        logits = prior[None, :] + gumbel
    top = torch.topk(logits, topk, dim=1).indices.reshape(-1)
    return torch.bincount(top, minlength=num_experts).numpy().astype(np.int64)


def offsets_from_sizes(sizes: np.ndarray) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


__all__ = [name for name in dir() if not name.startswith("_") and name not in ("math", "np", "torch")]
