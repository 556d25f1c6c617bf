"""GPU parity of the two quantizers against the oracle (bit-exact codes and scales).

PAPER.md:54-58 (Eq. (1), 128x128 weight blocks), PAPER.md:65,233 (dynamic 1x128
activation groups).  Bar (north_star): FP8 bytes and fp32 scales bit-exact.
All calls go through the C-ABI (libfp8q.so) via the thin binding.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import act_scales_logical, to_dev_bf16, to_host_f32, to_host_u8

pytestmark = pytest.mark.gpu


def _weight_case(bits):
    w = to_dev_bf16(bits)
    codes, scales = fp8q.quantize_weight_blockwise(w)
    torch.cuda.synchronize()
    oc, os_ = oracle.quantize_weight_blockwise(bits)
    return to_host_u8(codes), to_host_f32(scales), oc, os_


def _assert_weight_exact(bits):
    gc, gs, oc, os_ = _weight_case(bits)
    assert np.array_equal(gs.view(np.uint32), os_.view(np.uint32)), "scales differ"
    mism = np.count_nonzero(gc != oc)
    assert mism == 0, f"{mism} code mismatches"


@pytest.mark.parametrize("seed", range(5))
def test_weight_c1_seeds(seed):
    # configs[0]: single 256x256 BF16 weight, 2x2 blocks of 128
    _assert_weight_exact(synth.qwen3_weight(256, 256, seed))


@pytest.mark.parametrize("n,k", [(300, 200), (129, 136), (1, 8), (128, 128), (131, 392), (640, 1024),
                                 # k % 16 == 0: the bulk-staged path with ragged rows / columns
                                 (300, 208), (129, 144), (1, 16), (200, 400), (1000, 1040)])
def test_weight_ragged_shapes(n, k):
    _assert_weight_exact(synth.qwen3_weight(n, k, n * 7 + k))


@pytest.mark.parametrize("seed", range(3))
def test_weight_full_range_bits(seed):
    # random finite BF16 over the whole range (subnormal ... 3e38), random signs
    _assert_weight_exact(synth.uniform_bits((384, 512), seed))


def test_weight_structured_blocks():
    n, k = 256, 512
    x = np.zeros((n, k), np.float32)
    x[128:, 0:128] = 0.0                       # zero block
    x[0:128, 128:256] = 1e-38                  # subnormal-scale block (BF16 normal tiny)
    x[128:256, 256:384] = np.random.default_rng(0).normal(size=(128, 128)) * 1e-3
    x[130, 300] = 57.0                         # single outlier
    x[0:128, 384:512] = 2.0 ** -120            # amax below the 2^-104 fast-path guard
    bits = synth.f32_to_bf16_bits(x)
    bits[5, 5] = 0x8000                        # -0 inside a zero block
    bits[200, 0] = 0x8000
    bits[7, 130] = 0x0001                      # BF16 subnormal element
    bits[8, 131] = 0x8001
    _assert_weight_exact(bits)


@pytest.mark.parametrize("n,k", [(256, 256), (300, 200), (1024, 768)])
def test_weight_block_probe(n, k):
    bits, e = synth.block_probe_bits(n, k, seed=3)
    gc, gs, oc, os_ = _weight_case(bits)
    assert np.array_equal(gs, np.exp2(e).astype(np.float32))
    assert np.array_equal(gc, oc)


def test_weight_strided_input_and_outputs():
    bits = synth.qwen3_weight(256, 384, 9)
    big = np.zeros((256, 512), np.uint16)
    big[:, :384] = bits
    w = to_dev_bf16(big)[:, :384]
    codes = torch.full((256, 400), 0xAB, dtype=torch.uint8, device="cuda")[:, :384]
    scales = torch.full((2, 7), -1.0, dtype=torch.float32, device="cuda")[:, :3]
    fp8q.quantize_weight_blockwise(w, codes, scales)
    oc, os_ = oracle.quantize_weight_blockwise(bits)
    assert np.array_equal(to_host_u8(codes), oc)
    assert np.array_equal(to_host_f32(scales), os_)
    full = to_host_u8(codes.as_strided((256, 400), (400, 1)))
    assert np.all(full[:, 384:] == 0xAB)  # padding untouched


@pytest.mark.parametrize("name", ["qkv", "down"])
def test_weight_full_qwen3_8b_shapes(name):
    n, k = synth.QWEN3_8B_LINEARS[name]
    _assert_weight_exact(synth.qwen3_weight(n, k, seed=0))


def test_weight_moe_expert_stack():
    # 30B experts: [E][N][K] quantized as one [E*N, K] matrix (N % 128 == 0)
    e, n, k = 8, 1536, 2048
    _assert_weight_exact(synth.qwen3_weight(e * n, k, seed=1))


def test_nonfinite_flag():
    bits = synth.qwen3_weight(256, 256, 0)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    fp8q.quantize_weight_blockwise(to_dev_bf16(bits), nonfinite_flag=flag)
    assert int(flag.item()) == 0
    bits[3, 200] = 0x7F80  # +Inf
    fp8q.quantize_weight_blockwise(to_dev_bf16(bits), nonfinite_flag=flag)
    assert int(flag.item()) == 1
    flag.zero_()
    x = synth.qwen3_activation(4, 256, 0)
    x[2, 17] = 0xFFC0  # NaN
    fp8q.quantize_act_per_token_group(to_dev_bf16(x), nonfinite_flag=flag)
    assert int(flag.item()) == 1
    # every non-finite kind on both quantizers' production paths (NaN payloads, -Inf, a NaN
    # next to the block's finite amax), on shapes that take the wide / staged kernels
    for n, k in [(256, 256), (12288, 4096)]:
        for pos, val in [((5, 9), 0x7FC1), ((n - 1, k - 1), 0xFF80), ((130, 129), 0xFFFF)]:
            flag.zero_()
            w = synth.qwen3_weight(n, k, 1)
            w[pos] = val
            fp8q.quantize_weight_blockwise(to_dev_bf16(w), nonfinite_flag=flag)
            assert int(flag.item()) == 1, (n, k, pos, hex(val))
            flag.zero_()
            fp8q.quantize_act_per_token_group(to_dev_bf16(w), nonfinite_flag=flag)
            assert int(flag.item()) == 1, (n, k, pos, hex(val))
    flag.zero_()
    fp8q.quantize_weight_blockwise(to_dev_bf16(synth.qwen3_weight(4096, 4096, 1)), nonfinite_flag=flag)
    assert int(flag.item()) == 0


# ------------------------------------------------------------------------------ activations
def _assert_act_exact(bits, ld_pad=0):
    m, k = bits.shape
    x = to_dev_bf16(bits)
    ld = fp8q.act_scales_ld(m) + ld_pad
    scales = torch.full((k // 128, ld), -7.0, dtype=torch.float32, device="cuda")
    codes, scales = fp8q.quantize_act_per_token_group(x, scales=scales)
    torch.cuda.synchronize()
    oc, os_ = oracle.quantize_act_per_token_group(bits)
    gs = act_scales_logical(scales, m)
    assert np.array_equal(gs.view(np.uint32), os_.view(np.uint32)), "scales differ"
    mism = np.count_nonzero(to_host_u8(codes) != oc)
    assert mism == 0, f"{mism} code mismatches"
    assert np.all(to_host_f32(scales)[:, m:] == -7.0)  # MN-major padding untouched


@pytest.mark.parametrize("m,k,seed", [(4, 256, 0), (4, 256, 1), (37, 768, 2), (1, 4096, 3), (64, 12288, 4),
                                      (129, 2048, 5), (3, 128, 6), (5, 1152, 7)])
def test_act_shapes(m, k, seed):
    _assert_act_exact(synth.qwen3_activation(m, k, seed), ld_pad=4)


@pytest.mark.parametrize("seed", range(2))
def test_act_full_range_bits(seed):
    _assert_act_exact(synth.uniform_bits((96, 1024), seed + 10))


def test_act_prefill_full_size():
    # C2 qkv input: M = 8192 tokens x K = 4096
    _assert_act_exact(synth.qwen3_activation(8192, 4096, 0))


@pytest.mark.parametrize("m,k,kind", [(257, 2176, "uniform"), (300, 384, "zeros"), (1000, 128, "qwen"),
                                      (513, 12288, "qwen"), (263, 1024, "uniform")])
def test_act_staged_ragged_rows_and_groups(m, k, kind):
    # > 256 tokens: the TMA-staged kernel (one 3-D box of 8 token rows x 16 groups per ring stage);
    # token counts that are not a multiple of 8 (the last unit's rows past m are zero-filled and
    # skipped) and group counts that are not a multiple of 16 (zero-filled groups), with full-range
    # bit patterns and zero / negative-zero rows
    if kind == "uniform":
        bits = synth.uniform_bits((m, k), 31 + m)
    else:
        bits = synth.qwen3_activation(m, k, 41 + m)
    if kind == "zeros":
        bits[::7, :] = 0
        bits[3::7, :] = 0x8000
        bits[5, 5] = 0x0001
    _assert_act_exact(bits, ld_pad=4)


def test_act_zero_and_signed_zero_rows():
    bits = np.zeros((4, 256), np.uint16)
    bits[1, :] = 0x8000
    bits[2, 7] = 0x0001
    bits[3, 255] = 0x8001
    _assert_act_exact(bits)


def test_quantizers_deterministic():
    bits = synth.qwen3_weight(512, 512, 2)
    w = to_dev_bf16(bits)
    c1, s1 = fp8q.quantize_weight_blockwise(w)
    c2, s2 = fp8q.quantize_weight_blockwise(w)
    assert torch.equal(c1, c2) and torch.equal(s1, s2)


def test_weight_batched_equals_individual():
    # quantize_weight_blockwise_batched (one launch per <=16 tensors): bitwise what the
    # per-tensor calls produce, incl. a misaligned tensor (general kernel) and > 16 tensors.
    shapes = [(6144 // 8, 512), (256, 384), (300, 208), (128, 1024)] * 5
    items, refs = [], []
    for i, (n, k) in enumerate(shapes):
        bits = synth.qwen3_weight(n, k, seed=100 + i)
        if i == 2:
            big = np.zeros((n, k + 8), np.uint16)
            big[:, :k] = bits
            w = to_dev_bf16(big)[:, :k]          # ld_w = k + 8: not 32-byte aligned rows
        else:
            w = to_dev_bf16(bits)
        codes = torch.empty((n, k), dtype=torch.uint8, device="cuda")
        scales = torch.empty(((n + 127) // 128, (k + 127) // 128), dtype=torch.float32, device="cuda")
        items.append((w, codes, scales))
        refs.append(oracle.quantize_weight_blockwise(bits))
    before = fp8q.kernel_launches()
    fp8q.quantize_weight_blockwise_batched(items)
    torch.cuda.synchronize()
    assert fp8q.kernel_launches() - before == 3  # 19 wide tensors -> 2 launches, 1 general
    for (w, codes, scales), (oc, os_) in zip(items, refs):
        assert np.array_equal(to_host_u8(codes), oc)
        assert np.array_equal(to_host_f32(scales), os_)


_BULK_SCRIPT = r"""
import numpy as np, torch, oracle, synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16, to_host_u8, to_host_f32
shapes = [(300, 208), (129, 144), (1, 16), (200, 400), (1000, 1040), (128, 128), (640, 1024)]
for i, (n, k) in enumerate(shapes):
    bits = synth.qwen3_weight(n, k, 500 + i)
    c, s = fp8q.quantize_weight_blockwise(to_dev_bf16(bits))
    oc, os_ = oracle.quantize_weight_blockwise(bits)
    assert np.array_equal(to_host_f32(s).view(np.uint32), os_.view(np.uint32)), (n, k, "scales")
    assert np.array_equal(to_host_u8(c), oc), (n, k, "codes")
bits = synth.uniform_bits((384, 512), 7)
c, s = fp8q.quantize_weight_blockwise(to_dev_bf16(bits))
oc, os_ = oracle.quantize_weight_blockwise(bits)
assert np.array_equal(to_host_u8(c), oc) and np.array_equal(to_host_f32(s).view(np.uint32), os_.view(np.uint32))
# a batch spanning several tensors: one bulk launch, ranges crossing tensor boundaries
shapes = [(768, 512), (256, 384), (300, 208), (128, 1024)] * 5
items, refs = [], []
for i, (n, k) in enumerate(shapes):
    bits = synth.qwen3_weight(n, k, seed=900 + i)
    items.append((to_dev_bf16(bits), torch.empty((n, k), dtype=torch.uint8, device="cuda"),
                  torch.empty(((n + 127) // 128, (k + 127) // 128), dtype=torch.float32, device="cuda")))
    refs.append(oracle.quantize_weight_blockwise(bits))
fp8q.quantize_weight_blockwise_batched(items)
torch.cuda.synchronize()
for (w, c, s), (oc, os_) in zip(items, refs):
    assert np.array_equal(to_host_u8(c), oc) and np.array_equal(to_host_f32(s), os_)
print("bulk ok")
"""


@pytest.mark.parametrize("path", ["bulk", "wide"])
def test_weight_forced_path_ragged(path):
    # The library picks the bulk-staged (TMA ring) or the block-strided kernel by batch size;
    # force each on small ragged shapes (rows past n / columns past k, batches whose per-CTA
    # block ranges cross tensor boundaries) in a fresh process (the override is read once).
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FP8Q_WEIGHT_KERNEL=path, PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _BULK_SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "bulk ok" in r.stdout, r.stdout + r.stderr


# ------------------------------------------------------------------ batched activation launch
@pytest.mark.parametrize("shapes", [
    # a Qwen3-8B layer's four GEMM inputs (K = 4096 x 3, 12288) at a ragged token count
    [(300, 4096), (300, 4096), (300, 4096), (300, 12288)],
    # groups not a multiple of 16 (zero-filled tail items), one-row and empty tensors mixed in
    [(5, 384), (1, 128), (0, 256), (33, 2176), (130, 1024)],
    # more tensors than one launch takes (8): split over two launches
    [(17 + i, 128 * (i + 1)) for i in range(11)],
])
def test_act_batched_matches_oracle(shapes):
    items, ref = [], []
    for i, (m, k) in enumerate(shapes):
        bits = synth.qwen3_activation(m, k, seed=500 + i)
        x = to_dev_bf16(bits) if m else torch.empty((0, k), dtype=torch.bfloat16, device="cuda")
        codes = torch.full((m, k), 0xAB, dtype=torch.uint8, device="cuda")
        scales = torch.full((k // 128, fp8q.act_scales_ld(m)), -1.0, dtype=torch.float32, device="cuda")
        items.append((x, codes, scales))
        ref.append(oracle.quantize_act_per_token_group(bits) if m else None)
    before = fp8q.kernel_launches()
    fp8q.quantize_act_per_token_group_batched(items)
    torch.cuda.synchronize()
    # tensors of > 256 tokens share persistent staged launches (8 per launch); decode-sized ones
    # (<= 256 tokens) each take the register kernel (PDL-friendly: no shared memory)
    staged = len([s for s in shapes if s[0] > 256])
    small = len([s for s in shapes if 0 < s[0] <= 256])
    assert fp8q.kernel_launches() - before == small + (staged + 7) // 8
    for (m, k), (x, codes, scales), r in zip(shapes, items, ref):
        if not m:
            continue
        oc, os_ = r
        assert np.array_equal(to_host_u8(codes), oc), (m, k)
        assert np.array_equal(act_scales_logical(scales, m).view(np.uint32), os_.view(np.uint32)), (m, k)



_ACT_SCRIPT = r"""
import numpy as np, torch, oracle, synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import to_dev_bf16, to_host_u8, act_scales_logical
shapes = [(300, 4096), (257, 384), (1000, 2176), (513, 12288), (40, 1024), (1, 128)]
items, ref = [], []
for i, (m, k) in enumerate(shapes):
    bits = synth.qwen3_activation(m, k, seed=800 + i)
    items.append((to_dev_bf16(bits), torch.full((m, k), 0xAB, dtype=torch.uint8, device="cuda"),
                  torch.full((k // 128, fp8q.act_scales_ld(m)), -1.0, dtype=torch.float32, device="cuda")))
    ref.append(oracle.quantize_act_per_token_group(bits))
fp8q.quantize_act_per_token_group_batched(items)
torch.cuda.synchronize()
for (m, k), (x, codes, scales), (oc, os_) in zip(shapes, items, ref):
    assert np.array_equal(to_host_u8(codes), oc), (m, k)
    assert np.array_equal(act_scales_logical(scales, m).view(np.uint32), os_.view(np.uint32)), (m, k)
print("act ok")
"""


@pytest.mark.parametrize("env", [{"FP8Q_ACT_KERNEL": "wide"}, {"FP8Q_ACT_LOAD": "bulk"}])
def test_act_forced_path_ragged(env):
    # The dev switches pick another activation kernel (warp-persistent register kernel for
    # every size) or another load form (cp.async.bulk rows instead of TMA boxes); the bytes must
    # not change.  Fresh process: the switches are read once.
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _ACT_SCRIPT], cwd=root, env=dict(os.environ, PYTHONPATH=root, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "act ok" in r.stdout, r.stdout + r.stderr


def test_act_batched_equals_single_calls_full_size():
    # the bench step's inputs: [8192, 4096] x 3 + [8192, 12288] in one launch == four launches
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    items_b, items_s = [], []
    for k in (4096, 4096, 4096, 12288):
        x = torch.randn((8192, k), generator=g, device="cuda").to(torch.bfloat16)
        x[:, ::997] *= 50
        for lst in (items_b, items_s):
            lst.append((x, torch.empty((8192, k), dtype=torch.uint8, device="cuda"),
                        torch.empty((k // 128, 8192), dtype=torch.float32, device="cuda")))
    fp8q.quantize_act_per_token_group_batched(items_b)
    for x, c, s in items_s:
        fp8q.quantize_act_per_token_group(x, c, s)
    torch.cuda.synchronize()
    for (_, cb, sb), (_, cs, ss) in zip(items_b, items_s):
        assert torch.equal(cb, cs)
        assert torch.equal(sb.view(torch.int32), ss.view(torch.int32))
    # and a sampled slice of the batch against the oracle (rows spread over the whole range)
    x, c, s = items_b[3]
    rows = torch.arange(0, 8192, 401)
    bits = x[rows].view(torch.int16).cpu().numpy().view(np.uint16)
    oc, os_ = oracle.quantize_act_per_token_group(bits)
    assert np.array_equal(to_host_u8(c[rows]), oc)
    assert np.array_equal(to_host_f32(s[:, rows]).T.view(np.uint32), os_.view(np.uint32))
