"""GPU parity of the blockwise-scaled FP8 GEMM (dense and grouped) against the oracle.

Bar (north_star): relative Frobenius error <= 1e-3 against the fp64
product of the dequantized operands, on the kernel's F32 output (reading Q16).  Stronger
checks: the scale-probe GEMM is compared BITWISE with its closed form, BF16 output is
bitwise RNE of the F32 output, and repeated runs are bitwise identical.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2601_18150_b200 import fp8q
from tests.helpers import (act_scales_logical, act_scales_mn_from_logical, rel_frobenius,
                           to_dev_bf16)

pytestmark = pytest.mark.gpu
TOL = 1e-3  # north_star: rel. Frobenius <= 1e-3


def _operands(m, n, k, seed, kind="normal"):
    if kind == "normal":
        xb, wb = synth.qwen3_activation(m, k, seed), synth.qwen3_weight(n, k, seed)
    else:
        xb = synth.uniform_bits((m, k), seed, lo=0x3000, hi=0x4400)
        wb = synth.uniform_bits((n, k), seed + 1, lo=0x3000, hi=0x4400)
    a, sa = oracle.quantize_act_per_token_group(xb)
    b, sb = oracle.quantize_weight_blockwise(wb)
    return a, sa, b, sb


def _run(a, sa, b, sb, out_dtype=torch.float32):
    m = a.shape[0]
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda()
    dsa = act_scales_mn_from_logical(sa, fp8q.act_scales_ld(m))
    dsb = torch.from_numpy(sb).cuda()
    y = fp8q.fp8_block_gemm(da, dsa, db, dsb, out_dtype=out_dtype)
    torch.cuda.synchronize()
    return y


@pytest.mark.parametrize("m,n,k,seed", [
    (4, 256, 256, 0), (4, 256, 256, 1), (4, 256, 256, 2),  # configs[0] (C1)
    (1, 256, 128, 3), (37, 200, 384, 4), (128, 256, 512, 5), (129, 264, 256, 6),
    (300, 512, 640, 7), (256, 768, 1024, 8), (513, 1032, 256, 9),
])
def test_gemm_small_vs_oracle(m, n, k, seed):
    a, sa, b, sb = _operands(m, n, k, seed)
    y = _run(a, sa, b, sb).cpu().numpy()
    ref = oracle.gemm_rows(a, sa, b, sb)
    err = rel_frobenius(y, ref)
    assert err <= TOL, err
    assert err <= 1e-5  # fp32 promotion of exact partials: ~1e-7


def test_gemm_wide_dynamic_range():
    a, sa, b, sb = _operands(200, 512, 512, 11, kind="uniform")
    y = _run(a, sa, b, sb).cpu().numpy()
    assert rel_frobenius(y, oracle.gemm_rows(a, sa, b, sb)) <= 1e-5


@pytest.mark.parametrize("m", [160, 48, 5])
def test_gemm_scale_probe_bitwise(m):
    # every activation group / weight block is the constant +-448*2^e: codes 0x7E/0xFE,
    # scales exactly 2^e, partials exact, so D has an exact closed form.
    # m <= 128 runs the swap-AB decode kernel (gemm_skinny.cu), m = 160 the tile kernel.
    n, k = 512, 1024
    rng = np.random.default_rng(0)
    ea = rng.integers(-3, 4, size=(m, k // 128))
    ew = rng.integers(-3, 4, size=(n // 128, k // 128))
    sgn_a = rng.choice([-1, 1], size=(m, k // 128))
    sgn_w = rng.choice([-1, 1], size=(n // 128, k // 128))
    xa = np.repeat(sgn_a * 448.0 * np.exp2(ea), 128, axis=1).astype(np.float32)
    xw = np.repeat(np.repeat(sgn_w * 448.0 * np.exp2(ew), 128, 0), 128, 1).astype(np.float32)
    a, sa = oracle.quantize_act_per_token_group(synth.f32_to_bf16_bits(xa))
    b, sb = oracle.quantize_weight_blockwise(synth.f32_to_bf16_bits(xw))
    y = _run(a, sa, b, sb).cpu().numpy().astype(np.float64)
    coef = (sgn_a[:, None, :] * np.repeat(sgn_w, 128, axis=0)[None, :, :]) * \
        np.exp2(ea[:, None, :] + np.repeat(ew, 128, axis=0)[None, :, :])
    want = coef.sum(axis=2) * 128.0 * 448.0 * 448.0
    assert np.array_equal(y, want)


def test_gemm_bf16_is_rne_of_f32_and_deterministic():
    a, sa, b, sb = _operands(300, 768, 1024, 12)
    yf = _run(a, sa, b, sb, torch.float32)
    yb = _run(a, sa, b, sb, torch.bfloat16)
    assert torch.equal(yb.view(torch.int16), yf.to(torch.bfloat16).view(torch.int16))
    yf2 = _run(a, sa, b, sb, torch.float32)
    assert torch.equal(yf.view(torch.int32), yf2.view(torch.int32))


@pytest.mark.parametrize("m,n", [(1, 4096), (2, 4096), (8, 4096), (64, 4096), (192, 4096), (256, 4096),
                                 (96, 16384)])
def test_gemm_decode_shapes(m, n):
    # C3: decode-shaped GEMMs at Qwen3-8B o_proj width (K = N = 4096); (96, 16384) takes the
    # tile kernel (M > 32 with >= 64 column tiles), the other M <= 128 the swap-AB kernel
    a, sa, b, sb = _operands(m, n, 4096, 20 + m)
    y = _run(a, sa, b, sb).cpu().numpy()
    assert rel_frobenius(y, oracle.gemm_rows(a, sa, b, sb)) <= TOL


@pytest.mark.parametrize("name", ["qkv", "o", "gate_up", "down"])
def test_gemm_prefill_full_size_sampled(name):
    # C2 at full size: M = 8192, sampled rows against the oracle (incl. first/last tile rows)
    n, k = synth.QWEN3_8B_LINEARS[name]
    m = 8192
    a, sa, b, sb = _operands(m, n, k, 0)
    y = _run(a, sa, b, sb, torch.float32)
    rows = np.unique(np.concatenate([[0, 127, 128, m - 1], np.random.default_rng(1).integers(0, m, 12)]))
    ref = oracle.gemm_rows(a, sa, b, sb, rows)
    got = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert rel_frobenius(got, ref) <= TOL
    for i in range(len(rows)):
        assert rel_frobenius(got[i], ref[i]) <= 1e-4


def test_gemm_validation_errors():
    a = torch.zeros((4, 200), dtype=torch.uint8, device="cuda")  # k % 128 != 0
    sa = torch.ones((2, 4), dtype=torch.float32, device="cuda")
    b = torch.zeros((256, 200), dtype=torch.uint8, device="cuda")
    sb = torch.ones((2, 2), dtype=torch.float32, device="cuda")
    with pytest.raises(fp8q.Fp8qError, match="SHAPE"):
        fp8q.fp8_block_gemm(a, sa, b, sb)
    with pytest.raises(fp8q.Fp8qError):
        fp8q.fp8_block_gemm(a.cpu(), sa, b, sb)


# ------------------------------------------------------------------------------ grouped (C4)
def _grouped_case(sizes, n, k, seed):
    off = synth.offsets_from_sizes(np.asarray(sizes))
    m = int(off[-1])
    G = len(sizes)
    a, sa = oracle.quantize_act_per_token_group(synth.qwen3_activation(max(m, 1), k, seed)[:m])
    bq = [oracle.quantize_weight_blockwise(synth.qwen3_weight(n, k, seed * 1000 + g)) for g in range(G)]
    b = np.stack([t[0] for t in bq])
    sb = np.stack([t[1] for t in bq])
    da = torch.from_numpy(a).cuda()
    dsa = act_scales_mn_from_logical(sa, fp8q.act_scales_ld(m))
    y = fp8q.fp8_block_gemm_grouped(da, dsa, torch.from_numpy(b).cuda(), torch.from_numpy(sb).cuda(),
                                    torch.from_numpy(off).cuda(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    return a, sa, b, sb, off, y


@pytest.mark.parametrize("sizes,n,k", [
    ([3, 0, 130, 1, 20, 0, 256, 77], 256, 256),
    ([0, 0, 5], 512, 384),
    ([129, 1, 128, 255], 264, 128),
])
def test_grouped_vs_oracle(sizes, n, k):
    a, sa, b, sb, off, y = _grouped_case(sizes, n, k, 3)
    ref = oracle.gemm_grouped_rows(a, sa, b, sb, off)
    assert rel_frobenius(y.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("skew", [0.0, 1.2])
def test_grouped_qwen3_30b_fc1_sampled(skew):
    # C4: 128 experts, fc1 N = 1536, K = 2048, T = 1024 tokens routed top-8
    sizes = synth.moe_group_sizes(1024, seed=0, skew=skew)
    a, sa, b, sb, off, y = _grouped_case(sizes, 1536, 2048, 5)
    m = int(off[-1])
    rows = np.unique(np.concatenate([off[1:-1][::9] - 1, np.random.default_rng(2).integers(0, m, 24)]))
    rows = rows[(rows >= 0) & (rows < m)]
    ref = oracle.gemm_grouped_rows(a, sa, b, sb, off, rows)
    got = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert rel_frobenius(got, ref) <= TOL


def _run_unsplit(a, sa, b, sb):
    """fp8_block_gemm through the C-ABI with no workspace (never splits K), F32 output."""
    m, k = a.shape
    n = b.shape[0]
    lib = fp8q.load_library()
    da = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    dsa = act_scales_mn_from_logical(sa, fp8q.act_scales_ld(m))
    db = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    dsb = torch.from_numpy(np.ascontiguousarray(sb)).cuda()
    y = torch.empty((m, n), dtype=torch.float32, device="cuda")
    st = lib.fp8_block_gemm(da.data_ptr(), k, dsa.data_ptr(), dsa.stride(0), db.data_ptr(), k,
                            dsb.data_ptr(), dsb.shape[1], y.data_ptr(), n, 1, m, n, k, None, 0,
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert st == 0
    return y


def test_grouped_equals_dense_per_group_bitwise():
    # O8: grouped == per-group dense (unsplit), and the kernel is deterministic -> bitwise
    sizes = [70, 0, 200, 9]
    a, sa, b, sb, off, y = _grouped_case(sizes, 256, 384, 7)
    for g in range(len(sizes)):
        r0, r1 = int(off[g]), int(off[g + 1])
        if r1 == r0:
            continue
        yd = _run_unsplit(a[r0:r1], sa[r0:r1], b[g], sb[g])
        assert torch.equal(yd.view(torch.int32), y[r0:r1].contiguous().view(torch.int32))


@pytest.mark.parametrize("m,n,k", [(16, 4096, 4096), (1, 6144, 4096), (8, 4096, 12288)])
def test_gemm_splitk_decode(m, n, k):
    # small M: the binding passes a workspace, the kernel splits K; the last slice of each tile
    # sums the slices in slice order -> deterministic; the workspace is left zeroed (reusable)
    lib = fp8q.load_library()
    assert lib.fp8_block_gemm_workspace_size(m, n, k) > 0
    a, sa, b, sb = _operands(m, n, k, 31)
    y1 = _run(a, sa, b, sb)
    y2 = _run(a, sa, b, sb)
    assert torch.equal(y1.view(torch.int32), y2.view(torch.int32))
    ref = oracle.gemm_rows(a, sa, b, sb, np.arange(min(m, 16)))
    assert rel_frobenius(y1[:min(m, 16)].cpu().numpy(), ref) <= 1e-5
    # the same problem without a workspace runs unsplit: equal up to fp32 summation order
    da, db, dsb = (torch.from_numpy(t).cuda() for t in (a, b, sb))  # held until the kernel ran
    dsa = act_scales_mn_from_logical(sa, fp8q.act_scales_ld(m))
    yu = torch.empty((m, n), dtype=torch.float32, device="cuda")
    st = lib.fp8_block_gemm(da.data_ptr(), k, dsa.data_ptr(), dsa.stride(0), db.data_ptr(), k,
                            dsb.data_ptr(), sb.shape[1], yu.data_ptr(), n, 1,
                            m, n, k, None, 0, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert st == 0
    assert rel_frobenius(y1.cpu().numpy(), yu.cpu().numpy()) <= 1e-6


def test_splitk_workspace_reused_across_shapes():
    # the cached workspace is shared by GEMMs of different shapes: its counters must always be
    # found zeroed (regression: counters once lived after the shape-dependent partials)
    cases = [(16, 4096, 4096), (8, 6144, 4096), (16, 4096, 4096), (1, 4096, 12288), (8, 6144, 4096)]
    for i, (m, n, k) in enumerate(cases):
        a, sa, b, sb = _operands(m, n, k, 40 + i)
        y = _run(a, sa, b, sb).cpu().numpy()
        assert rel_frobenius(y, oracle.gemm_rows(a, sa, b, sb)) <= 1e-5, (m, n, k)


# ------------------------------------------------------------------- decode kernel (swap-AB)
@pytest.mark.parametrize("m,n,k", [
    (1, 256, 128), (3, 200, 256), (16, 1000, 512), (17, 384, 1024), (33, 4096, 4096),
    (64, 6144, 4096), (100, 1032, 1536), (127, 512, 12288), (128, 4096, 4096),
    # cluster split-K sizes 7, 4 (ragged last tile), 4 (148 CTAs) and 2
    (5, 128 * 21, 2048), (40, 128 * 29 + 64, 1024), (2, 128 * 37, 4096), (9, 128 * 74, 512),
    # M = 129..256: the swap-AB kernel with 256 token columns, cluster split-K only
    (200, 4096, 4096), (256, 1000, 2048), (129, 6144, 1024),
    # >= 148 weight tiles: ordered stream-K (every range >= one tile of k-blocks; gate_up at M = 1,
    # a ragged last tile, 4-k-block tiles) and, with ranges < one tile, the atomic fixup
    (1, 24576, 4096), (7, 128 * 150 + 40, 1024), (20, 128 * 300, 512), (1, 128 * 100, 4096),
])
def test_skinny_decode_vs_oracle(m, n, k):
    # 1 <= m <= 128 (dense) runs gemm_skinny.cu: tokens in the MMA N dimension (16..128 padded
    # by the tensor map's zero fill), split-K over a persistent grid with a deterministic fixup
    a, sa, b, sb = _operands(m, n, k, 50 + m)
    y = _run(a, sa, b, sb)
    rows = np.arange(m) if m <= 40 else np.unique(np.r_[0, m - 1, np.random.default_rng(m).integers(0, m, 24)])
    ref = oracle.gemm_rows(a, sa, b, sb, rows)
    got = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert rel_frobenius(got, ref) <= 1e-5
    for i in range(len(rows)):
        assert rel_frobenius(got[i], ref[i]) <= 1e-4
    yb = _run(a, sa, b, sb, torch.bfloat16)  # BF16 = RNE(F32), and deterministic
    assert torch.equal(yb.view(torch.int16), y.to(torch.bfloat16).view(torch.int16))
    assert torch.equal(_run(a, sa, b, sb).view(torch.int32), y.view(torch.int32))


@pytest.mark.parametrize("m,with_ws", [(24, False), (8, True), (3, True)])
def test_skinny_matches_tile_kernel_when_scales_misaligned(m, with_ws):
    # activation scales at a pointer that is not 16-byte aligned cannot be TMA-loaded: the call
    # falls back to the one-CTA tile kernel, whose result must agree; with a workspace and
    # M <= 16 that kernel splits K (deterministic serial fixup)
    n, k = 768, 1024
    a, sa, b, sb = _operands(m, n, k, 61)
    y = _run(a, sa, b, sb)
    ld = fp8q.act_scales_ld(m)
    mn = act_scales_mn_from_logical(sa, ld)
    big = torch.zeros((mn.shape[0], ld + 4), dtype=torch.float32, device="cuda")
    big[:, 1:1 + ld] = mn
    lib = fp8q.load_library()
    yt = torch.empty((m, n), dtype=torch.float32, device="cuda")
    da, db, dsb = (torch.from_numpy(t).cuda() for t in (a, b, sb))  # held until the kernel ran
    wsb = int(lib.fp8_block_gemm_workspace_size(m, n, k)) if with_ws else 0
    ws = torch.zeros(max(wsb, 1), dtype=torch.uint8, device="cuda")
    for _ in range(2):  # twice: the workspace must be left reusable
        st = lib.fp8_block_gemm(da.data_ptr(), k, big.data_ptr() + 4, ld + 4, db.data_ptr(), k, dsb.data_ptr(),
                                sb.shape[1], yt.data_ptr(), n, 1, m, n, k, ws.data_ptr() if wsb else None, wsb,
                                torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert st == 0
        assert rel_frobenius(yt.cpu().numpy(), y.cpu().numpy()) <= 1e-6


_STREAMK_SCRIPT = r"""
import numpy as np, torch, oracle
from tests.test_gpu_gemm import _operands, _run
from tests.helpers import rel_frobenius
for i, (m, n, k) in enumerate([(1, 6144, 4096), (64, 4096, 4096), (17, 384, 1024), (128, 4096, 12288)]):
    a, sa, b, sb = _operands(m, n, k, 70 + i)
    y = _run(a, sa, b, sb)
    rows = np.arange(min(m, 8))
    assert rel_frobenius(y[:len(rows)].cpu().numpy(), oracle.gemm_rows(a, sa, b, sb, rows)) <= 1e-5, (m, n, k)
    assert torch.equal(_run(a, sa, b, sb).view(torch.int32), y.view(torch.int32))
print("streamk ok")
"""


def test_skinny_streamk_path_when_cluster_split_disabled():
    # Shapes with few weight tiles run the cluster split-K mode (DSMEM reduction); with it
    # disabled (dev override, read once per process) the same shapes take the stream-K path
    # (global-workspace fixup), which must stay correct and deterministic.
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FP8Q_SKINNY_CLUSTER="0", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _STREAMK_SCRIPT], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "streamk ok" in r.stdout, r.stdout + r.stderr


_ORDERED_SCRIPT = r"""
import hashlib, sys, torch
from tests.test_gpu_gemm import _operands, _run
h = hashlib.sha256()
for i, (m, n, k) in enumerate([(1, 24576, 4096), (16, 24576, 4096), (32, 128 * 151 + 8, 2048), (5, 128 * 300, 512)]):
    a, sa, b, sb = _operands(m, n, k, 120 + i)
    h.update(_run(a, sa, b, sb).cpu().numpy().tobytes())
print("digest", h.hexdigest())
"""


def test_skinny_ordered_streamk_equals_atomic_fixup():
    # The ordered stream-K form (shared heads parked and flagged first, the owner combining them
    # last) adds the same two partials in the same order as the atomic last-arriver fixup: the
    # outputs are bitwise identical (FP8Q_SKINNY_ORDERED=0 forces the atomic form; fresh processes).
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = []
    for flag in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", _ORDERED_SCRIPT], cwd=root,
                           env=dict(os.environ, FP8Q_SKINNY_ORDERED=flag, PYTHONPATH=root),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "digest" in r.stdout, r.stdout + r.stderr
        out.append(r.stdout.split("digest")[1].strip())
    assert out[0] == out[1]


_KIND_SCRIPT = r"""
import numpy as np, torch, oracle
from tests.test_gpu_gemm import _operands, _run
from tests.helpers import rel_frobenius
for i, (m, n, k) in enumerate([(512, 512, 512), (300, 1000, 384), (1024, 2048, 1024)]):
    a, sa, b, sb = _operands(m, n, k, 90 + i)
    y = _run(a, sa, b, sb)
    rows = np.unique(np.r_[0, m - 1, np.random.default_rng(i).integers(0, m, 16)])
    got = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert rel_frobenius(got, oracle.gemm_rows(a, sa, b, sb, rows)) <= 1e-5, (m, n, k)
    yb = _run(a, sa, b, sb, torch.bfloat16)  # the BF16 store path (store warps / staging)
    assert torch.equal(yb.view(torch.int16), y.to(torch.bfloat16).view(torch.int16))
print("kind ok")
"""


@pytest.mark.parametrize("kind", ["256", "1256"])
def test_gemm_forced_kinds(kind):
    # Both tile kernels (FP8Q_GEMM_KIND forces one: 256 = one-CTA 128 x 256 tiles, 1256 = CTA pair
    # 256 x 256) are correct on every shape, including the shapes production sends to the other
    # one.  A fresh process per kind: the override is read once.
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FP8Q_GEMM_KIND=kind, PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _KIND_SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "kind ok" in r.stdout, r.stdout + r.stderr


def _unsplit_dev(xq, xs, wq, ws):
    """fp8_block_gemm through the C-ABI with no workspace (never splits K), F32 output."""
    m, k = xq.shape
    n = wq.shape[0]
    lib = fp8q.load_library()
    y = torch.empty((m, n), dtype=torch.float32, device="cuda")
    st = lib.fp8_block_gemm(xq.data_ptr(), k, xs.data_ptr(), xs.stride(0), wq.data_ptr(), k,
                            ws.data_ptr(), ws.stride(0), y.data_ptr(), n, 1, m, n, k, None, 0,
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert st == 0
    return y


@pytest.mark.parametrize("m,n,k", [(8192, 768, 4096), (2048, 512, 12288), (8192, 6144, 4096),
                                   (1100, 1000, 4096), (8192, 256, 4096), (4096, 384, 4096),
                                   (256, 4096, 12288), (256, 6144, 4096)])
def test_tail_split(m, n, k):
    # Tail-wave split of the CTA-pair kernel (gemm.cu plan_split): the last T mod 74 tiles are cut
    # into K slices whose fp32 partials the last slice sums in slice order (bulk-copied through
    # the idle shared-memory ring).  Ragged rows / columns: (1100, 1000).  Decode M = 256 down /
    # qkv: the split pair replaces the swap-AB cluster kernel (the unsplit reference, called
    # without a workspace, runs the latter).  Every element against the unsplit
    # kernel (equal up to fp32 summation order), sampled rows against the oracle, deterministic,
    # BF16 = RNE(F32) (whole tiles through the store warps, split tiles stored directly), and
    # the workspace left zeroed (the second call reuses it).
    lib = fp8q.load_library()
    assert lib.fp8_block_gemm_workspace_size(m, n, k) > 0
    wb = synth.qwen3_weight(n, k, 13)
    xb = synth.qwen3_activation(m, k, 14)
    wq, ws = fp8q.quantize_weight_blockwise(to_dev_bf16(wb))
    xq, xs = fp8q.quantize_act_per_token_group(to_dev_bf16(xb))
    y = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=torch.float32)
    yb = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=torch.bfloat16)
    y2 = fp8q.fp8_block_gemm(xq, xs, wq, ws, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32), y2.view(torch.int32))
    assert torch.equal(yb.view(torch.int16), y.to(torch.bfloat16).view(torch.int16))
    yu = _unsplit_dev(xq, xs, wq, ws)
    assert torch.isfinite(y).all()
    d = (y.double() - yu.double()).norm() / yu.double().norm()
    assert d <= 1e-6, float(d)
    # per 256-row band: a wrong or missing slice shows up as a whole band off
    for r0 in range(0, m, 256):
        nb = (y[r0:r0 + 256].double() - yu[r0:r0 + 256].double()).norm()
        assert nb <= 1e-6 * max(float(yu[r0:r0 + 256].double().norm()), 1e-30), (r0, float(nb))
    rows = np.unique(np.r_[0, m - 1, np.random.default_rng(m + n).integers(0, m, 16)])
    oa, osa = oracle.quantize_act_per_token_group(xb[rows])
    ow, osw = oracle.quantize_weight_blockwise(wb)
    ref = oracle.gemm_rows(oa, osa, ow, osw)
    assert rel_frobenius(y[torch.from_numpy(rows).cuda()].cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("m,n,k", [(1100, 1000, 4096), (8192, 768, 4096)])
def test_tail_split_bounds(m, n, k):
    # compute-sanitizer is closed on this pool, so the split path's memory footprint is checked
    # directly: an exact-size workspace followed by a canary, an output with guard rows, and the
    # counter region left zeroed (the reusable-workspace invariant of include/fp8q.h).
    lib = fp8q.load_library()
    need = int(lib.fp8_block_gemm_workspace_size(m, n, k))
    assert need > 0
    wb = synth.qwen3_weight(n, k, 21)
    xb = synth.qwen3_activation(m, k, 22)
    wq, ws = fp8q.quantize_weight_blockwise(to_dev_bf16(wb))
    xq, xs = fp8q.quantize_act_per_token_group(to_dev_bf16(xb))
    canary = 1 << 20
    wsp = torch.zeros(need + canary, dtype=torch.uint8, device="cuda")
    wsp[need:] = 0xA5
    guard = 3
    y = torch.full((m + guard, n), float("nan"), dtype=torch.float32, device="cuda")
    st = lib.fp8_block_gemm(xq.data_ptr(), k, xs.data_ptr(), xs.stride(0), wq.data_ptr(), k,
                            ws.data_ptr(), ws.stride(0), y.data_ptr(), n, 1, m, n, k, wsp.data_ptr(), need,
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert st == 0
    assert bool((wsp[need:] == 0xA5).all())              # nothing written past the workspace
    assert bool((wsp[:4096] == 0).all())                  # split counters left zeroed
    assert bool(torch.isnan(y[m:]).all())                 # nothing written past row m
    assert bool(torch.isfinite(y[:m]).all())              # every output written
    yu = _unsplit_dev(xq, xs, wq, ws)
    assert float((y[:m].double() - yu.double()).norm() / yu.double().norm()) <= 1e-6
