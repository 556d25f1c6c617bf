"""The C-ABI library loads and exports every symbol include/fp8q.h declares, and its
synchronous validation paths return the documented status codes (no GPU needed: these
return before any CUDA call).  Also: the product package never imports the oracle."""
import ast
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fp8q.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2601_18150_b200 import build
    build.build()
    from paper_2601_18150_b200 import fp8q
    return fp8q.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*[A-Za-z_][A-Za-z0-9_ \*]*?\b([a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("defined",)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ["quantize_weight_blockwise", "quantize_act_per_token_group", "fp8_block_gemm",
                     "fp8_block_gemm_grouped", "fp8_block_gemm_workspace_size",
                     "fp8_block_gemm_grouped_workspace_size", "fp8q_status_string", "fp8q_version",
                     "fp8q_kernel_launches", "rmsnorm_quantize_act_per_token_group",
                     "silu_mul_quantize_act_per_token_group", "kv_amax_update", "kv_scale_from_amax",
                     "kv_quantize_append", "quantize_weight_blockwise_fanout", "mx_scale_bytes", "mx_quantize",
                     "fp8_mx_gemm", "quantize_act_per_token_group_batched", "quantize_weight_blockwise_batched", "fp8_linear_dynamic", "fp8_linear_dynamic_workspace_size"]:
        assert required in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_status_strings_and_version(lib):
    for s in range(7):
        assert lib.fp8q_status_string(s).startswith(b"FP8Q_")
    assert lib.fp8q_version() == 10000
    assert lib.fp8q_kernel_launches() >= 0


def test_validation_paths_without_gpu(lib):
    P = ctypes.c_void_p
    fake = P(0x10000)  # 16-byte aligned, never dereferenced: validation returns first
    odd = P(0x10001)
    # negative dimension -> EINVAL
    assert lib.quantize_weight_blockwise(fake, -1, 128, 128, fake, 128, fake, 1, None, None) == 1
    # k % 8 -> ESHAPE
    assert lib.quantize_weight_blockwise(fake, 4, 12, 12, fake, 12, fake, 1, None, None) == 2
    # misaligned input -> EALIGN
    assert lib.quantize_weight_blockwise(odd, 4, 128, 128, fake, 128, fake, 1, None, None) == 3
    # ld too small -> EINVAL
    assert lib.quantize_weight_blockwise(fake, 4, 128, 64, fake, 128, fake, 1, None, None) == 1
    # empty -> OK, nothing enqueued
    assert lib.quantize_weight_blockwise(None, 0, 128, 128, None, 128, None, 1, None, None) == 0
    # activations: k % 128 -> ESHAPE, ld_s % 4 -> EALIGN
    assert lib.quantize_act_per_token_group(fake, 4, 200, 200, fake, 200, fake, 4, None, None) == 2
    assert lib.quantize_act_per_token_group(fake, 3, 128, 128, fake, 128, fake, 3, None, None) == 3
    # batched activations: every descriptor is validated first (second one bad -> its status)
    from paper_2601_18150_b200.fp8q import ActTensorDesc
    arr = (ActTensorDesc * 2)(ActTensorDesc(0x10000, 4, 128, 128, 0x10000, 128, 0x10000, 4),
                              ActTensorDesc(0x10000, 4, 200, 200, 0x10000, 200, 0x10000, 4))
    assert lib.quantize_act_per_token_group_batched(arr, 2, None, None) == 2
    arr[1] = ActTensorDesc(0x10001, 4, 128, 128, 0x10000, 128, 0x10000, 4)
    assert lib.quantize_act_per_token_group_batched(arr, 2, None, None) == 3
    assert lib.quantize_act_per_token_group_batched(arr, -1, None, None) == 1
    assert lib.quantize_act_per_token_group_batched(None, 0, None, None) == 0
    # GEMM: n % 8 -> ESHAPE; k % 128 -> ESHAPE; misaligned ld_a -> EALIGN
    assert lib.fp8_block_gemm(fake, 128, fake, 4, fake, 128, fake, 1, fake, 12, 0, 4, 12, 128, None, 0, None) == 2
    assert lib.fp8_block_gemm(fake, 200, fake, 4, fake, 200, fake, 1, fake, 16, 0, 4, 16, 200, None, 0, None) == 2
    assert lib.fp8_block_gemm(fake, 136, fake, 4, fake, 128, fake, 1, fake, 16, 0, 4, 16, 128, None, 0, None) == 3
    assert lib.fp8_block_gemm_grouped(fake, 128, fake, 4, fake, 128, 2048, fake, 1, 1, fake, 16, 0,
                                      4, 16, 128, fake, -1, None, 0, None) == 2
    # prefill: only the tail wave splits (148 SMs / 74 CTA pairs; gemm.cu plan_split).  o_proj:
    # 512 pair tiles = 6 x 74 + 68, 74 // 68 = 1 slice -> no split; qkv: 768 = 10 x 74 + 28 ->
    # 2 slices of 28 tiles, each parking 2 CTAs x 128 x 256 fp32 behind a 4 KB counter region
    assert lib.fp8_block_gemm_workspace_size(8192, 4096, 4096) == 0
    assert lib.fp8_block_gemm_workspace_size(8192, 6144, 4096) == 4096 + 28 * 2 * 2 * 128 * 256 * 4
    # the tail plan (S = min(74 // R, k-blocks // 16, 8), CTA pair, M >= 1024) on the shapes
    # DESIGN §5.2 names: R tail tiles x S slices x 2 CTAs x 128 KB behind the counters
    part = 2 * 128 * 256 * 4
    for (m, n, k), (r, sl) in {(8192, 768, 4096): (22, 2), (8192, 2048, 12288): (34, 2),
                               (2048, 512, 12288): (16, 4), (8192, 256, 4096): (32, 2),
                               (256, 4096, 12288): (16, 4), (256, 6144, 4096): (24, 2)}.items():
        assert lib.fp8_block_gemm_workspace_size(m, n, k) == 4096 + r * sl * part, (m, n, k)
    for m, n, k in [(256, 24576, 4096),   # M < 1024 with a whole wave: no gain (decode gate_up)
                    (256, 4096, 4096),    # M < 1024, slices on 64 SMs: the cluster kernel wins
                    (8192, 640, 2048),    # K = 2048: slices under 16 k-blocks
                    (8192, 24576, 4096),  # 3072 = 41 x 74 + 38: 74 // 38 = 1
                    (8192, 4096, 12288)]:  # 512 = 6 x 74 + 68
        assert lib.fp8_block_gemm_workspace_size(m, n, k) == 0, (m, n, k)
    # NEXT-3 KV cache: ld < cols -> EINVAL; identity slots with rows > num_slots -> ESHAPE;
    # misaligned amax / scale -> EALIGN; empty -> OK
    assert lib.kv_amax_update(fake, 4, 1024, 512, fake, None, None) == 1
    assert lib.kv_amax_update(fake, 4, 1024, 1024, odd, None, None) == 3
    assert lib.kv_amax_update(None, 0, 1024, 1024, None, None, None) == 0
    assert lib.kv_scale_from_amax(fake, -1, fake, None) == 1
    assert lib.kv_quantize_append(fake, 8, 1024, 1024, fake, None, fake, 1024, 4, None, None, None) == 2
    assert lib.kv_quantize_append(fake, 8, 1024, 1024, odd, fake, fake, 1024, 4, None, None, None) == 3
    assert lib.kv_quantize_append(fake, 8, 1024, 1024, fake, fake, fake, 512, 16, None, None, None) == 1
    # NEXT-4 MXFP8: k % 128 -> ESHAPE; n % 256 -> ESHAPE; scale bytes per (128 rows, k-block) = 512
    assert lib.mx_scale_bytes(300, 4096) == 3 * 32 * 512 and lib.mx_scale_bytes(4, 100) == 0
    assert lib.mx_quantize(fake, 4, 200, 200, fake, 200, fake, None, None) == 2
    assert lib.fp8_mx_gemm(fake, 128, fake, fake, 128, fake, fake, 128, 0, 4, 128, 128, None) == 2
    # NEXT-1 fan-out: no destination -> EINVAL; misaligned delta -> EALIGN
    from paper_2601_18150_b200.fp8q import WeightTensorDesc
    arr = (WeightTensorDesc * 1)(WeightTensorDesc(0x10000, 128, 256, 256, 0x10000, 256, 0x10000, 2))
    d0 = (ctypes.c_int64 * 2)(0, 8)
    assert lib.quantize_weight_blockwise_fanout(arr, 1, 0, d0, d0, None, None) == 1
    assert lib.quantize_weight_blockwise_fanout(arr, 1, 2, d0, d0, None, None) == 3


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2601_18150_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", f
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                for line in open(os.path.join(dirpath, f)):
                    if line.lstrip().startswith("#include"):
                        assert "oracle" not in line, (f, line)


def test_oracle_never_includes_product_headers():
    src = open(os.path.join(ROOT, "oracle", "fp8q_oracle.c")).read()
    assert "#include \"" not in src
    tree = ast.parse(open(os.path.join(ROOT, "oracle", "__init__.py")).read())
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            assert not any(a.name.startswith("paper_2601_18150_b200") for a in node.names)
        if isinstance(node, ast.ImportFrom):
            assert not (node.module or "").startswith("paper_2601_18150_b200")
