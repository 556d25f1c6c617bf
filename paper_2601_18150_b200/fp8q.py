"""Thin Python binding of libfp8q (include/fp8q.h) -- argument marshalling only.

Every step of the hot path runs in the sm_100a kernels behind the C-ABI; this module only
turns torch tensors (device memory from PyTorch's caching allocator) into pointers, leading
dimensions and the current CUDA stream.  There is no CPU fallback: if libfp8q.so is missing
or a tensor is not on a CUDA device, the call raises.

Names follow the C-ABI and the paper (§2.1.1, Eq. (1)).
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FP8Q_LIB (dev A/B only): load another build of the same library
LIB_PATH = os.environ.get("FP8Q_LIB") or os.path.join(_HERE, "libfp8q.so")

FP8Q_OUT_BF16 = 0
FP8Q_OUT_F32 = 1

_lock = threading.Lock()
_lib = None


class WeightTensorDesc(ctypes.Structure):
    """fp8q_weight_tensor (include/fp8q.h)."""
    _fields_ = [("w_bf16", ctypes.c_void_p), ("n", ctypes.c_int64), ("k", ctypes.c_int64),
                ("ld_w", ctypes.c_int64), ("codes", ctypes.c_void_p), ("ld_q", ctypes.c_int64),
                ("scales", ctypes.c_void_p), ("ld_s", ctypes.c_int64)]


class ActTensorDesc(ctypes.Structure):
    """fp8q_act_tensor (include/fp8q.h)."""
    _fields_ = [("x_bf16", ctypes.c_void_p), ("m", ctypes.c_int64), ("k", ctypes.c_int64),
                ("ld_x", ctypes.c_int64), ("codes", ctypes.c_void_p), ("ld_q", ctypes.c_int64),
                ("scales", ctypes.c_void_p), ("ld_s", ctypes.c_int64)]


class Fp8qError(RuntimeError):
    """A libfp8q entry point returned a non-OK fp8q_status."""


def load_library() -> ctypes.CDLL:
    """Load libfp8q.so from the package directory; raise if it was not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise Fp8qError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2601_18150_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        lib.fp8q_status_string.argtypes = [ctypes.c_int]
        lib.fp8q_status_string.restype = ctypes.c_char_p
        lib.fp8q_version.restype = I32
        if hasattr(lib, "fp8q_last_cuda_error"):  # (older builds loaded via FP8Q_LIB lack it)
            lib.fp8q_last_cuda_error.restype = ctypes.c_char_p
        lib.fp8q_kernel_launches.restype = I64
        lib.quantize_weight_blockwise.argtypes = [P, I64, I64, I64, P, I64, P, I64, P, P]
        lib.quantize_weight_blockwise.restype = ctypes.c_int
        lib.quantize_weight_blockwise_batched.argtypes = [ctypes.POINTER(WeightTensorDesc), I32, P, P]
        lib.quantize_weight_blockwise_batched.restype = ctypes.c_int
        lib.quantize_weight_blockwise_fanout.argtypes = [ctypes.POINTER(WeightTensorDesc), I32, I32, P, P, P, P]
        lib.quantize_weight_blockwise_fanout.restype = ctypes.c_int
        lib.e4m3_encode_f32.argtypes = [P, I64, P, P]
        lib.e4m3_encode_f32.restype = ctypes.c_int
        lib.quantize_act_per_token_group.argtypes = [P, I64, I64, I64, P, I64, P, I64, P, P]
        lib.quantize_act_per_token_group.restype = ctypes.c_int
        lib.quantize_act_per_token_group_batched.argtypes = [ctypes.POINTER(ActTensorDesc), I32, P, P]
        lib.quantize_act_per_token_group_batched.restype = ctypes.c_int
        lib.rmsnorm_quantize_act_per_token_group.argtypes = [P, P, ctypes.c_float, I64, I64, I64, P, I64, P, I64,
                                                             P, I64, P, P]
        lib.rmsnorm_quantize_act_per_token_group.restype = ctypes.c_int
        lib.silu_mul_quantize_act_per_token_group.argtypes = [P, I64, I64, I64, P, I64, P, I64, P, I64, P, P]
        lib.silu_mul_quantize_act_per_token_group.restype = ctypes.c_int
        lib.fp8_block_gemm_workspace_size.argtypes = [I64, I64, I64]
        lib.fp8_block_gemm_workspace_size.restype = ctypes.c_size_t
        lib.fp8_block_gemm.argtypes = [P, I64, P, I64, P, I64, P, I64, P, I64, ctypes.c_int,
                                       I64, I64, I64, P, ctypes.c_size_t, P]
        lib.fp8_block_gemm.restype = ctypes.c_int
        lib.fp8_linear_dynamic_workspace_size.argtypes = [I64, I64, I64]
        lib.fp8_linear_dynamic_workspace_size.restype = ctypes.c_size_t
        lib.fp8_linear_dynamic.argtypes = [P, I64, P, I64, P, I64, P, I64, ctypes.c_int, I64, I64, I64, P, P,
                                           ctypes.c_size_t, P]
        lib.fp8_linear_dynamic.restype = ctypes.c_int
        lib.fp8_block_gemm_grouped_workspace_size.argtypes = [I64, I64, I64, I32]
        lib.fp8_block_gemm_grouped_workspace_size.restype = ctypes.c_size_t
        lib.fp8_block_gemm_grouped.argtypes = [P, I64, P, I64, P, I64, I64, P, I64, I64, P, I64,
                                               ctypes.c_int, I64, I64, I64, P, I32, P,
                                               ctypes.c_size_t, P]
        lib.fp8_block_gemm_grouped.restype = ctypes.c_int
        lib.kv_amax_update.argtypes = [P, I64, I64, I64, P, P, P]
        lib.kv_amax_update.restype = ctypes.c_int
        lib.kv_scale_from_amax.argtypes = [P, I64, P, P]
        lib.kv_scale_from_amax.restype = ctypes.c_int
        lib.kv_quantize_append.argtypes = [P, I64, I64, I64, P, P, P, I64, I64, P, P, P]
        lib.kv_quantize_append.restype = ctypes.c_int
        lib.mx_scale_bytes.argtypes = [I64, I64]
        lib.mx_scale_bytes.restype = ctypes.c_size_t
        lib.mx_quantize.argtypes = [P, I64, I64, I64, P, I64, P, P, P]
        lib.mx_quantize.restype = ctypes.c_int
        lib.fp8_mx_gemm.argtypes = [P, I64, P, P, I64, P, P, I64, ctypes.c_int, I64, I64, I64, P]
        lib.fp8_mx_gemm.restype = ctypes.c_int
        _lib = lib
        return lib


def _check(status: int, what: str) -> None:
    if status != 0:
        lib = load_library()
        msg = lib.fp8q_status_string(status).decode()
        if "ECUDA" in msg and hasattr(lib, "fp8q_last_cuda_error"):
            msg += f" ({lib.fp8q_last_cuda_error().decode()})"
        raise Fp8qError(f"{what}: {msg}")


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _cuda2d(t: torch.Tensor, name: str, dtype: torch.dtype) -> torch.Tensor:
    if not t.is_cuda:
        raise Fp8qError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != dtype:
        raise Fp8qError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() != 2 or (t.numel() and t.stride(1) != 1):
        raise Fp8qError(f"{name} must be 2-D with unit stride in the last dimension")
    return t


def _ld(t: torch.Tensor) -> int:
    return t.stride(0) if t.shape[0] > 1 else max(t.stride(0), t.shape[1])


def kernel_launches() -> int:
    """Kernels libfp8q has launched in this process (for bench.py's gpu_launches)."""
    return int(load_library().fp8q_kernel_launches())


def version() -> int:
    return int(load_library().fp8q_version())


# ------------------------------------------------------------------------------ quantizers
def quantize_weight_blockwise(w: torch.Tensor, codes: torch.Tensor | None = None,
                              scales: torch.Tensor | None = None,
                              nonfinite_flag: torch.Tensor | None = None, stream=None):
    """Eq. (1): BF16 [n, k] -> (E4M3 codes uint8 [n, k], fp32 scales
    [ceil(n/128), ceil(k/128)]), one scale = RN32(amax/448) per 128x128 block."""
    _cuda2d(w, "w", torch.bfloat16)
    n, k = w.shape
    if codes is None:
        codes = torch.empty((n, k), dtype=torch.uint8, device=w.device)
    if scales is None:
        scales = torch.empty(((n + 127) // 128, (k + 127) // 128), dtype=torch.float32, device=w.device)
    _cuda2d(codes, "codes", torch.uint8)
    _cuda2d(scales, "scales", torch.float32)
    if codes.shape != (n, k) or scales.shape[0] < (n + 127) // 128 or scales.shape[1] < (k + 127) // 128:
        raise Fp8qError("output shape mismatch")
    flag = nonfinite_flag.data_ptr() if nonfinite_flag is not None else None
    _check(load_library().quantize_weight_blockwise(
        w.data_ptr(), n, k, _ld(w), codes.data_ptr(), _ld(codes), scales.data_ptr(), _ld(scales),
        flag, _stream(stream)), "quantize_weight_blockwise")
    return codes, scales


def quantize_weight_blockwise_batched(items, nonfinite_flag: torch.Tensor | None = None, stream=None):
    """Several blockwise weight quantizations (Eq. (1)) in as few launches as possible -- the
    per-step weight sync of PAPER.md:72.  items: sequence of (w, codes, scales) CUDA tensors
    with the shapes of quantize_weight_blockwise's inputs/outputs."""
    items = list(items)
    arr = (WeightTensorDesc * max(1, len(items)))()
    for i, (w, codes, scales) in enumerate(items):
        _cuda2d(w, "w", torch.bfloat16)
        _cuda2d(codes, "codes", torch.uint8)
        _cuda2d(scales, "scales", torch.float32)
        n, k = w.shape
        if codes.shape != (n, k) or scales.shape[0] < (n + 127) // 128 or scales.shape[1] < (k + 127) // 128:
            raise Fp8qError(f"item {i}: output shape mismatch")
        arr[i] = WeightTensorDesc(w.data_ptr(), n, k, _ld(w), codes.data_ptr(), _ld(codes),
                                  scales.data_ptr(), _ld(scales))
    flag = nonfinite_flag.data_ptr() if nonfinite_flag is not None else None
    _check(load_library().quantize_weight_blockwise_batched(arr, len(items), flag, _stream(stream)),
           "quantize_weight_blockwise_batched")


def quantize_weight_blockwise_fanout(items, codes_delta, scales_delta, nonfinite_flag: torch.Tensor | None = None,
                                     stream=None):
    """NEXT-1: quantize_weight_blockwise_batched whose code / scale stores go to every
    destination: pointer + codes_delta[d] / scales_delta[d] (bytes; peer-mapped buffers of
    identical layout, delta 0 = the local buffer)."""
    items = list(items)
    arr = (WeightTensorDesc * max(1, len(items)))()
    for i, (w, codes, scales) in enumerate(items):
        _cuda2d(w, "w", torch.bfloat16)
        _cuda2d(codes, "codes", torch.uint8)
        _cuda2d(scales, "scales", torch.float32)
        n, k = w.shape
        if codes.shape != (n, k) or scales.shape[0] < (n + 127) // 128 or scales.shape[1] < (k + 127) // 128:
            raise Fp8qError(f"item {i}: output shape mismatch")
        arr[i] = WeightTensorDesc(w.data_ptr(), n, k, _ld(w), codes.data_ptr(), _ld(codes),
                                  scales.data_ptr(), _ld(scales))
    nd = len(codes_delta)
    if nd != len(scales_delta):
        raise Fp8qError("codes_delta and scales_delta must have one entry per destination")
    cd = (ctypes.c_int64 * max(1, nd))(*[int(v) for v in codes_delta])
    sd = (ctypes.c_int64 * max(1, nd))(*[int(v) for v in scales_delta])
    flag = nonfinite_flag.data_ptr() if nonfinite_flag is not None else None
    _check(load_library().quantize_weight_blockwise_fanout(arr, len(items), nd, ctypes.cast(cd, ctypes.c_void_p),
                                                           ctypes.cast(sd, ctypes.c_void_p), flag, _stream(stream)),
           "quantize_weight_blockwise_fanout")


def e4m3_encode_f32(x: torch.Tensor, codes: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Step a3 alone: E4M3_RNE_satfinite of raw fp32 values through the
    quantizers' hardware cvt -- for checking the encode on every fp32 bit pattern."""
    if not (x.is_cuda and x.dtype == torch.float32 and x.dim() == 1 and x.is_contiguous()):
        raise Fp8qError("x must be a contiguous 1-D CUDA float32 tensor")
    if codes is None:
        codes = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
    if not (codes.is_cuda and codes.dtype == torch.uint8 and codes.is_contiguous() and codes.numel() == x.numel()):
        raise Fp8qError("codes must be a contiguous CUDA uint8 tensor with x.numel() elements")
    _check(load_library().e4m3_encode_f32(x.data_ptr(), x.numel(), codes.data_ptr(), _stream(stream)),
           "e4m3_encode_f32")
    return codes


def act_scales_ld(m: int) -> int:
    """Leading dimension of the MN-major activation-scale array (>= m, multiple of 4)."""
    return max(4, (m + 3) // 4 * 4)


def quantize_act_per_token_group(x: torch.Tensor, codes: torch.Tensor | None = None,
                                 scales: torch.Tensor | None = None,
                                 nonfinite_flag: torch.Tensor | None = None, stream=None):
    """Dynamic 1x128 activation quantization: BF16 [m, k] -> (codes uint8
    [m, k], scales fp32 MN-major [k/128, ld_s] with scales[g, m] the scale of token m, group g)."""
    _cuda2d(x, "x", torch.bfloat16)
    m, k = x.shape
    if codes is None:
        codes = torch.empty((m, k), dtype=torch.uint8, device=x.device)
    if scales is None:
        scales = torch.empty((k // 128, act_scales_ld(m)), dtype=torch.float32, device=x.device)
    _cuda2d(codes, "codes", torch.uint8)
    _cuda2d(scales, "scales", torch.float32)
    if codes.shape != (m, k) or scales.shape[0] < k // 128 or scales.shape[1] < m:
        raise Fp8qError("output shape mismatch")
    flag = nonfinite_flag.data_ptr() if nonfinite_flag is not None else None
    _check(load_library().quantize_act_per_token_group(
        x.data_ptr(), m, k, _ld(x), codes.data_ptr(), _ld(codes), scales.data_ptr(),
        scales.stride(0) if scales.shape[0] > 1 else scales.shape[1], flag, _stream(stream)),
        "quantize_act_per_token_group")
    return codes, scales


def quantize_act_per_token_group_batched(items, nonfinite_flag: torch.Tensor | None = None, stream=None):
    """Several dynamic activation quantizations in as few launches as
    possible -- a layer's GEMM inputs in one persistent launch.  items: sequence of
    (x, codes, scales) CUDA tensors with the shapes of quantize_act_per_token_group's
    inputs/outputs (scales MN-major [k/128, >= m])."""
    items = list(items)
    arr = (ActTensorDesc * max(1, len(items)))()
    for i, (x, codes, scales) in enumerate(items):
        _cuda2d(x, "x", torch.bfloat16)
        _cuda2d(codes, "codes", torch.uint8)
        _cuda2d(scales, "scales", torch.float32)
        m, k = x.shape
        if codes.shape != (m, k) or scales.shape[0] < k // 128 or scales.shape[1] < m:
            raise Fp8qError(f"item {i}: output shape mismatch")
        arr[i] = ActTensorDesc(x.data_ptr(), m, k, _ld(x), codes.data_ptr(), _ld(codes), scales.data_ptr(),
                               scales.stride(0) if scales.shape[0] > 1 else scales.shape[1])
    flag = nonfinite_flag.data_ptr() if nonfinite_flag is not None else None
    _check(load_library().quantize_act_per_token_group_batched(arr, len(items), flag, _stream(stream)),
           "quantize_act_per_token_group_batched")


def _act_outputs(m, k, device, codes, scales):
    if codes is None:
        codes = torch.empty((m, k), dtype=torch.uint8, device=device)
    if scales is None:
        scales = torch.empty((k // 128, act_scales_ld(m)), dtype=torch.float32, device=device)
    _cuda2d(codes, "codes", torch.uint8)
    _cuda2d(scales, "scales", torch.float32)
    if codes.shape != (m, k) or scales.shape[0] < k // 128 or scales.shape[1] < m:
        raise Fp8qError("output shape mismatch")
    return codes, scales


def rmsnorm_quantize_act_per_token_group(x: torch.Tensor, gamma: torch.Tensor, eps: float,
                                         codes=None, scales=None, y_out=None, nonfinite_flag=None,
                                         stream=None):
    """NEXT-2: BF16(RMSNorm(x) * gamma) quantized per token per 128 channels, y never stored
    unless y_out is given.  Returns (codes, scales MN-major)."""
    _cuda2d(x, "x", torch.bfloat16)
    if not (gamma.is_cuda and gamma.dtype == torch.bfloat16 and gamma.dim() == 1 and gamma.is_contiguous()):
        raise Fp8qError("gamma must be a contiguous CUDA bfloat16 vector")
    m, k = x.shape
    if gamma.numel() != k:
        raise Fp8qError(f"gamma must have k={k} elements, got {gamma.numel()}")
    codes, scales = _act_outputs(m, k, x.device, codes, scales)
    y_ptr, ld_y = (None, 0)
    if y_out is not None:
        _cuda2d(y_out, "y_out", torch.bfloat16)
        y_ptr, ld_y = y_out.data_ptr(), _ld(y_out)
    flag = nonfinite_flag.data_ptr() if nonfinite_flag is not None else None
    _check(load_library().rmsnorm_quantize_act_per_token_group(
        x.data_ptr(), gamma.data_ptr(), float(eps), m, k, _ld(x), codes.data_ptr(), _ld(codes),
        scales.data_ptr(), scales.stride(0) if scales.shape[0] > 1 else scales.shape[1], y_ptr, ld_y, flag,
        _stream(stream)), "rmsnorm_quantize_act_per_token_group")
    return codes, scales


def silu_mul_quantize_act_per_token_group(gate_up: torch.Tensor, codes=None, scales=None, y_out=None,
                                          nonfinite_flag=None, stream=None):
    """NEXT-2: BF16(silu(gate) * up) for gate_up = [gate | up], quantized per token per 128
    channels.  Returns (codes [m, inter], scales MN-major)."""
    _cuda2d(gate_up, "gate_up", torch.bfloat16)
    m, k2 = gate_up.shape
    inter = k2 // 2
    codes, scales = _act_outputs(m, inter, gate_up.device, codes, scales)
    y_ptr, ld_y = (None, 0)
    if y_out is not None:
        _cuda2d(y_out, "y_out", torch.bfloat16)
        y_ptr, ld_y = y_out.data_ptr(), _ld(y_out)
    flag = nonfinite_flag.data_ptr() if nonfinite_flag is not None else None
    _check(load_library().silu_mul_quantize_act_per_token_group(
        gate_up.data_ptr(), m, inter, _ld(gate_up), codes.data_ptr(), _ld(codes), scales.data_ptr(),
        scales.stride(0) if scales.shape[0] > 1 else scales.shape[1], y_ptr, ld_y, flag, _stream(stream)),
        "silu_mul_quantize_act_per_token_group")
    return codes, scales


# ------------------------------------------------------------------------------ GEMMs
def _out(out, m, n, out_dtype, device):
    if out is None:
        out = torch.empty((m, n), dtype=out_dtype, device=device)
    if out_dtype not in (torch.bfloat16, torch.float32) or out.dtype != out_dtype:
        raise Fp8qError("out dtype must be torch.bfloat16 or torch.float32")
    _cuda2d(out, "out", out_dtype)
    if out.shape != (m, n):
        raise Fp8qError("out shape mismatch")
    return out


_WS: dict = {}


def _stream_obj(stream, device) -> torch.cuda.Stream:
    if stream is None:
        return torch.cuda.current_stream(device)
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(stream), device=device)


def _workspace(device, stream, nbytes: int):
    """Zero-filled split-K workspace cached per (device, stream); the kernels leave it zeroed.

    Allocated and zero-filled ON the stream the GEMM runs on, so the caching allocator ties the
    block to that stream: the memset is ordered before the GEMM, and a replaced (smaller)
    workspace is only recycled for later work on the same stream, after the GEMMs that used it."""
    if nbytes == 0:
        return None, 0
    st = _stream_obj(stream, device)
    key = (device.index, st.cuda_stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        with torch.cuda.stream(st):
            ws = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws.data_ptr(), ws.numel()


def _check_act_scales(sc: torch.Tensor, m: int, k: int, name: str) -> int:
    """MN-major activation scales [k/128, ld_s >= m]: returns ld_s."""
    _cuda2d(sc, name, torch.float32)
    if sc.shape[0] < k // 128 or (sc.shape[1] < m and m > 0):
        raise Fp8qError(f"{name} must be at least [k/128={k // 128}, m={m}], got {tuple(sc.shape)}")
    return sc.stride(0) if sc.shape[0] > 1 else sc.shape[1]


def _check_weight_scales(sc: torch.Tensor, n: int, k: int, name: str) -> int:
    """Weight scales [ceil(n/128), >= k/128]: returns ld_sb."""
    _cuda2d(sc, name, torch.float32)
    if sc.shape[0] < (n + 127) // 128 or sc.shape[1] < k // 128:
        raise Fp8qError(f"{name} must be at least [ceil(n/128)={(n + 127) // 128}, k/128={k // 128}], "
                        f"got {tuple(sc.shape)}")
    return sc.stride(0) if sc.shape[0] > 1 else sc.shape[1]


def fp8_block_gemm(a: torch.Tensor, a_scales: torch.Tensor, b: torch.Tensor, b_scales: torch.Tensor,
                   out_dtype: torch.dtype = torch.bfloat16, out: torch.Tensor | None = None,
                   stream=None) -> torch.Tensor:
    """W8A8 linear Y = X W^T: a codes [m,k], a_scales MN-major [k/128, >=m],
    b codes [n,k], b_scales [ceil(n/128), >=k/128] -> D [m, n] (BF16 or F32)."""
    _cuda2d(a, "a", torch.uint8)
    _cuda2d(b, "b", torch.uint8)
    _cuda2d(a_scales, "a_scales", torch.float32)
    _cuda2d(b_scales, "b_scales", torch.float32)
    m, k = a.shape
    n, kb = b.shape
    if kb != k:
        raise Fp8qError("fp8_block_gemm: inner dimensions differ")
    out = _out(out, m, n, out_dtype, a.device)
    ld_sa = _check_act_scales(a_scales, m, k, "a_scales")
    ld_sb = _check_weight_scales(b_scales, n, k, "b_scales")
    lib = load_library()
    sh = _stream(stream)
    ws_ptr, ws_bytes = _workspace(a.device, stream, int(lib.fp8_block_gemm_workspace_size(m, n, k)))
    _check(lib.fp8_block_gemm(
        a.data_ptr(), _ld(a), a_scales.data_ptr(), ld_sa, b.data_ptr(), _ld(b), b_scales.data_ptr(),
        ld_sb, out.data_ptr(), _ld(out), FP8Q_OUT_F32 if out_dtype == torch.float32 else FP8Q_OUT_BF16,
        m, n, k, ws_ptr, ws_bytes, sh), "fp8_block_gemm")
    return out


def fp8_linear_dynamic(x: torch.Tensor, b: torch.Tensor, b_scales: torch.Tensor,
                       out_dtype: torch.dtype = torch.bfloat16, out: torch.Tensor | None = None,
                       nonfinite_flag: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """One W8A8 linear with dynamic activation quantization: BF16 x [m,k],
    b codes [n,k], b_scales [ceil(n/128), >=k/128] -> D [m, n]; bit-identical to
    quantize_act_per_token_group followed by fp8_block_gemm (two PDL-chained launches)."""
    _cuda2d(x, "x", torch.bfloat16)
    _cuda2d(b, "b", torch.uint8)
    _cuda2d(b_scales, "b_scales", torch.float32)
    m, k = x.shape
    n, kb = b.shape
    if kb != k:
        raise Fp8qError("fp8_linear_dynamic: inner dimensions differ")
    out = _out(out, m, n, out_dtype, x.device)
    ld_sb = _check_weight_scales(b_scales, n, k, "b_scales")
    lib = load_library()
    ws_ptr, ws_bytes = _workspace(x.device, stream, int(lib.fp8_linear_dynamic_workspace_size(m, n, k)))
    flag = nonfinite_flag.data_ptr() if nonfinite_flag is not None else None
    _check(lib.fp8_linear_dynamic(
        x.data_ptr(), _ld(x), b.data_ptr(), _ld(b), b_scales.data_ptr(), ld_sb, out.data_ptr(), _ld(out),
        FP8Q_OUT_F32 if out_dtype == torch.float32 else FP8Q_OUT_BF16, m, n, k, flag, ws_ptr, ws_bytes,
        _stream(stream)), "fp8_linear_dynamic")
    return out


def fp8_block_gemm_grouped(a: torch.Tensor, a_scales: torch.Tensor, b: torch.Tensor,
                           b_scales: torch.Tensor, offsets: torch.Tensor,
                           out_dtype: torch.dtype = torch.bfloat16, out: torch.Tensor | None = None,
                           stream=None) -> torch.Tensor:
    """MoE experts: rows [offsets[g], offsets[g+1]) of a times expert g.
    b codes [G, n, k]; b_scales [G, ceil(n/128), k/128]; offsets int32 [G+1] on the device."""
    _cuda2d(a, "a", torch.uint8)
    _cuda2d(a_scales, "a_scales", torch.float32)
    if not (b.is_cuda and b.dtype == torch.uint8 and b.dim() == 3 and b.stride(2) == 1):
        raise Fp8qError("b must be a CUDA uint8 [G, n, k] tensor with unit inner stride")
    if not (b_scales.is_cuda and b_scales.dtype == torch.float32 and b_scales.dim() == 3 and b_scales.stride(2) == 1):
        raise Fp8qError("b_scales must be a CUDA float32 [G, nb, kb] tensor")
    if not (offsets.is_cuda and offsets.dtype == torch.int32 and offsets.dim() == 1 and offsets.is_contiguous()):
        raise Fp8qError("offsets must be a contiguous CUDA int32 tensor [G+1]")
    G, n, k = b.shape
    if offsets.numel() != G + 1:
        raise Fp8qError("offsets must have num_groups + 1 entries")
    m = a.shape[0]
    if a.shape[1] != k:
        raise Fp8qError("inner dimensions differ")
    out = _out(out, m, n, out_dtype, a.device)
    ld_sa = _check_act_scales(a_scales, m, k, "a_scales")
    if b_scales.shape[0] < G or b_scales.shape[1] < (n + 127) // 128 or b_scales.shape[2] < k // 128:
        raise Fp8qError(f"b_scales must be at least [G={G}, ceil(n/128)={(n + 127) // 128}, k/128={k // 128}], "
                        f"got {tuple(b_scales.shape)}")
    _check(load_library().fp8_block_gemm_grouped(
        a.data_ptr(), _ld(a), a_scales.data_ptr(), ld_sa, b.data_ptr(), b.stride(1), b.stride(0),
        b_scales.data_ptr(), b_scales.stride(1), b_scales.stride(0), out.data_ptr(), _ld(out),
        FP8Q_OUT_F32 if out_dtype == torch.float32 else FP8Q_OUT_BF16, m, n, k, offsets.data_ptr(),
        G, None, 0, _stream(stream)), "fp8_block_gemm_grouped")
    return out


# ------------------------------------------------------------------ NEXT-3 FP8 KV cache
def _opt_ptr(t, name, dtype):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == dtype):
        raise Fp8qError(f"{name} must be a CUDA {dtype} tensor")
    return t.data_ptr()


def kv_amax_update(x: torch.Tensor, amax_bits: torch.Tensor, flag: torch.Tensor | None = None, stream=None):
    """amax_bits (int32 [1] on the device, BF16 bits) = max(amax_bits, max |x|)."""
    _cuda2d(x, "x", torch.bfloat16)
    ap = _opt_ptr(amax_bits, "amax_bits", torch.int32)
    if ap is None:
        raise Fp8qError("amax_bits is required")
    _check(load_library().kv_amax_update(x.data_ptr(), x.shape[0], x.shape[1], _ld(x), ap,
                                         _opt_ptr(flag, "flag", torch.int32), _stream(stream)), "kv_amax_update")
    return amax_bits


def kv_scale_from_amax(amax_bits: torch.Tensor, scales: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """scales[i] = RN32(amax_i / 448), amax 0 -> 1, for every entry of amax_bits (int32)."""
    if not (amax_bits.is_cuda and amax_bits.dtype == torch.int32 and amax_bits.is_contiguous()):
        raise Fp8qError("amax_bits must be a contiguous CUDA int32 tensor")
    if scales is None:
        scales = torch.empty(amax_bits.shape, dtype=torch.float32, device=amax_bits.device)
    _check(load_library().kv_scale_from_amax(amax_bits.data_ptr(), amax_bits.numel(),
                                             _opt_ptr(scales, "scales", torch.float32), _stream(stream)),
           "kv_scale_from_amax")
    return scales


def kv_quantize_append(x: torch.Tensor, scale: torch.Tensor, cache: torch.Tensor, slots: torch.Tensor | None = None,
                       saturated: torch.Tensor | None = None, flag: torch.Tensor | None = None, stream=None):
    """cache[slots[r]] = E4M3 codes of x[r] / scale (scale: CUDA float32 scalar tensor);
    saturated (int32 [1]) accumulates the saturated-element count."""
    _cuda2d(x, "x", torch.bfloat16)
    _cuda2d(cache, "cache", torch.uint8)
    if not (scale.is_cuda and scale.dtype == torch.float32 and scale.numel() >= 1):
        raise Fp8qError("scale must be a CUDA float32 tensor")
    if slots is not None and not (slots.is_cuda and slots.dtype == torch.int32 and slots.is_contiguous()
                                  and slots.numel() == x.shape[0]):
        raise Fp8qError("slots must be a contiguous CUDA int32 tensor with one entry per row of x")
    _check(load_library().kv_quantize_append(
        x.data_ptr(), x.shape[0], x.shape[1], _ld(x), scale.data_ptr(),
        slots.data_ptr() if slots is not None else None, cache.data_ptr(), _ld(cache), cache.shape[0],
        _opt_ptr(saturated, "saturated", torch.int32), _opt_ptr(flag, "flag", torch.int32), _stream(stream)),
        "kv_quantize_append")
    return cache


# ------------------------------------------------------------------ NEXT-4 MXFP8 variant
def mx_quantize(x: torch.Tensor, codes: torch.Tensor | None = None, scales: torch.Tensor | None = None,
                nonfinite_flag: torch.Tensor | None = None, stream=None):
    """MXFP8: E4M3 codes [rows, k] + native E8M0 scale bytes (mx_scale_bytes(rows, k))."""
    _cuda2d(x, "x", torch.bfloat16)
    rows, k = x.shape
    lib = load_library()
    if codes is None:
        codes = torch.empty((rows, k), dtype=torch.uint8, device=x.device)
    need = int(lib.mx_scale_bytes(rows, k))
    if scales is None:
        scales = torch.empty(max(1, need), dtype=torch.uint8, device=x.device)
    _cuda2d(codes, "codes", torch.uint8)
    if codes.shape != (rows, k):
        raise Fp8qError("codes shape mismatch")
    if not (scales.is_cuda and scales.dtype == torch.uint8 and scales.is_contiguous() and scales.numel() >= need):
        raise Fp8qError(f"scales must be a contiguous CUDA uint8 buffer of >= mx_scale_bytes = {need} bytes")
    _check(lib.mx_quantize(x.data_ptr(), rows, k, _ld(x), codes.data_ptr(), _ld(codes), scales.data_ptr(),
                           _opt_ptr(nonfinite_flag, "nonfinite_flag", torch.int32), _stream(stream)), "mx_quantize")
    return codes, scales


def fp8_mx_gemm(a: torch.Tensor, a_scales: torch.Tensor, b: torch.Tensor, b_scales: torch.Tensor,
                out_dtype: torch.dtype = torch.bfloat16, out: torch.Tensor | None = None, stream=None):
    """MXFP8 linear Y = X W^T with the block-scaled tcgen05 MMA (scales from mx_quantize)."""
    _cuda2d(a, "a", torch.uint8)
    _cuda2d(b, "b", torch.uint8)
    m, k = a.shape
    n = b.shape[0]
    if b.shape[1] != k:
        raise Fp8qError("fp8_mx_gemm: inner dimensions differ")
    out = _out(out, m, n, out_dtype, a.device)
    lib = load_library()
    for t, rows, nm in ((a_scales, m, "a_scales"), (b_scales, n, "b_scales")):
        need = int(lib.mx_scale_bytes(rows, k))
        if not (t.is_cuda and t.dtype == torch.uint8 and t.is_contiguous() and t.numel() >= need):
            raise Fp8qError(f"{nm} must be a contiguous CUDA uint8 buffer of >= mx_scale_bytes = {need} bytes")
    _check(load_library().fp8_mx_gemm(a.data_ptr(), _ld(a), a_scales.data_ptr(), b.data_ptr(), _ld(b),
                                      b_scales.data_ptr(), out.data_ptr(), _ld(out),
                                      FP8Q_OUT_F32 if out_dtype == torch.float32 else FP8Q_OUT_BF16, m, n, k,
                                      _stream(stream)), "fp8_mx_gemm")
    return out


def mx_scales_logical(native, rows: int, k: int):
    """Native scale bytes -> the logical [rows, k/32] array (for tests and inspection)."""
    import numpy as np
    nat = np.asarray(native.cpu().numpy() if hasattr(native, "cpu") else native, dtype=np.uint8)
    kb = k // 128
    blocks = (rows + 127) // 128
    t = nat[: blocks * kb * 512].reshape(blocks, kb, 128, 4)      # [rb][kb][r%128][j%4]
    t = t.transpose(0, 2, 1, 3).reshape(blocks * 128, kb * 4)     # [r][j]
    return t[:rows]
