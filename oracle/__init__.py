"""CPU oracle for the FP8 W8A8 hot path (arXiv 2601.18150, §2.1.1 Eq. (1)).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this package.
The product package ``paper_2601_18150_b200`` never imports it, and this package
imports nothing from the product package: the two share no code.

Every function is a thin ctypes marshaller around ``fp8q_oracle.c`` (plain C,
binary32 where the DESIGN.md readings fix binary32, binary64 for the GEMM), except the NEXT-2
producers, which are plain Python (integers, fractions, decimal, numpy binary32) in
``producers.py``; the arithmetic and its citations live in those files.  Parity pins: ``tests/test_oracle_*.py``.
No function here is "parity unpinned" (see DESIGN.md §3.3 for the pin of each one).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from . import producers as _producers

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fp8q_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

GCC_FLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    """Compile fp8q_oracle.c with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            I64 = ctypes.c_int64
            lib.oracle_e4m3_decode.argtypes = [ctypes.c_uint8]
            lib.oracle_e4m3_decode.restype = ctypes.c_double
            lib.oracle_e4m3_encode.argtypes = [ctypes.c_float]
            lib.oracle_e4m3_encode.restype = ctypes.c_uint8
            lib.oracle_e4m3_encode_array.argtypes = [P, I64, P, ctypes.c_int]
            lib.oracle_e4m3_encode_array.restype = None
            lib.oracle_block_scale.argtypes = [ctypes.c_float]
            lib.oracle_block_scale.restype = ctypes.c_float
            lib.oracle_quantize_element.argtypes = [ctypes.c_float, ctypes.c_float]
            lib.oracle_quantize_element.restype = ctypes.c_uint8
            lib.oracle_quantize_weight_blockwise.argtypes = [P, I64, I64, I64, P, I64, P, I64, ctypes.c_int]
            lib.oracle_quantize_weight_blockwise.restype = ctypes.c_int
            lib.oracle_quantize_act_per_token_group.argtypes = [P, I64, I64, I64, P, I64, P, ctypes.c_int]
            lib.oracle_quantize_act_per_token_group.restype = ctypes.c_int
            lib.oracle_gemm_rows.argtypes = [P, I64, P, I64, P, I64, P, I64, I64, I64, P, I64, P, ctypes.c_int]
            lib.oracle_gemm_rows.restype = ctypes.c_int
            lib.oracle_f64_to_bf16.argtypes = [ctypes.c_double]
            lib.oracle_f64_to_bf16.restype = ctypes.c_uint16
            lib.oracle_kv_amax.argtypes = [P, I64, I64, I64, P]
            lib.oracle_kv_amax.restype = ctypes.c_int
            lib.oracle_kv_quantize_append.argtypes = [P, I64, I64, I64, ctypes.c_float, P, P, I64]
            lib.oracle_kv_quantize_append.restype = ctypes.c_int64
            lib.oracle_mx_exponent.argtypes = [ctypes.c_float]
            lib.oracle_mx_exponent.restype = ctypes.c_int
            lib.oracle_mx_quantize.argtypes = [P, I64, I64, I64, P, P]
            lib.oracle_mx_quantize.restype = ctypes.c_int
            lib.oracle_mx_gemm_rows.argtypes = [P, P, P, P, I64, I64, P, I64, P]
            lib.oracle_mx_gemm_rows.restype = ctypes.c_int
            _lib = lib
    return _lib


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


class OracleError(ValueError):
    pass


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------- scalars (O1, O2, O4, O5)
def e4m3_decode(code: int) -> float:
    """O1."""
    return _load().oracle_e4m3_decode(code)


def e4m3_decode_table() -> np.ndarray:
    """All 256 codes decoded, float64 (NaN at 0x7F, 0xFF)."""
    lib = _load()
    return np.array([lib.oracle_e4m3_decode(c) for c in range(256)], dtype=np.float64)


def e4m3_encode(q: float) -> int:
    """O2: nearest E4M3, ties-to-even code, saturating, sign kept."""
    return _load().oracle_e4m3_encode(float(np.float32(q)))


def e4m3_encode_array(q: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    """O2 applied to every element of a float32 array (the same scalar function)."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    out = np.empty(q.shape, dtype=np.uint8)
    _load().oracle_e4m3_encode_array(_ptr(q), q.size, _ptr(out), nthreads or default_threads())
    return out


def block_scale(amax: float) -> np.float32:
    """O4: RN32(amax/448), 0 -> 1."""
    return np.float32(_load().oracle_block_scale(float(np.float32(amax))))


def quantize_element(x: float, s: float) -> int:
    """O5: O2(RN32(x/s)) (Eq. (1))."""
    return _load().oracle_quantize_element(float(np.float32(x)), float(np.float32(s)))


# ---------------------------------------------------------------- tensors
def _as_bf16_bits(x: np.ndarray) -> np.ndarray:
    if x.dtype != np.uint16:
        raise TypeError("oracle inputs are BF16 bit patterns (numpy uint16)")
    return np.ascontiguousarray(x)


def quantize_weight_blockwise(w_bits: np.ndarray, nthreads: int | None = None):
    """O3-O6 on a BF16 [n, k] matrix (uint16 bits).  Returns (codes u8 [n,k], scales f32
    [ceil(n/128), ceil(k/128)]).  Raises OracleError on NaN/Inf input."""
    w = _as_bf16_bits(w_bits)
    n, k = w.shape
    codes = np.empty((n, k), dtype=np.uint8)
    nbn, nbk = (n + 127) // 128, (k + 127) // 128
    scales = np.empty((nbn, nbk), dtype=np.float32)
    rc = _load().oracle_quantize_weight_blockwise(
        _ptr(w), n, k, k, _ptr(codes), k, _ptr(scales), nbk, nthreads or default_threads())
    if rc == 1:
        raise OracleError("non-finite input")
    if rc != 0:
        raise OracleError(f"invalid arguments (rc={rc})")
    return codes, scales


def quantize_act_per_token_group(x_bits: np.ndarray, nthreads: int | None = None):
    """Per token, per 128-channel group.  Returns (codes u8 [m,k],
    scales f32 [m, k/128]) -- the LOGICAL scale layout; the C-ABI stores its transpose."""
    x = _as_bf16_bits(x_bits)
    m, k = x.shape
    if k % 128:
        raise OracleError("k must be a multiple of 128")
    codes = np.empty((m, k), dtype=np.uint8)
    scales = np.empty((m, k // 128), dtype=np.float32)
    rc = _load().oracle_quantize_act_per_token_group(
        _ptr(x), m, k, k, _ptr(codes), k, _ptr(scales), nthreads or default_threads())
    if rc == 1:
        raise OracleError("non-finite input")
    if rc != 0:
        raise OracleError(f"invalid arguments (rc={rc})")
    return codes, scales


def gemm_rows(a_codes: np.ndarray, a_scales: np.ndarray, b_codes: np.ndarray,
              b_scales: np.ndarray, rows=None, nthreads: int | None = None) -> np.ndarray:
    """O7: fp64 reference rows.  a_codes u8 [m,k]; a_scales f32 LOGICAL [m,k/128];
    b_codes u8 [n,k]; b_scales f32 [ceil(n/128), k/128].  Returns float64 [len(rows), n]."""
    a = np.ascontiguousarray(a_codes, dtype=np.uint8)
    sa = np.ascontiguousarray(a_scales, dtype=np.float32)
    b = np.ascontiguousarray(b_codes, dtype=np.uint8)
    sb = np.ascontiguousarray(b_scales, dtype=np.float32)
    m, k = a.shape
    n, kb = b.shape
    if kb != k or k % 128:
        raise OracleError("shape mismatch")
    if sa.shape != (m, k // 128) or sb.shape != ((n + 127) // 128, k // 128):
        raise OracleError("scale shape mismatch")
    if rows is None:
        rows = np.arange(m, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    if rows.size and (rows.min() < 0 or rows.max() >= m):
        raise OracleError("row index out of range")
    out = np.empty((rows.size, n), dtype=np.float64)
    rc = _load().oracle_gemm_rows(_ptr(a), k, _ptr(sa), k // 128, _ptr(b), k, _ptr(sb), k // 128,
                                  n, k, _ptr(rows), rows.size, _ptr(out),
                                  nthreads or default_threads())
    if rc != 0:
        raise OracleError(f"invalid arguments (rc={rc})")
    return out


def gemm_grouped_rows(a_codes, a_scales, b_codes, b_scales, offsets, rows=None, nthreads=None):
    """O8: O7 per group.  b_codes u8 [G,n,k], b_scales f32 [G, ceil(n/128), k/128];
    group g owns A rows [offsets[g], offsets[g+1]).  Returns float64 [len(rows), n]."""
    offsets = np.asarray(offsets, dtype=np.int64)
    m = a_codes.shape[0]
    if rows is None:
        rows = np.arange(m, dtype=np.int64)
    rows = np.asarray(rows, dtype=np.int64)
    n = b_codes.shape[1]
    out = np.empty((rows.size, n), dtype=np.float64)
    grp = np.searchsorted(offsets, rows, side="right") - 1
    for g in np.unique(grp):
        sel = np.nonzero(grp == g)[0]
        out[sel] = gemm_rows(a_codes, a_scales, b_codes[g], b_scales[g], rows[sel], nthreads)
    return out


# ---------------------------------------------------------------- NEXT-2 producers
def f64_to_bf16(d: float) -> int:
    """binary64 -> BF16 bits, round to nearest even (no double rounding)."""
    return int(_load().oracle_f64_to_bf16(float(d)))


def rmsnorm_bf16(x_bits: np.ndarray, gamma_bits: np.ndarray, eps: float) -> np.ndarray:
    """NEXT-2 RMSNorm (reading N2; oracle/producers.py): Qwen3RMSNorm with every
    binary32 step correctly rounded and the sum of squares exact, rounded to BF16 twice."""
    x = _as_bf16_bits(x_bits)
    g = _as_bf16_bits(gamma_bits)
    m, k = x.shape
    if g.shape != (k,):
        raise OracleError("gamma must have shape [k]")
    return _producers.rmsnorm_bf16(x, g, eps)


def silu_mul_bf16(gate_up_bits: np.ndarray) -> np.ndarray:
    """NEXT-2 SiLU-mul (reading N2): y = RN_BF16(RN32(RN_BF16(silu(gate)) * up)) for
    gate_up = [gate | up] (each [m, I]), silu correctly rounded from its real value."""
    gu = _as_bf16_bits(gate_up_bits)
    m, k2 = gu.shape
    if k2 % 2:
        raise OracleError("gate_up must have an even number of columns")
    return _producers.silu_mul_bf16(gu)


def silu_bf16_table() -> np.ndarray:
    """RN_BF16(silu(g)) for every BF16 bit pattern g (65,536 entries; NaN for non-finite g)."""
    return _producers.silu_bf16_table()


def rmsnorm_quantize(x_bits, gamma_bits, eps, nthreads=None):
    """NEXT-2 definition: per-token-group quantization (O3-O6) of the BF16 RMSNorm output."""
    y = rmsnorm_bf16(x_bits, gamma_bits, eps)
    return (y,) + quantize_act_per_token_group(y, nthreads)


def silu_mul_quantize(gate_up_bits, nthreads=None):
    """NEXT-2 definition: per-token-group quantization of the BF16 SiLU(gate) * up output."""
    y = silu_mul_bf16(gate_up_bits)
    return (y,) + quantize_act_per_token_group(y, nthreads)


# ---------------------------------------------------------------- NEXT-3 FP8 KV cache
def kv_amax(x_bits: np.ndarray) -> np.float32:
    """K1: exact max |x| over a BF16 [rows, cols] tensor.  Raises on NaN/Inf."""
    x = _as_bf16_bits(x_bits)
    x2 = x.reshape(x.shape[0], -1) if x.ndim > 1 else x.reshape(1, -1)
    out = np.zeros(1, dtype=np.float32)
    if _load().oracle_kv_amax(_ptr(x2), x2.shape[0], x2.shape[1], x2.shape[1], _ptr(out)) != 0:
        raise OracleError("non-finite input")
    return out[0]


def kv_scale(amax: float) -> np.float32:
    """K1: the layer's scalar K/V scale = O4(amax) = RN32(amax/448), 0 -> 1."""
    return block_scale(amax)


def kv_calibrate(batches) -> np.float32:
    """K1 over several calibration batches (trainer side: a subset of prompts + responses):
    the scale of the max of the per-batch amax values."""
    return kv_scale(max(float(kv_amax(b)) for b in batches))


def kv_quantize_append(x_bits: np.ndarray, scale: float, cache: np.ndarray, slots=None) -> int:
    """K2-K4: codes of x's rows (scalar scale) into cache rows slots[r] (identity if None);
    returns the saturated-element count (|RN32(x/s)| >= 464)."""
    x = _as_bf16_bits(x_bits)
    rows, cols = x.shape
    if cache.dtype != np.uint8 or not cache.flags.c_contiguous or cache.shape[1] < cols:
        raise OracleError("cache must be a C-contiguous uint8 [slots, >= cols] array")
    sl = None
    if slots is not None:
        sl = np.ascontiguousarray(slots, dtype=np.int32)
        if sl.shape != (rows,) or (rows and (sl.min() < 0 or sl.max() >= cache.shape[0])):
            raise OracleError("slot out of range")
    elif rows > cache.shape[0]:
        raise OracleError("cache too small")
    return int(_load().oracle_kv_quantize_append(_ptr(x), rows, cols, cols, float(np.float32(scale)),
                                                 _ptr(sl) if sl is not None else None, _ptr(cache),
                                                 cache.shape[1]))


# ---------------------------------------------------------------- NEXT-4 MXFP8 variant
def mx_exponent(amax: float) -> int:
    """X2: the smallest e (>= -127) with 448 * 2^e >= amax; amax == 0 -> 0."""
    return int(_load().oracle_mx_exponent(float(np.float32(amax))))


def mx_quantize(x_bits: np.ndarray):
    """X1-X3 on a BF16 [rows, cols] matrix: codes u8 [rows, cols] and E8M0 scale bytes
    [rows, ceil(cols/32)] (logical layout)."""
    x = _as_bf16_bits(x_bits)
    rows, cols = x.shape
    codes = np.empty((rows, cols), np.uint8)
    sf = np.empty((rows, (cols + 31) // 32), np.uint8)
    if _load().oracle_mx_quantize(_ptr(x), rows, cols, cols, _ptr(codes), _ptr(sf)) != 0:
        raise OracleError("non-finite input")
    return codes, sf


def mx_gemm_rows(a, sfa, b, sfb, rows=None) -> np.ndarray:
    """fp64 Y[m, n] = sum_k dec(a) 2^(sfa-127) dec(b) 2^(sfb-127) for the listed rows."""
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    sfa = np.ascontiguousarray(sfa, np.uint8)
    sfb = np.ascontiguousarray(sfb, np.uint8)
    m, k = a.shape
    n = b.shape[0]
    if b.shape[1] != k or sfa.shape != (m, (k + 31) // 32) or sfb.shape != (n, (k + 31) // 32):
        raise OracleError("shape mismatch")
    rows = np.arange(m, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    out = np.empty((rows.size, n), np.float64)
    _load().oracle_mx_gemm_rows(_ptr(a), _ptr(sfa), _ptr(b), _ptr(sfb), n, k, _ptr(rows), rows.size, _ptr(out))
    return out
