"""Test-side helpers: moving seeded host inputs to the device and bringing CUDA results back
into the oracle's logical layouts.  No arithmetic of the method lives here."""
from __future__ import annotations

import numpy as np
import torch


def to_dev_bf16(bits: np.ndarray, device="cuda") -> torch.Tensor:
    """uint16 BF16 bit patterns (host) -> torch.bfloat16 on the device, same bytes."""
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)
    return t.to(device)


def to_host_u8(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.uint8, copy=False)


def to_host_f32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.float32, copy=False)


def act_scales_logical(scales_mn: torch.Tensor, m: int) -> np.ndarray:
    """MN-major [k/128, ld_s] device scales -> logical [m, k/128] host array."""
    return np.ascontiguousarray(to_host_f32(scales_mn)[:, :m].T)


def act_scales_mn_from_logical(sl: np.ndarray, ld: int, device="cuda") -> torch.Tensor:
    m, g = sl.shape
    out = np.zeros((g, ld), dtype=np.float32)
    out[:, :m] = sl.T
    return torch.from_numpy(out).to(device)


def rel_frobenius(y: np.ndarray, ref: np.ndarray) -> float:
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    num = np.linalg.norm(np.asarray(y, dtype=np.float64) - ref)
    if den == 0:
        return 0.0 if num == 0 else float("inf")
    return float(num / den)


def bf16_rne_of_f32(x: torch.Tensor) -> torch.Tensor:
    """torch's float32 -> bfloat16 cast (round to nearest even), for the BF16-output check."""
    return x.to(torch.bfloat16)
