"""Seeded FP8 E4M3 inputs for the FP8 expert GEMM (reading R15) — input generation only.

The same counter-based hash as ``workloads.counter_values`` gives an integer ``c`` per element
("normal": Irwin-Hall c in [-254, 254]; "int": c in {-4..4}).  The element is the FP8 E4M3 code
of ``c * 2**-shift`` with ``|c|`` truncated toward zero to 4 significant bits (sign | exponent
field | 3 mantissa bits, built with integer operations only), so the numpy twin (oracle side) and
the torch twin (device side) produce identical BYTES and no floating-point rounding step exists.
"normal" uses shift 6 (|value| <= 3.75, std ~1.1) for X and W alike; the W ~ N(0,1)/sqrt(H)
magnitude of the bf16 recipe is carried by the per-expert fp32 scale 2**-w_scale_exp(H)
(``w_scale``), the way FP8 weights are stored with a per-tensor scale.  "int" uses shift 0.
"full": the code is the low byte of h itself — every finite E4M3 value, subnormals and
+-448 included, exponents spread over the whole format (the two NaN codes 0x7F / 0xFF map to
+-448, 0x7E / 0xFE); products and sums then need fp32 rounding (``w_scale``: 2**-(w_scale_exp(H)+8)).
"""
from __future__ import annotations

import numpy as np

from .workloads import STREAM_W, STREAM_X, _M32, _fmix32_np, _key, w_scale_exp

SHIFT = {"normal": 6, "int": 0, "full": 0}


def _c_np(seed: int, stream: int, idx: np.ndarray, mode: str) -> np.ndarray:
    h = _fmix32_np((np.asarray(idx, dtype=np.int64).astype(np.uint64) ^ np.uint64(_key(seed, stream))).astype(np.uint32))
    if mode == "int":
        return (h % np.uint32(9)).astype(np.int32) - 4
    if mode == "normal":
        c = ((h & np.uint32(127)) + ((h >> np.uint32(8)) & np.uint32(127))
             + ((h >> np.uint32(16)) & np.uint32(127)) + ((h >> np.uint32(24)) & np.uint32(127)))
        return c.astype(np.int32) - 254
    raise ValueError(mode)


def encode_np(c: np.ndarray, shift: int) -> np.ndarray:
    """E4M3 codes of c * 2**-shift, |c| < 256 truncated to 4 significant bits (integer ops)."""
    c = np.asarray(c, dtype=np.int32)
    a = np.abs(c)
    b = np.zeros_like(a)
    for i in range(1, 8):
        b += (a >= (1 << i)).astype(np.int32)
    mant = np.where(b >= 3, a >> np.maximum(b - 3, 0), a << np.maximum(3 - b, 0)) & 7
    field = b - shift + 7
    if np.any((a > 0) & ((field < 1) | (field > 15))):
        raise ValueError("value outside the E4M3 normal range")
    code = ((c < 0).astype(np.int32) << 7) | (field << 3) | mant
    return np.where(a == 0, 0, code).astype(np.uint8)


def encode_torch(c, shift: int):
    import torch

    a = c.abs()
    b = torch.zeros_like(a)
    for i in range(1, 8):
        b += (a >= (1 << i)).to(a.dtype)
    mant = torch.where(b >= 3, a >> (b - 3).clamp(min=0), a << (3 - b).clamp(min=0)) & 7
    field = b - shift + 7
    code = ((c < 0).to(a.dtype) << 7) | (field << 3) | mant
    return torch.where(a == 0, torch.zeros_like(code), code).to(torch.uint8)


def _codes_np(seed, stream, idx, mode):
    if mode == "full":
        h = _fmix32_np((np.asarray(idx, dtype=np.int64).astype(np.uint64)
                        ^ np.uint64(_key(seed, stream))).astype(np.uint32))
        b = (h & np.uint32(255)).astype(np.uint8)
        return np.where((b & np.uint8(127)) == 127, b ^ np.uint8(1), b).astype(np.uint8)
    return encode_np(_c_np(seed, stream, idx, mode), SHIFT[mode])


def make_x_fp8(seed: int, T: int, H: int, mode: str = "normal") -> np.ndarray:
    """X [T, H] E4M3 codes (uint8)."""
    return _codes_np(seed, STREAM_X, np.arange(T * H, dtype=np.int64), mode).reshape(T, H)


def make_w_fp8(seed: int, E: int, H: int, N: int, mode: str = "normal") -> np.ndarray:
    """W [E, H, N] E4M3 codes (uint8)."""
    return _codes_np(seed, STREAM_W, np.arange(E * H * N, dtype=np.int64), mode).reshape(E, H, N)


def x_fp8_rows(seed: int, T: int, H: int, rows, mode: str = "normal") -> np.ndarray:
    rows = np.asarray(rows, dtype=np.int64)
    return _codes_np(seed, STREAM_X, rows[:, None] * H + np.arange(H, dtype=np.int64)[None, :], mode)


def w_fp8_columns(seed: int, E: int, H: int, N: int, e: int, cols, mode: str = "normal") -> np.ndarray:
    """W[e][:, cols] codes [H, len(cols)] without materialising W."""
    cols = np.asarray(cols, dtype=np.int64)
    return _codes_np(seed, STREAM_W, e * H * N + np.arange(H, dtype=np.int64)[:, None] * N + cols[None, :], mode)


def w_scale(E: int, H: int, mode: str = "normal") -> np.ndarray:
    """Per-expert fp32 scale paired with make_w_fp8: 2**-w_scale_exp(H) ("normal"), 1 ("int")."""
    if mode == "full":
        return np.full(E, 2.0 ** -(w_scale_exp(H) + 8), dtype=np.float32)
    return np.full(E, 2.0 ** -w_scale_exp(H) if mode == "normal" else 1.0, dtype=np.float32)


def _codes_torch(seed, stream, start, count, mode, device):
    import torch

    idx = torch.arange(start, start + count, dtype=torch.int64, device=device)
    h = (idx ^ _key(seed, stream)) & _M32
    h = h ^ (h >> 16)
    h = (h * 0x85EBCA6B) & _M32
    h = h ^ (h >> 13)
    h = (h * 0xC2B2AE35) & _M32
    h = h ^ (h >> 16)
    if mode == "int":
        c = (h % 9) - 4
    elif mode == "normal":
        c = (h & 127) + ((h >> 8) & 127) + ((h >> 16) & 127) + ((h >> 24) & 127) - 254
    elif mode == "full":
        b = h & 255
        return torch.where((b & 127) == 127, b ^ 1, b).to(torch.uint8)
    else:
        raise ValueError(mode)
    return encode_torch(c.to(torch.int32), SHIFT[mode])


def make_x_fp8_torch(seed: int, T: int, H: int, mode: str = "normal", device="cpu", row0: int = 0):
    """Rows [row0, row0 + T) of X (one expert-parallel rank's tokens when row0 > 0)."""
    return _codes_torch(seed, STREAM_X, row0 * H, T * H, mode, device).reshape(T, H)


def make_w_fp8_torch(seed: int, E: int, H: int, N: int, mode: str = "normal", device="cpu", chunk=1 << 26,
                     experts: range | None = None):
    """W [E, H, N] codes, or the contiguous expert range `experts` of it (one EP rank's share)."""
    import torch

    ex = range(E) if experts is None else experts
    start, total = ex.start * H * N, len(ex) * H * N
    out = torch.empty(total, dtype=torch.uint8, device=device)
    for s in range(0, total, chunk):
        n = min(chunk, total - s)
        out[s:s + n] = _codes_torch(seed, STREAM_W, start + s, n, mode, device)
    return out.reshape(len(ex), H, N)
