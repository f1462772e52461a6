"""FP8 E4M3 expert GEMM — fp64 oracle.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Not in the paper (which runs bf16): the FP8 variant is SURVEY §8(f) row 4
("optionally FP8"), reading R15.  What it computes:
* e4m3_value: the OCP 8-bit floating point E4M3 format written out — sign bit s, exponent field
  e (4 bits, bias 7), mantissa field m (3 bits): e > 0 -> (-1)^s 2^(e-7) (1 + m/8);
  e = 0 -> (-1)^s 2^-6 (m/8) (subnormal); e = 15 and m = 7 -> NaN (the format has no infinities).
* expert_gemm_fp8: Y[row_off[e] + r, :] = scale[e] * (x(X[token_idx_e[r], :]) @ x(W[e])), the
  per-expert product of P:100-101 on the decoded values, in fp64 (numpy matmul per expert is the
  library primitive), then the per-expert scale (1 when scale is None).
"""
from __future__ import annotations

import math

import numpy as np

from . import moe


def e4m3_value(code: int) -> float:
    s = (code >> 7) & 1
    e = (code >> 3) & 15
    m = code & 7
    if e == 15 and m == 7:
        return math.nan
    mag = 2.0 ** (e - 7) * (1.0 + m / 8.0) if e > 0 else 2.0 ** -6 * (m / 8.0)
    return -mag if s else mag


_TABLE = np.array([e4m3_value(c) for c in range(256)], dtype=np.float64)


def e4m3_decode(codes: np.ndarray) -> np.ndarray:
    """float64 values of E4M3 codes (uint8 array of any shape)."""
    return _TABLE[np.asarray(codes, dtype=np.uint8)]


def expert_gemm_fp8(X_codes, W_codes, token_idx, row_off, scale=None) -> np.ndarray:
    """[sum m_e, N] fp64: scale[e] * (X_e @ W_e) on decoded E4M3 values."""
    Y = moe.expert_gemm(e4m3_decode(X_codes), e4m3_decode(W_codes), token_idx, row_off)
    if scale is not None:
        row_off = np.asarray(row_off)
        for e in range(len(row_off) - 1):
            Y[row_off[e]:row_off[e + 1]] *= float(scale[e])
    return Y


def expert_gemm_fp8_entries(x_rows_codes, w_cols_codes, scale_e: float = 1.0) -> np.ndarray:
    """Sampled entries: scale_e * (x_rows @ w_cols) on decoded values (rows x cols, fp64)."""
    return scale_e * (e4m3_decode(x_rows_codes) @ e4m3_decode(w_cols_codes))
