"""Full MoE FFN layer around the expert GEMM — fp64 oracle.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions followed:
* the MoE layer "first selects the subset of experts for a token, then computes the
  products of the token tensor and each selected expert weight tensor, and finally sums
  them up as the output": out[t] = sum_j w[t, j] * FFN_{e(t, j)}(x_t) over the
  token's top-k slots j with e(t, j) >= 0 (negative ids are masked slots, R13);
* the expert FFN of the Mixtral shape BASELINE.json names (not given by the paper, which
  stops at the products; reading R14): FFN_e(x) = (silu(x W_gate[e]) * (x W_up[e]))
  W_down[e], silu(z) = z / (1 + exp(-z)), '*' elementwise;
* the intermediate activation h = silu(x W_gate) * (x W_up) is stored in bf16 between the
  two GEMMs (R14: the CUDA path keeps activations in bf16); with ``h_bf16=False`` it stays
  fp64.  Rounding is round-to-nearest-even from the fp32 value of h.
"""
from __future__ import annotations

import math

import numpy as np


def silu(z):
    """silu(z) = z * sigmoid(z) = z / (1 + exp(-z)), evaluated in fp64 without overflow."""
    z = np.asarray(z, dtype=np.float64)
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = z[pos] / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])                       # z < 0: z * e^z / (1 + e^z)
    out[~pos] = z[~pos] * ez / (1.0 + ez)
    return out


def round_bf16(x):
    """fp64 -> fp32 (RNE) -> bf16 (RNE on the fp32 bit pattern), returned as fp64."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def expert_ffn(x, W_gate, W_up, W_down, e: int, h_bf16: bool = True):
    """FFN of expert e for the rows of x (R14), fp64."""
    x = np.asarray(x, dtype=np.float64)
    g = x @ np.asarray(W_gate[e], dtype=np.float64)
    u = x @ np.asarray(W_up[e], dtype=np.float64)
    h = silu(g) * u
    if h_bf16:
        h = round_bf16(h)
    return h @ np.asarray(W_down[e], dtype=np.float64)


def moe_ffn(X, W_gate, W_up, W_down, topk_ids, topk_w, h_bf16: bool = True):
    """out[t] = sum_j topk_w[t, j] * expert_ffn(X[t], e = topk_ids[t, j]) (R14)."""
    topk_ids = np.asarray(topk_ids)
    T, k = topk_ids.shape
    out = np.zeros((T, np.asarray(W_down).shape[2]))
    for t in range(T):
        for j in range(k):
            e = int(topk_ids[t, j])
            if e < 0:
                continue
            out[t] += float(topk_w[t, j]) * expert_ffn(np.asarray(X)[t:t + 1], W_gate, W_up, W_down, e, h_bf16)[0]
    return out


def swiglu_rows(X, W_gate, W_up, token_idx, row_off, h_bf16: bool = True):
    """The gated first GEMM in the expert GEMM's CSR row order: row row_off[e] + r holds
    h for token token_idx[row_off[e] + r] under expert e (the layout moe_gemm_swiglu writes)."""
    E = len(row_off) - 1
    out = np.zeros((int(row_off[-1]), np.asarray(W_gate).shape[2]))
    for e in range(E):
        a, b = int(row_off[e]), int(row_off[e + 1])
        if b > a:
            x = np.asarray(X, dtype=np.float64)[np.asarray(token_idx[a:b])]
            h = silu(x @ np.asarray(W_gate[e], dtype=np.float64)) * (x @ np.asarray(W_up[e], dtype=np.float64))
            out[a:b] = round_bf16(h) if h_bf16 else h
    return out


def sigmoid_scalar(z: float) -> float:
    """Reference scalar for pins: 1 / (1 + e^-z)."""
    return 1.0 / (1.0 + math.exp(-z))


def moe_ffn_entries(x_row, w_gate_e, w_up_e, w_down_cols, topk_ids, topk_w, tokens, cols, h_bf16: bool = True):
    """Sampled entries of moe_ffn: out[i, c] = sum_j topk_w[t_i, j] * expert_ffn(X[t_i], e(t_i, j))[cols[c]]
    (R14), the same definition with inputs fetched on demand so a full-size layer can be checked
    without materialising every weight on the host: x_row(t) -> [H], w_gate_e(e) / w_up_e(e) -> [H, I],
    w_down_cols(e, cols) -> [I, len(cols)].  Experts are visited one at a time (one expert's
    weights in memory)."""
    topk_ids = np.asarray(topk_ids)
    tokens = [int(t) for t in tokens]
    out = np.zeros((len(tokens), len(cols)))
    xs = {t: np.asarray(x_row(t), dtype=np.float64)[None, :] for t in set(tokens)}
    experts = sorted({int(topk_ids[t, j]) for t in tokens for j in range(topk_ids.shape[1]) if topk_ids[t, j] >= 0})
    for e in experts:
        g_w, u_w = np.asarray(w_gate_e(e), dtype=np.float64), np.asarray(w_up_e(e), dtype=np.float64)
        d_w = np.asarray(w_down_cols(e, cols), dtype=np.float64)
        for i, t in enumerate(tokens):
            for j in range(topk_ids.shape[1]):
                if int(topk_ids[t, j]) != e:
                    continue
                h = silu(xs[t] @ g_w) * (xs[t] @ u_w)
                if h_bf16:
                    h = round_bf16(h)
                out[i] += float(topk_w[t, j]) * (h @ d_w)[0]
        del g_w, u_w, d_w
    return out
