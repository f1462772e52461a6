"""Pins for oracle/ffn.py (the MoE FFN layer oracle; R14)."""
import math

import numpy as np
import pytest
import torch

from oracle import ffn


def test_silu_values_and_identities():
    # silu(z) = z / (1 + e^-z): printed values at 0, +-1, and the exact identity silu(z) - silu(-z) = z
    assert ffn.silu(np.array([0.0]))[0] == 0.0
    assert ffn.silu(np.array([1.0]))[0] == pytest.approx(0.7310585786300049, abs=1e-16)
    assert ffn.silu(np.array([-1.0]))[0] == pytest.approx(-0.2689414213699951, abs=1e-16)
    z = np.linspace(-30, 30, 1201)
    assert np.allclose(ffn.silu(z) - ffn.silu(-z), z, atol=1e-13)
    assert ffn.silu(np.array([40.0]))[0] == 40.0                          # sigmoid(40) rounds to 1
    assert np.isfinite(ffn.silu(np.array([-800.0, 800.0]))).all()         # no overflow
    assert ffn.silu(np.array([-800.0]))[0] == 0.0
    for v in (-3.5, -0.25, 0.5, 2.0):
        assert ffn.silu(np.array([v]))[0] == pytest.approx(v * ffn.sigmoid_scalar(v), rel=1e-15)


def test_round_bf16_ties_and_library():
    # spacing at 1 is 2^-7: halfway points tie to the even mantissa
    assert ffn.round_bf16(np.array([1.0 + 2 ** -8]))[0] == 1.0
    assert ffn.round_bf16(np.array([1.0 + 3 * 2 ** -8]))[0] == 1.0 + 2 ** -6
    assert ffn.round_bf16(np.array([1.0 + 2 ** -8 + 2 ** -20]))[0] == 1.0 + 2 ** -7
    rng = np.random.default_rng(0)
    x = rng.standard_normal(10000) * 10.0 ** rng.integers(-5, 5, 10000)
    ref = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).double().numpy()   # library RNE
    assert np.array_equal(ffn.round_bf16(x), ref)


def _ids_w(T, k, E, seed):
    rng = np.random.default_rng(seed)
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int64)
    w = rng.random((T, k))
    return ids, w


def test_identity_weights_closed_form():
    """W_gate = W_up = W_down = I, one slot of weight 1: out = bf16(silu(x) * x) elementwise."""
    T, H, E = 6, 5, 3
    rng = np.random.default_rng(1)
    X = rng.standard_normal((T, H))
    I = np.stack([np.eye(H)] * E)
    ids = rng.integers(0, E, size=(T, 1))
    out = ffn.moe_ffn(X, I, I, I, ids, np.ones((T, 1)))
    assert np.array_equal(out, ffn.round_bf16(ffn.silu(X) * X))
    out64 = ffn.moe_ffn(X, I, I, I, ids, np.ones((T, 1)), h_bf16=False)
    assert np.allclose(out64, ffn.silu(X) * X, rtol=0, atol=1e-15)


def test_selection_matrices_non_square():
    """H=3, I=5, Hout=2 selection matrices: g_i = x[i mod 3], u_i = sum(x), out_c = h_c — any
    transposed operand or swapped gate/up breaks the shapes or the values."""
    T, H, I, Ho, E = 4, 3, 5, 2, 2
    rng = np.random.default_rng(2)
    X = rng.standard_normal((T, H))
    Wg = np.zeros((E, H, I))
    for i in range(I):
        Wg[:, i % H, i] = 1.0
    Wu = np.ones((E, H, I))
    Wd = np.zeros((E, I, Ho))
    for c in range(Ho):
        Wd[:, c, c] = 1.0
    ids = np.zeros((T, 1), dtype=np.int64)
    out = ffn.moe_ffn(X, Wg, Wu, Wd, ids, np.ones((T, 1)), h_bf16=False)
    for t in range(T):
        s = X[t].sum()
        for c in range(Ho):
            sg = X[t, c % H] / (1.0 + math.exp(-X[t, c % H]))
            assert out[t, c] == pytest.approx(sg * s, rel=1e-14, abs=1e-14)


def test_combine_cancellation_linearity_and_masking():
    T, k, E, H, I, Ho = 5, 2, 4, 6, 7, 3
    rng = np.random.default_rng(3)
    X = rng.standard_normal((T, H))
    Wg, Wu, Wd = rng.standard_normal((E, H, I)), rng.standard_normal((E, H, I)), rng.standard_normal((E, I, Ho))
    # experts 0 and 1 identical except W_down[1] = -W_down[0]: equal weights cancel exactly
    Wg[1], Wu[1], Wd[1] = Wg[0], Wu[0], -Wd[0]
    ids = np.tile(np.array([[0, 1]]), (T, 1))
    assert np.array_equal(ffn.moe_ffn(X, Wg, Wu, Wd, ids, np.full((T, k), 0.5)), np.zeros((T, Ho)))
    ids, w = _ids_w(T, k, E, 4)
    a = ffn.moe_ffn(X, Wg, Wu, Wd, ids, w)
    assert np.allclose(ffn.moe_ffn(X, Wg, Wu, Wd, ids, 2 * w), 2 * a, rtol=1e-14, atol=1e-13)
    masked = ids.copy()
    masked[:, 1] = -1
    assert np.array_equal(ffn.moe_ffn(X, Wg, Wu, Wd, masked, w), ffn.moe_ffn(X, Wg, Wu, Wd, ids[:, :1], w[:, :1]))


def test_swiglu_rows_layout_matches_layer():
    """Rows of swiglu_rows (CSR order) pushed through W_down and combined reproduce moe_ffn."""
    from oracle import moe as omoe
    T, k, E, H, I, Ho = 9, 2, 4, 6, 10, 3
    rng = np.random.default_rng(5)
    X = rng.standard_normal((T, H))
    Wg, Wu, Wd = rng.standard_normal((E, H, I)), rng.standard_normal((E, H, I)), rng.standard_normal((E, I, Ho))
    ids, w = _ids_w(T, k, E, 6)
    counts, row_off, tok, slot = omoe.buckets(ids, E)
    h = ffn.swiglu_rows(X, Wg, Wu, tok, row_off)
    out = np.zeros((T, Ho))
    for e in range(E):
        for r in range(row_off[e], row_off[e + 1]):
            out[tok[r]] += w[tok[r], slot[r]] * (h[r] @ Wd[e])
    assert np.allclose(out, ffn.moe_ffn(X, Wg, Wu, Wd, ids, w), rtol=1e-12, atol=1e-12)


def test_moe_ffn_entries_equals_layer():
    """The on-demand sampled form equals the whole-layer definition on the sampled entries."""
    rng = np.random.default_rng(3)
    T, E, k, H, I, Ho = 9, 4, 2, 6, 10, 5
    X = rng.standard_normal((T, H))
    Wg, Wu, Wd = rng.standard_normal((E, H, I)), rng.standard_normal((E, H, I)), rng.standard_normal((E, I, Ho))
    ids = np.array([rng.permutation(E)[:k] for _ in range(T)])
    ids[2, 1] = -1
    w = rng.random((T, k))
    full = ffn.moe_ffn(X, Wg, Wu, Wd, ids, w)
    toks, cols = [0, 2, 7, 8], [4, 1]
    got = ffn.moe_ffn_entries(lambda t: X[t], lambda e: Wg[e], lambda e: Wu[e], lambda e, cs: Wd[e][:, cs],
                              ids, w, toks, cols)
    assert np.allclose(got, full[np.ix_(toks, cols)], rtol=1e-13, atol=1e-13)
