"""The full-mantissa parity corpora (synth "generic" bf16 mode, FP8 "full" codes) and why they bite.

These inputs exist so that GPU parity tests exercise fp32 accumulation ROUNDING ("the
parity corpus never reaches accumulation rounding"): the "normal" lattice corpus keeps every fp32
partial sum exact.  Here the exact dot products are computed in int64 (every value is an integer
multiple of a power of two), and the tests prove that
  * most exact results need more than 24 significant bits (fp32 cannot hold them), and a plain
    fp32 accumulation differs from the exact value on most outputs;
  * the fp64 oracle (oracle.moe.expert_gemm / oracle.fp8.expert_gemm_fp8) is within 2^-45 relative
    of the exact integer result on these corpora — a pin independent of the oracle's own formula.
"""
import numpy as np
import pytest

import synth
from oracle import fp8 as ofp8
from oracle import moe as omoe
from synth import fp8 as sfp8
from synth import workloads as wl


def _bits_to_int(bits: np.ndarray):
    """bf16 patterns -> (signed integer mantissa, exponent) with value = mant * 2^exp."""
    b = bits.astype(np.int64)
    sign = np.where(b >> 15 & 1, -1, 1)
    bexp = (b >> 7) & 255
    mant = 128 + (b & 127)
    return sign * mant, bexp - 127 - 7


def _exact_int_dot(xm, xe, wm, we):
    """Exact sum_h x[h] w[h] as (int64 numerator, exponent base) for one row / column."""
    e = xe + we
    base = int(e.min())
    terms = (xm * wm) << (e - base)
    return int(terms.sum()), base


def _sig_bits(n: int) -> int:
    n = abs(int(n))
    if n == 0:
        return 0
    while n % 2 == 0:
        n //= 2
    return n.bit_length()


def test_generic_twins_identical():
    torch = pytest.importorskip("torch")
    for seed, stream, shift in ((0, wl.STREAM_X, 6), (3, wl.STREAM_W, 12)):
        a = synth.counter_values(seed, stream, np.arange(70000), "generic", shift)
        b = synth.counter_values_torch(seed, stream, 0, 70000, "generic", shift).double().numpy()
        assert np.array_equal(a, b)
        # exact in bf16 (a bf16 bit pattern by construction)
        assert np.array_equal(torch.from_numpy(a).to(torch.bfloat16).double().numpy(), a)


def test_generic_spans_mantissas_and_octaves():
    v = synth.counter_values(1, wl.STREAM_X, np.arange(200000), "generic", 6)
    e = np.floor(np.log2(np.abs(v)))
    assert e.max() - e.min() == 15                               # 16 octaves
    m = np.round((np.abs(v) / 2.0 ** e - 1) * 128).astype(int)
    assert len(np.unique(m)) == 128                               # every 7-bit mantissa
    assert 0.45 < (v < 0).mean() < 0.55


def test_generic_corpus_needs_fp32_rounding_and_pins_oracle():
    """Mix shape (H = 4096): exact int64 dot products of sampled (token, column) pairs."""
    seed, H, N, E, T = 0, 4096, 14336, 8, 64
    sx, sw = wl._shift_x(), wl._shift_w(H)
    rows = np.arange(T)
    cols = np.arange(0, N, N // 16)[:16]
    hx = wl._fmix32_np((rows[:, None] * H + np.arange(H)[None, :]).astype(np.uint64).__xor__(
        np.uint64(wl._key(seed, wl.STREAM_X))).astype(np.uint32))
    xm, xe = _bits_to_int(wl.generic_bits_np(hx, sx))
    e = 3
    idx = e * H * N + np.arange(H)[:, None] * N + cols[None, :]
    hw = wl._fmix32_np((idx.astype(np.uint64) ^ np.uint64(wl._key(seed, wl.STREAM_W))).astype(np.uint32))
    wm, we = _bits_to_int(wl.generic_bits_np(hw, sw))
    X = wl.x_rows(seed, T, H, rows, "generic")
    Wc = wl.w_columns(seed, E, H, N, e, cols, "generic")
    oracle = omoe.expert_gemm(X, Wc[None], rows, np.array([0, T]))
    n_wide, n_diff, worst = 0, 0, 0.0
    for i in range(T):
        x32 = X[i].astype(np.float32)
        for j in range(len(cols)):
            num, base = _exact_int_dot(xm[i], xe[i], wm[:, j], we[:, j])
            exact = float(num) * 2.0 ** base                       # rounding only at the very end
            n_wide += _sig_bits(num) > 24
            acc = np.float32(0)
            w32 = Wc[:, j].astype(np.float32)
            for h in range(H):                                      # plain fp32 accumulation, in order
                acc = np.float32(acc + x32[h] * w32[h])
            n_diff += float(acc) != exact
            worst = max(worst, abs(oracle[i, j] - exact) / abs(exact))
    total = T * len(cols)
    assert n_wide >= 0.95 * total, f"only {n_wide}/{total} exact sums exceed 24 significant bits"
    assert n_diff >= 0.9 * total, f"fp32 accumulation was exact on {total - n_diff}/{total} outputs"
    assert worst < 2.0 ** -45, f"oracle vs exact integer sum: relative {worst}"


def test_fp8_full_codes_twins_and_range():
    torch = pytest.importorskip("torch")
    a = sfp8.make_x_fp8(2, 300, 256, "full")
    b = sfp8.make_x_fp8_torch(2, 300, 256, "full").numpy()
    assert np.array_equal(a, b)
    assert not np.any((a & 127) == 127)                           # no NaN code
    assert len(np.unique(a)) == 254                               # every finite code
    w = sfp8.make_w_fp8(2, 2, 64, 256, "full")
    assert np.array_equal(w, sfp8.make_w_fp8_torch(2, 2, 64, 256, "full").numpy())


def test_fp8_full_corpus_needs_fp32_rounding_and_pins_oracle():
    seed, H, N, E, T = 1, 2048, 1408, 4, 48
    X = sfp8.make_x_fp8(seed, T, H, "full")
    cols = np.arange(0, N, 88)
    Wc = sfp8.w_fp8_columns(seed, E, H, N, 2, cols, "full")
    xv = ofp8.e4m3_decode(X)
    wv = ofp8.e4m3_decode(Wc)
    xi = np.round(xv * 512).astype(np.int64)                      # every E4M3 value is k * 2^-9
    wi = np.round(wv * 512).astype(np.int64)
    assert np.array_equal(xi / 512.0, xv) and np.array_equal(wi / 512.0, wv)
    scale = np.float32(2.0 ** -8)
    oracle = ofp8.expert_gemm_fp8(X, Wc[None], np.arange(T), np.array([0, T]), [scale])
    exact_num = xi @ wi                                           # int64, exact (|sum| < 2^48)
    exact = exact_num.astype(np.float64) * 2.0 ** -18 * float(scale)
    wide = np.vectorize(_sig_bits)(exact_num) > 24
    acc = np.zeros(exact.shape, dtype=np.float32)
    x32, w32 = xv.astype(np.float32), wv.astype(np.float32)
    for h in range(H):
        acc = (acc + x32[:, h:h + 1] * w32[h:h + 1, :]).astype(np.float32)
    assert wide.mean() > 0.9
    assert (acc.astype(np.float64) * float(scale) != exact).mean() > 0.8
    rel = np.abs(oracle - exact) / np.maximum(np.abs(exact), 1e-300)
    assert rel.max() < 2.0 ** -45
