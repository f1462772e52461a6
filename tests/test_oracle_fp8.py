"""Pins of oracle/fp8.py (E4M3 decode, FP8 expert GEMM) and of the FP8 input generator (synth/fp8.py).

The decode is pinned by values the OCP FP8 specification fixes (1.0, the largest finite 448, the
smallest normal 2^-6 and subnormal 2^-9, NaN, signed zero) and by torch's float8_e4m3fn conversion
over all 256 codes (a library routine); the GEMM by closed forms (identity weights, a rank-1 case)."""
import math

import numpy as np
import pytest

from oracle import fp8 as ofp8
from oracle import moe as omoe
from synth import fp8 as sfp8


def test_e4m3_spec_values():
    v = ofp8.e4m3_value
    assert v(0x38) == 1.0 and v(0xB8) == -1.0
    assert v(0x7E) == 448.0 and v(0xFE) == -448.0          # max finite S.1111.110
    assert v(0x08) == 2.0 ** -6                             # min normal
    assert v(0x01) == 2.0 ** -9                             # min subnormal
    assert v(0x07) == 7 * 2.0 ** -9                         # max subnormal
    assert v(0x40) == 2.0 and v(0x44) == 3.0 and v(0x48) == 4.0 and v(0x3C) == 1.5
    assert v(0x00) == 0.0 and math.copysign(1.0, v(0x80)) == -1.0
    assert math.isnan(v(0x7F)) and math.isnan(v(0xFF))


def test_e4m3_decode_matches_torch_all_codes():
    torch = pytest.importorskip("torch")
    codes = np.arange(256, dtype=np.uint8)
    ref = torch.from_numpy(codes).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    got = ofp8.e4m3_decode(codes)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])


def test_encoder_truncates_to_four_significant_bits():
    # every c the generators draw: the code decodes (torch's conversion) to c truncated toward zero to
    # 4 significant bits, times 2^-shift
    torch = pytest.importorskip("torch")
    for shift in (0, 6):
        c = np.arange(-254, 255, dtype=np.int32)
        codes = sfp8.encode_np(c, shift)
        dec = torch.from_numpy(codes).view(torch.float8_e4m3fn).to(torch.float64).numpy()
        a = np.abs(c)
        q = np.array([x if x < 16 else (x >> (x.bit_length() - 4)) << (x.bit_length() - 4) for x in map(int, a)])
        assert np.array_equal(dec, np.sign(c) * q * 2.0 ** -shift)
        assert np.array_equal(sfp8.encode_torch(torch.from_numpy(c), shift).numpy(), codes)


@pytest.mark.parametrize("mode", ["normal", "int"])
def test_numpy_torch_twins_identical(mode):
    torch = pytest.importorskip("torch")
    X = sfp8.make_x_fp8(3, 7, 48, mode)
    assert np.array_equal(sfp8.make_x_fp8_torch(3, 7, 48, mode).numpy(), X)
    W = sfp8.make_w_fp8(3, 3, 32, 40, mode)
    assert np.array_equal(sfp8.make_w_fp8_torch(3, 3, 32, 40, mode, chunk=1000).numpy(), W)
    assert np.array_equal(sfp8.w_fp8_columns(3, 3, 32, 40, 2, [0, 5, 39], mode), W[2][:, [0, 5, 39]])
    assert np.array_equal(sfp8.x_fp8_rows(3, 7, 48, [6, 1], mode), X[[6, 1]])
    if mode == "int":
        assert set(np.unique(ofp8.e4m3_decode(X))) <= set(range(-4, 5))


def test_expert_gemm_fp8_identity_weights_closed_form():
    # W[e] = I (code 0x38 on the diagonal): Y rows = scale[e] * X[token] exactly
    rng = np.random.default_rng(0)
    T, E, k, H = 12, 3, 2, 32
    ids = np.stack([rng.choice(E, k, replace=False) for _ in range(T)]).astype(np.int32)
    counts, row_off, tok, _ = omoe.buckets(ids, E)
    X = sfp8.make_x_fp8(0, T, H)
    W = np.zeros((E, H, H), dtype=np.uint8)
    for e in range(E):
        np.fill_diagonal(W[e], 0x38)
    scale = np.array([0.5, 2.0, 0.25], dtype=np.float32)
    Y = ofp8.expert_gemm_fp8(X, W, tok, row_off, scale)
    for e in range(E):
        for r in range(row_off[e], row_off[e + 1]):
            assert np.array_equal(Y[r], scale[e] * ofp8.e4m3_decode(X[tok[r]]))


def test_expert_gemm_fp8_rank_one_closed_form():
    # X rows all 1.5 (0x3C), W[e] all 2.0 (0x40): every Y entry = scale[e] * H * 3
    T, E, H, N = 5, 2, 64, 128
    ids = np.array([[0, 1]] * T, dtype=np.int32)
    counts, row_off, tok, _ = omoe.buckets(ids, E)
    X = np.full((T, H), 0x3C, dtype=np.uint8)
    W = np.full((E, H, N), 0x40, dtype=np.uint8)
    Y = ofp8.expert_gemm_fp8(X, W, tok, row_off, np.array([1.0, 0.125], dtype=np.float32))
    assert np.all(Y[:T] == H * 3.0) and np.all(Y[T:] == 0.125 * H * 3.0)
    assert np.array_equal(ofp8.expert_gemm_fp8_entries(X[:2], W[1][:, :3], 0.125), np.full((2, 3), 0.125 * H * 3.0))


def test_rank_slices_match_full_generation():
    """Expert-parallel ranks generate their own token rows / expert range of the same codes."""
    torch = pytest.importorskip("torch")
    X = sfp8.make_x_fp8(2, 12, 32)
    assert np.array_equal(sfp8.make_x_fp8_torch(2, 4, 32, row0=8).numpy(), X[8:12])
    W = sfp8.make_w_fp8(2, 4, 16, 24)
    assert np.array_equal(sfp8.make_w_fp8_torch(2, 4, 16, 24, experts=range(2, 4), chunk=100).numpy(), W[2:4])
    assert np.array_equal(sfp8.w_scale(3, 4096), np.full(3, 2.0 ** -6, dtype=np.float32))
