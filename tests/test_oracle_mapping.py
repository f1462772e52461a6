"""Pins for oracle/mapping.py (Alg. 1, 2, 4) — no GPU.

Each pin is something other than the oracle itself: SPEC worked examples
(S:n), the bit semantics of vote/popcount, and a brute-force enumeration of the
(task, tile) lattice written independently below.
"""
import random

import pytest

from oracle import mapping as om

INT32_MAX = 2**31 - 1


# ---- Alg. 1 -----------------------------------------------------------------
def test_prefix_spec_vectors():
    assert om.build_tile_prefix([3, 1, 4]) == [3, 4, 8]
    assert om.build_tile_prefix([1]) == [1]
    assert om.pad_tile_prefix([3, 4, 8], 4, "repeat") == [3, 4, 8, 8]
    assert om.pad_tile_prefix([3, 4, 8], 4, "max") == [3, 4, 8, INT32_MAX]
    assert len(om.pad_tile_prefix(list(range(1, 41)), 32)) == 64


def test_prefix_against_sequential_sum():
    rng = random.Random(1)
    for _ in range(200):
        nu = [rng.randint(0, 9) for _ in range(rng.randint(1, 70))]
        acc, ref = 0, []
        for v in nu:
            acc += v
            ref.append(acc)
        assert om.build_tile_prefix(nu) == ref


# ---- Alg. 4 stage ----------------------------------------------------------
def test_nonempty_stage_spec_vectors():
    assert om.nonempty_stage([2, 0, 3]) == ([0, 2], [2, 5])                # S:118 (1-based {1->1, 2->3})
    assert om.nonempty_stage([0, 0, 7]) == ([2], [7])
    assert om.nonempty_stage([4, 1, 2]) == ([0, 1, 2], [4, 5, 7])          # S:119 identity sigma


# ---- vote / popcount ---------------------------------------------------------
def test_vote_and_popcount_bits():
    assert om.warp_vote([False] * 32) == 0
    assert om.popcount(0) == 0
    assert om.warp_vote([True, False, True, False]) == 0b0101
    assert om.popcount(0b0101) == 2
    rng = random.Random(2)
    for _ in range(100):
        p = [rng.random() < 0.5 for _ in range(32)]
        m = om.warp_vote(p)
        assert om.popcount(m) == sum(p)
        assert all(((m >> i) & 1) == int(p[i]) for i in range(32))


# ---- Alg. 2 ------------------------------------------------------------------
def test_mapping_spec_vectors():
    pre = om.pad_tile_prefix([3, 4, 8], 32)
    assert om.mapping_single_warp(pre, 0) == (0, 0)
    assert om.mapping_single_warp(pre, 5) == (2, 1)
    assert om.mapping_single_warp(pre, 3) == (1, 0)
    pre64 = om.pad_tile_prefix(list(range(1, 65)), 32)
    assert om.mapping_chunked(pre64, 40) == (40, 0)


def test_extended_spec_vectors():
    sigma, pre = om.nonempty_stage([2, 0, 3])
    assert om.mapping_extended(om.pad_tile_prefix(pre, 32), sigma, 3) == (1, 2, 1)   # S:254 (1-based task 3)
    sigma, pre = om.nonempty_stage([0, 5, 0])
    assert om.mapping_extended(om.pad_tile_prefix(pre, 32), sigma, 4) == (0, 1, 4)   # S:256 (1-based task 2)


def _brute_force(nu):
    """Enumerate blocks in order: for each non-empty task j, for each tile l."""
    out = []
    h = 0
    for j, n in enumerate(nu):
        if n == 0:
            continue
        for l in range(n):
            out.append((h, j, l))
        h += 1
    return out


@pytest.mark.parametrize("warp", [8, 16, 32, 64])
@pytest.mark.parametrize("pad", ["max", "repeat"])
def test_mapping_bijection_brute_force(warp, pad):
    rng = random.Random(warp * 7 + len(pad))
    for _ in range(150):
        n_tasks = rng.randint(1, 140)
        nu = [0 if rng.random() < 0.3 else rng.randint(1, 12) for _ in range(n_tasks)]
        if sum(nu) == 0:
            nu[rng.randrange(n_tasks)] = 1
        sigma, pre = om.nonempty_stage(nu)
        padded = om.pad_tile_prefix(pre, warp, pad)
        expect = _brute_force(nu)
        got = [om.mapping_extended(padded, sigma, B, warp) for B in range(sum(nu))]
        assert got == expect


def test_single_warp_equals_chunked_and_linear_scan():
    rng = random.Random(5)
    for _ in range(100):
        nu = [rng.randint(1, 9) for _ in range(rng.randint(1, 32))]
        pre = om.build_tile_prefix(nu)
        padded = om.pad_tile_prefix(pre, 32)
        for B in range(pre[-1]):
            # linear scan: first j with pre[j] > B  (SPEC S:172 oracle)
            j = next(i for i, v in enumerate(pre) if v > B)
            lin = (j, B - (pre[j - 1] if j else 0))
            assert om.mapping_single_warp(padded, B) == lin
            assert om.mapping_chunked(padded, B) == lin


def test_padding_neutrality():
    rng = random.Random(9)
    for _ in range(50):
        nu = [rng.randint(1, 6) for _ in range(rng.randint(1, 90))]
        pre = om.build_tile_prefix(nu)
        a = om.pad_tile_prefix(pre, 32, "max")
        b = om.pad_tile_prefix(pre, 32, "repeat")
        for B in range(pre[-1]):
            assert om.mapping_chunked(a, B) == om.mapping_chunked(b, B)


def test_monotone():
    nu = [3, 1, 4, 1, 5, 9, 2, 6]
    pre = om.pad_tile_prefix(om.build_tile_prefix(nu), 8)
    res = [om.mapping_chunked(pre, B, 8) for B in range(sum(nu))]
    assert res == sorted(res)
