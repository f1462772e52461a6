"""Pins for oracle/moe.py — no GPU.

Pins: SPEC worked examples (S:n), a hand-derived golden (tests/golden/tiny_a.json),
conservation / membership invariants, SURVEY seed-0 plan fingerprints, closed
forms of the GEMM (identity W, all-ones W, rank-1 operands), a pure-Python
scalar triple loop on integer data, and the P:90 per-(token, slot) definition
for the expert-parallel simulator.
"""
import json
import os
import random

import numpy as np
import pytest

import synth
from oracle import moe

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _tiny_a():
    return synth.route_tiny_a(16)


# ---- c1 buckets --------------------------------------------------------------
def test_buckets_spec_example():
    counts, row_off, tok, slot = moe.buckets(np.array([[1, 3], [2, 3]]), 4)
    assert counts.tolist() == [0, 1, 1, 2]
    assert tok.tolist() == [0, 1, 0, 1]
    assert row_off.tolist() == [0, 0, 1, 2, 4]
    assert slot.tolist() == [0, 0, 1, 1]


def test_buckets_tiny_a_golden():
    g = json.load(open(os.path.join(GOLD, "tiny_a.json")))
    counts, row_off, tok, _ = moe.buckets(_tiny_a(), 4)
    assert counts.tolist() == g["counts"]
    assert row_off.tolist() == g["row_off"]
    for e in range(4):
        assert tok[row_off[e]:row_off[e + 1]].tolist() == g["bucket"][str(e)]


def test_buckets_conservation_membership():
    rng = np.random.default_rng(3)
    for _ in range(20):
        E = int(rng.integers(2, 40))
        k = int(rng.integers(1, min(E, 8) + 1))
        T = int(rng.integers(0, 300))
        ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]) if T else np.zeros((0, k), np.int32)
        counts, row_off, tok, slot = moe.buckets(ids, E)
        assert counts.sum() == T * k
        for e in range(E):
            b = tok[row_off[e]:row_off[e + 1]].tolist()
            assert b == sorted(b) and len(set(b)) == len(b)
            assert set(b) == {t for t in range(T) if e in ids[t]}
            for r in range(row_off[e], row_off[e + 1]):
                assert ids[tok[r], slot[r]] == e


def test_buckets_reject_bad_input():
    with pytest.raises(ValueError):
        moe.buckets(np.array([[1, 1]]), 4)
    with pytest.raises(ValueError):
        moe.buckets(np.array([[0, 4]]), 4)


# ---- c2 plan -----------------------------------------------------------------
def test_tile_count_spec_examples():
    assert moe.tiles_of(0, 256, 128, 256) == 0
    assert moe.tiles_of(128, 256, 128, 256) == 1
    assert moe.tiles_of(100, 70, 64, 32) == 6


def test_plan_tiny_a_golden():
    g = json.load(open(os.path.join(GOLD, "tiny_a.json")))
    counts, _, _, _ = moe.buckets(_tiny_a(), 4)
    p = moe.plan(counts, 128, 128, 128)
    assert p["sigma"] == g["plan_128x128_N128"]["sigma"]
    assert p["prefix"] == g["plan_128x128_N128"]["prefix"]
    p = moe.plan(counts, 128, 4, 32)
    assert p["nu"] == g["plan_4x32_N128"]["nu"]
    assert p["prefix"] == g["plan_4x32_N128"]["prefix"]


def test_plan_invariants_random():
    rng = random.Random(4)
    for _ in range(100):
        E = rng.randint(1, 100)
        counts = [0 if rng.random() < 0.3 else rng.randint(1, 600) for _ in range(E)]
        if sum(counts) == 0:
            continue
        N = rng.choice([64, 128, 200, 1408])
        bm, bn = rng.choice([(128, 256), (128, 128), (64, 64)])
        p = moe.plan(counts, N, bm, bn)
        pre = p["prefix"]
        assert all(pre[i] < pre[i + 1] for i in range(len(pre) - 1))      # strictly increasing
        assert pre[-1] == sum(p["nu"])
        assert len(set(p["sigma"])) == len(p["sigma"])
        assert all(counts[e] > 0 for e in p["sigma"])                       # no empty expert in sigma
        assert len(p["padded"]) % 32 == 0


def test_plan_fingerprints_seed0():
    """SURVEY §8(d) seed-0 fingerprints (computed independently by the survey)."""
    c = synth.CONFIGS["mix"]
    counts = np.bincount(synth.route(c, 0).ravel(), minlength=c.E)
    p = moe.plan(counts, c.N, 128, 256)
    assert (p["M"], p["total"]) == (8, 3864)
    c = synth.CONFIGS["ds"]
    counts = np.bincount(synth.route(c, 0).ravel(), minlength=c.E)
    p = moe.plan(counts, c.N, 128, 128)
    assert (p["M"], p["total"]) == (48, 4444)
    assert len(p["padded"]) == 64                                            # two 32-wide chunks


def test_paper_best_case_empty_extension():
    """all tokens to 8 of 64 experts -> M = 8 and total = sum of 8 single plans."""
    c = synth.CONFIGS["paper_best"]
    counts = np.bincount(synth.route(c).ravel(), minlength=c.E)
    p = moe.plan(counts, c.N, 128, 256)
    assert p["M"] == 8
    assert p["total"] == sum(moe.plan([m], c.N, 128, 256)["total"] for m in counts[:8])


def test_expert_ordering_spec_examples():
    assert moe.order_tasks([9, 1, 8, 2], "alternating") == [0, 3, 2, 1]            # S:345 (a, d, c, b)
    # 8 experts, loads 8..1 -> busiest at slots {0, 4, 2, 6, 1, 5, 3, 7}
    order = moe.order_tasks([8, 7, 6, 5, 4, 3, 2, 1], "half_interval")
    assert [order.index(j) for j in range(8)] == [0, 4, 2, 6, 1, 5, 3, 7]
    assert moe.order_tasks([3, 3, 3], "natural") == [0, 1, 2]
    rng = random.Random(8)
    for _ in range(100):
        loads = [0 if rng.random() < 0.3 else rng.randint(1, 50) for _ in range(rng.randint(1, 70))]
        for st in ("natural", "alternating", "half_interval", "light_last"):
            o = moe.order_tasks(loads, st)
            assert sorted(o) == [j for j in range(len(loads)) if loads[j] > 0]     # a permutation of eta


def test_gemv_kind_by_hand():
    """kind 2 (GEMV): whole tasks of m <= m_max < bm only; they have no tiles (nu = 0, not in sigma)."""
    cat = ((2, 4), (1, 64))
    assert [moe.tail_kind(m, 256, cat) for m in (0, 1, 4, 5, 64, 65, 257, 260, 320)] == [0, 2, 2, 1, 1, 0, 1, 1, 1]
    p = moe.plan([1, 456, 4, 0, 5, 257, 3], 16384, 256, 512, catalog=cat)
    assert p["nu"] == [0, 64, 0, 0, 32, 64, 0] and p["sigma"] == [1, 4, 5] and p["gemv"] == [0, 2, 6]
    assert p["total"] == 160
    # 10 other tiles < GEMV_MIN_TILES: no GEMV, the 1-4 row tasks take the next rule (SWAP)
    q = moe.plan([1, 456, 4, 0, 5, 257, 3], 1024, 256, 512, catalog=cat)
    assert q["gemv"] == [] and [t["kind"] for t in q["tasks"]] == [1, 0, 1, 0, 1, 1, 1]


def test_light_last_order_by_hand():
    """light_last: tasks of > 64 rows in expert order, then the light ones in expert order (R7)."""
    assert moe.order_tasks([65, 64, 0, 1, 300, 2, 65], "light_last") == [0, 4, 6, 1, 3, 5]
    assert moe.order_tasks([1, 2, 3], "light_last") == [0, 1, 2]                    # all light: natural
    assert moe.order_tasks([100, 200], "light_last") == [0, 1]                      # none light: natural


def test_ordering_keeps_the_tile_partition():
    """ordering changes only the tile order, never the partition (hence never Y)."""
    counts = [4096] * 7 + [4096 - 56] + [1] * 56
    row_off = np.concatenate([[0], np.cumsum(counts)])
    for st in ("alternating", "half_interval", "light_last"):
        p = moe.plan(counts, 2560, 128, 256, order=st)
        assert sorted(p["sigma"]) == list(range(64))
        cover = np.zeros((sum(counts), 2560), dtype=np.int8)
        seen = set()
        for B in range(p["total"]):
            d = moe.decode(p, row_off, B)
            seen.add((d["expert"], d["rt"], d["ct"]))
        assert len(seen) == p["total"] == moe.plan(counts, 2560, 128, 256)["total"]


# ---- c3 decode ---------------------------------------------------------------
def test_decode_enumeration_rt_fastest_and_cover():
    rng = random.Random(6)
    for _ in range(30):
        E = rng.randint(1, 12)
        counts = [0 if rng.random() < 0.3 else rng.randint(1, 40) for _ in range(E)]
        if sum(counts) == 0:
            counts[0] = 3
        N = rng.choice([16, 40, 64])
        bm, bn = rng.choice([(8, 16), (16, 16), (4, 32)])
        p = moe.plan(counts, N, bm, bn)
        row_off = np.concatenate([[0], np.cumsum(counts)])
        B = 0
        for e in range(E):                      # independent enumeration: experts, then ct, then rt
            if counts[e] == 0:
                continue
            R = -(-counts[e] // bm)
            for ct in range(-(-N // bn)):
                for rt in range(R):
                    d = moe.decode(p, row_off, B)
                    assert (d["expert"], d["rt"], d["ct"]) == (e, rt, ct)
                    assert d["rows"] == (row_off[e] + rt * bm, row_off[e] + min(rt * bm + bm, counts[e]))
                    assert d["cols"] == (ct * bn, min(ct * bn + bn, N))
                    B += 1
        assert B == p["total"]
        assert (moe.tile_cover(p, row_off, sum(counts)) == 1).all()          # exactly-once


def test_split_tail_tasks_cover_exactly_once():
    """Two tiling strategies in one plan: the tail tile of each expert (kind 1)
    covers exactly its m mod 256 rows and Y is still tiled exactly once."""
    rng = random.Random(7)
    for _ in range(20):
        E = rng.randint(1, 6)
        counts = [0 if rng.random() < 0.2 else rng.randint(1, 700) for _ in range(E)]
        if sum(counts) == 0:
            counts[0] = 1
        N = rng.choice([200, 256, 600])
        p = moe.plan(counts, N, 256, 256, split_tail=True)
        assert p["total"] == moe.plan(counts, N, 256, 256)["total"]
        row_off = np.concatenate([[0], np.cumsum(counts)])
        assert (moe.tile_cover(p, row_off, sum(counts)) == 1).all()
        for B in range(p["total"]):
            d = moe.decode(p, row_off, B)
            m = counts[d["expert"]]
            if d["kind"] == 1:
                assert m % 256 and d["rows"] == (row_off[d["expert"]] + m // 256 * 256, row_off[d["expert"]] + m)
                assert d["height"] % 16 == 0 and d["height"] - 16 < m % 256 <= d["height"]
            else:
                assert d["rows"][1] - d["rows"][0] == 256 or m % 256 == 0 or d["rt"] < m // 256


def test_ride_tasks_cover_exactly_once():
    """MOE_KIND_RIDE: an expert of 256 R + r rows (r <= 32) keeps its ceil(m/256) tile slots
    per column block; slots R-2 / R-1 are the two 256-column halves of row tile R-2 plus the tail rows, and Y is
    still tiled exactly once.  Experts without a full row tile, or N % 512 != 0, do not ride."""
    rng = random.Random(11)
    for _ in range(25):
        E = rng.randint(1, 6)
        counts = [0 if rng.random() < 0.2 else rng.choice([rng.randint(1, 700), 256 * rng.randint(1, 3) +
                                                           rng.randint(1, 40)]) for _ in range(E)]
        if sum(counts) == 0:
            counts[0] = 300
        N = rng.choice([512, 1024, 1536])
        p = moe.plan(counts, N, 256, 512, catalog=((3, 32),))
        assert p["total"] == moe.plan(counts, N, 256, 512)["total"] and p["prefix"] == moe.plan(counts, N, 256, 512)["prefix"]
        row_off = np.concatenate([[0], np.cumsum(counts)])
        assert (moe.tile_cover(p, row_off, sum(counts)) == 1).all()
        for t in p["tasks"]:
            m = t["rows"]
            assert (t["kind"] == 3) == (m > 256 and 0 < m % 256 <= 32)
        for B in range(p["total"]):
            d = moe.decode(p, row_off, B)
            m = counts[d["expert"]]
            if d["kind"] == 3:
                assert d["rows"] == (row_off[d["expert"]] + (m // 256 - 1) * 256, row_off[d["expert"]] + m)
                assert d["cols"] == (d["ct"] * 512 + 256 * d["half"], d["ct"] * 512 + 256 * d["half"] + 256)
                assert d["height"] in (16, 32) and d["height"] - 16 < m % 256 <= d["height"]
    assert all(t["kind"] == 0 for t in moe.plan([300, 260, 20], 1408, 256, 512, catalog=((3, 32),))["tasks"])


# ---- c4 GEMM -----------------------------------------------------------------
def _route(T, E, k, seed):
    return synth.route_gumbel(seed, T, E, k)


def test_gemm_identity_weights():
    """S:404 analogue: W[e] = (e+1) I  =>  Y row = (e+1) * X[token] exactly."""
    T, E, k, H = 37, 5, 2, 32
    ids = _route(T, E, k, 1)
    counts, row_off, tok, _ = moe.buckets(ids, E)
    X = synth.make_x(1, T, H)
    W = synth.make_w(1, E, H, H, mode="identity")
    Y = moe.expert_gemm(X, W, tok, row_off)
    for e in range(E):
        for r in range(row_off[e], row_off[e + 1]):
            assert np.array_equal(Y[r], (e + 1) * X[tok[r]])


def test_gemm_integer_triple_loop():
    """Integer data, pure-Python scalar loops in token order, placed by search."""
    T, E, k, H, N = 13, 4, 2, 8, 6
    ids = _route(T, E, k, 2)
    X = synth.make_x(2, T, H, "int")
    W = synth.make_w(2, E, H, N, "int")
    counts, row_off, tok, _ = moe.buckets(ids, E)
    Y = moe.expert_gemm(X, W, tok, row_off)
    for t in range(T):
        for j in range(k):
            e = int(ids[t, j])
            row = [r for r in range(row_off[e], row_off[e + 1]) if tok[r] == t]
            assert len(row) == 1
            for n in range(N):
                s = 0
                for h in range(H):
                    s += int(X[t, h]) * int(W[e, h, n])
                assert Y[row[0], n] == s


def test_gemm_closed_forms():
    T, E, k, H, N = 20, 3, 2, 16, 12
    ids = _route(T, E, k, 3)
    counts, row_off, tok, _ = moe.buckets(ids, E)
    X = synth.make_x(3, T, H)
    # all-ones W: Y[r, n] = sum_h X[t, h]
    Y = moe.expert_gemm(X, np.ones((E, H, N)), tok, row_off)
    assert np.allclose(Y, X[tok].sum(axis=1)[:, None] * np.ones(N), rtol=0, atol=1e-12)
    # rank-1: X = a b^T, W[e] = c_e b' d^T  =>  Y[r, n] = a_t c_e (b . b') d_n
    rng = np.random.default_rng(0)
    a, b, bp, d, c = rng.normal(size=T), rng.normal(size=H), rng.normal(size=H), rng.normal(size=N), rng.normal(size=E)
    Xr = np.outer(a, b)
    Wr = np.stack([c[e] * np.outer(bp, d) for e in range(E)])
    Y = moe.expert_gemm(Xr, Wr, tok, row_off)
    for e in range(E):
        for r in range(row_off[e], row_off[e + 1]):
            assert np.allclose(Y[r], a[tok[r]] * c[e] * (b @ bp) * d, rtol=1e-12, atol=1e-12)


def test_gemm_entries_match_full():
    T, E, k, H, N = 40, 6, 3, 24, 20
    ids = _route(T, E, k, 4)
    counts, row_off, tok, _ = moe.buckets(ids, E)
    X = synth.make_x(4, T, H)
    W = synth.make_w(4, E, H, N)
    Y = moe.expert_gemm(X, W, tok, row_off)
    rows = [0, 5, int(row_off[-1]) - 1]
    cols = np.array([0, 7, N - 1])
    got = moe.expert_gemm_entries(lambda t: synth.workloads.x_rows(4, T, H, [t])[0],
                                  lambda e, cs: synth.workloads.w_columns(4, E, H, N, e, cs),
                                  tok, row_off, rows, cols)
    assert np.allclose(got, Y[rows][:, cols], rtol=1e-13, atol=1e-13)


# ---- c5 EP ---------------------------------------------------------------------
@pytest.mark.parametrize("G", [1, 2, 4])
def test_ep_simulator_matches_definition(G):
    T, E, k, H, N = 16, 8, 2, 8, 10
    ids = _route(T, E, k, 5)
    X = synth.make_x(5, T, H, "int")
    W = synth.make_w(5, E, H, N, "int")
    ref = moe.per_slot_outputs(ids, X, W)
    sim = moe.ep_simulate(ids, X, W, G)
    got = np.concatenate(sim["out"])
    assert np.array_equal(got, ref)
    # conservation of dispatched rows: sum_t |{owner(e) : e in topk[t]}|
    El = E // G
    assert sim["sent_rows"].sum() == sum(len({int(e) // El for e in ids[t]}) for t in range(T))
    assert sim["local_counts"].sum() == T * k


def test_per_slot_matches_bucketed_gemm():
    T, E, k, H, N = 30, 5, 2, 8, 6
    ids = _route(T, E, k, 6)
    X = synth.make_x(6, T, H, "int")
    W = synth.make_w(6, E, H, N, "int")
    counts, row_off, tok, slot = moe.buckets(ids, E)
    Y = moe.expert_gemm(X, W, tok, row_off)
    ref = moe.per_slot_outputs(ids, X, W)
    for r in range(len(tok)):
        assert np.array_equal(Y[r], ref[tok[r] * k + slot[r]])
