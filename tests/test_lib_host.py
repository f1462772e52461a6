"""C-ABI library on the host (no GPU): it loads, exports every declared symbol, and
its planner (moe_plan_build) matches the oracle plan bit-exactly."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

import paper_2501_16103_b200 as moe_lib
import synth
from oracle import mapping as om
from oracle import moe as omoe

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2501_16103_b200 import build
    build.build()


def _declared_functions():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(moe_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    L = moe_lib.lib()
    declared = _declared_functions()
    assert "moe_gemm" in declared and "moe_plan_build" in declared and "moe_route" in declared
    for name in declared:
        assert hasattr(L, name), name
    assert set(moe_lib.EXPORTED) == declared
    assert b"sm_100a" in L.moe_version()


ORDER_FLAG = {"natural": 0, "alternating": 4, "half_interval": 8, "light_last": 4096}


def _compare(counts, N, bm, bn, pad, split=False, order="natural", catalog=None):
    """catalog None: the library's built-in catalog, whose rule the test states independently
    ((GEMV, 4) on wide pair plans, bm 256 and bn > 256; none otherwise)."""
    flags = (moe_lib.MOE_PAD_REPEAT if pad == "repeat" else 0) | (moe_lib.MOE_SPLIT_TAIL if split else 0)
    blob = moe_lib.moe_plan_build(counts, 64, N, bm, bn, flags | ORDER_FLAG[order], catalog=catalog)
    p = moe_lib.parse_plan_blob(blob)
    if catalog is None:
        catalog = ((2, 4),) if (bm == 256 and bn > 256) else ()
    if split:
        catalog = ((1, bm),)
    assert p["catalog"] == tuple(catalog)
    ref = omoe.plan(counts, N, bm, bn, pad_mode=pad, split_tail=split, order=order, catalog=catalog)
    assert p["M"] == ref["M"] and p["total"] == ref["total"]
    if ref["M"] == 0:
        return
    assert p["prefix"].tolist() == ref["padded"]
    assert p["sigma"][: p["M"]].tolist() == ref["sigma"]
    row_off = np.concatenate([[0], np.cumsum(counts)])
    assert p["row_off"].tolist() == row_off.tolist()
    for i, t in enumerate(ref["tasks"]):
        q = p["params"][i]
        assert q[0] == t["expert"] and q[1] == row_off[t["expert"]] + t["row_begin"] and q[2] == t["rows"]
        assert q[3] == t["kind"] and q[4] == t["bm"] and q[5] == t["bn"]
        assert (0 if t["kind"] == 2 else q[6] * q[7]) == ref["nu"][i]
        assert q[6] == -(-t["rows"] // bm)


def test_planner_matches_oracle_configs():
    _compare(np.array([11, 0, 11, 10]), 128, 128, 128, "max")          # tiny-A
    c = synth.CONFIGS["mix"]
    _compare(np.bincount(synth.route(c, 0).ravel(), minlength=8), c.N, 128, 256, "max")
    c = synth.CONFIGS["ds"]
    counts = np.bincount(synth.route(c, 0).ravel(), minlength=64)
    for bn in (128, 176, 256):
        _compare(counts, c.N, 128, bn, "max")
        _compare(counts, c.N, 128, bn, "repeat")
    c = synth.CONFIGS["paper_worst"]
    _compare(np.bincount(synth.route(c).ravel(), minlength=64), c.N, 128, 256, "max")


def test_planner_matches_oracle_random_corpus():
    rng = random.Random(11)
    for _ in range(300):
        E = rng.randint(1, 300)
        counts = np.array([0 if rng.random() < 0.4 else rng.randint(1, 3000) for _ in range(E)])
        N = 8 * rng.randint(1, 2500)
        bm = rng.choice([128, 256])
        bn = (32 if bm == 256 else 16) * rng.randint(1, 256 // (32 if bm == 256 else 16))
        _compare(counts, N, bm, bn, rng.choice(["max", "repeat"]))


def test_planner_expert_ordering_matches_oracle():
    rng = random.Random(14)
    for _ in range(200):
        E = rng.randint(1, 300)
        counts = np.array([0 if rng.random() < 0.3 else rng.randint(1, 3000) for _ in range(E)])
        counts[rng.randrange(E)] = counts[rng.randrange(E)]          # ties
        _compare(counts, 8 * rng.randint(1, 800), 128, 256, "max",
                 order=rng.choice(["alternating", "half_interval", "light_last"]))
    c = synth.CONFIGS["paper_worst"]
    counts = np.bincount(synth.route(c).ravel(), minlength=c.E)
    for order in ("alternating", "half_interval", "light_last"):
        _compare(counts, c.N, 256, 256, "max", order=order)
    for bad in (4 | 8, 4 | 4096, 8 | 4096):
        with pytest.raises(moe_lib.MoeError):
            moe_lib.moe_plan_build([1, 2], 64, 128, 128, 128, bad)


def test_planner_split_tail_matches_oracle():
    rng = random.Random(13)
    for _ in range(200):
        E = rng.randint(1, 200)
        counts = np.array([0 if rng.random() < 0.3 else rng.randint(1, 3000) for _ in range(E)])
        _compare(counts, 8 * rng.randint(1, 3000), 256, rng.choice([256, 512]), rng.choice(["max", "repeat"]),
                 split=True)
    with pytest.raises(moe_lib.MoeError):
        moe_lib.moe_plan_build([5, 5], 64, 512, 256, 128, moe_lib.MOE_SPLIT_TAIL)   # needs bn = 256


def test_planner_auto_tile_choice():
    """bm = 0: pair tiles unless their padding rows exceed 1.10x the 128-row padding (header rule)."""
    rng = random.Random(12)
    for _ in range(200):
        E = rng.randint(1, 64)
        counts = [0 if rng.random() < 0.3 else rng.randint(1, 5000) for _ in range(E)]
        if sum(counts) == 0:
            continue
        bn = rng.choice([64, 128, 176, 256])
        blob = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 64, 1024, 0, bn))
        r128 = sum(-(-m // 128) * 128 for m in counts)
        r256 = sum(-(-m // 256) * 256 for m in counts)
        expect = 256 if (r256 * 100 <= r128 * 110 and bn % 32 == 0) else 128
        assert blob["bm"] == expect
        assert not blob["flags"] & moe_lib.MOE_SPLIT_TAIL
        _compare(np.array(counts), 1024, expect, bn, "max")
    c = synth.CONFIGS["mix_balanced"]
    counts = np.bincount(synth.route(c).ravel(), minlength=c.E)
    assert moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, c.H, c.N, 0, 256))["bm"] == 256


def test_planner_wide_tiles_match_oracle():
    """bm = 256, bn = 512 (wide pair tiles): the same Alg. 1/4 mapping over 512-column tiles."""
    rng = random.Random(15)
    for _ in range(200):
        E = rng.randint(1, 300)
        counts = np.array([0 if rng.random() < 0.3 else rng.randint(1, 3000) for _ in range(E)])
        _compare(counts, 8 * rng.randint(1, 3000), 256, rng.choice([288, 384, 480, 512]), rng.choice(["max", "repeat"]),
                 order=rng.choice(["natural", "alternating", "half_interval"]))
    with pytest.raises(moe_lib.MoeError):
        moe_lib.moe_plan_build([5, 5], 64, 1024, 128, 512)                 # wide tiles are pair tiles
    with pytest.raises(moe_lib.MoeError):
        moe_lib.moe_plan_build([5, 5], 64, 1024, 256, 400)                 # block width 200: not a multiple of 16
    with pytest.raises(moe_lib.MoeError):
        moe_lib.moe_plan_build([5, 5], 64, 1024, 256, 544)


def test_planner_auto_tile_width():
    """bn = 0: 512 when bm resolves to 256 and N >= 512; else 256 (header rule)."""
    rng = random.Random(16)
    for _ in range(200):
        E = rng.randint(1, 64)
        counts = [0 if rng.random() < 0.3 else rng.randint(1, 5000) for _ in range(E)]
        N = 8 * rng.randint(1, 400)
        bm = rng.choice([0, 128, 256])
        split = rng.random() < 0.2 and bm == 256
        blob = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 64, N, bm, 0,
                                                              moe_lib.MOE_SPLIT_TAIL if split else 0))
        r128 = sum(-(-m // 128) * 128 for m in counts)
        r256 = sum(-(-m // 256) * 256 for m in counts)
        bm_exp = bm or (256 if r256 * 100 <= r128 * 110 else 128)
        assert blob["bm"] == bm_exp
        assert blob["bn"] == (512 if bm_exp == 256 and N >= 512 else 256)
    c = synth.CONFIGS["mix"]
    counts = np.bincount(synth.route(c).ravel(), minlength=c.E)
    b = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, c.H, c.N))
    assert (b["bm"], b["bn"]) == (256, 512)


def test_planner_decode_regime_tiles():
    """bm = 64 (opt-in 64-token swap-AB decode tiles, bn 256): the mapping is Alg. 1/4 over those
    tiles; bm = 0 never picks them."""
    rng = random.Random(17)
    for _ in range(100):
        E = rng.randint(1, 64)
        counts = [0 if rng.random() < 0.4 else rng.randint(1, 300) for _ in range(E)]
        if not any(counts):
            continue
        _compare(np.array(counts), 8 * rng.randint(1, 2000), 64, 256, rng.choice(["max", "repeat"]))
        assert moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 64, 14336))["bm"] != 64
    with pytest.raises(moe_lib.MoeError):
        moe_lib.moe_plan_build([3, 4], 64, 1024, 64, 256, moe_lib.MOE_SPLIT_TAIL)


def test_planner_decode_bijection_through_blob():
    """Decode every block of a library-built blob with the oracle's Alg. 2 and check the lattice."""
    counts = np.array([300, 0, 5, 129, 0, 1000, 1])
    blob = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 64, 200, 128, 64))
    seen = set()
    for B in range(blob["total"]):
        h, l = om.mapping_chunked(blob["prefix"].tolist(), B)
        task = int(blob["sigma"][h])
        q = blob["params"][task]
        rt, ct = l % q[6], l // q[6]
        assert 0 <= ct < q[7]
        seen.add((task, rt, ct))
    assert len(seen) == blob["total"]


def test_planner_errors():
    L = moe_lib.lib()
    with pytest.raises(moe_lib.MoeError) as e:
        moe_lib.moe_plan_build([1, 2], 63, 128)
    assert e.value.status == -2
    with pytest.raises(moe_lib.MoeError) as e:
        moe_lib.moe_plan_build([1, 2], 64, 128, bm=32)
    assert e.value.status == -2
    with pytest.raises(moe_lib.MoeError) as e:                  # decode tiles are 64 x 256
        moe_lib.moe_plan_build([1, 2], 64, 128, bm=64, bn=128)
    assert e.value.status == -2
    with pytest.raises(moe_lib.MoeError) as e:
        moe_lib.moe_plan_build([1, 2], 64, 128, bn=24)
    assert e.value.status == -2
    with pytest.raises(moe_lib.MoeError) as e:
        moe_lib.moe_plan_build([1, -2], 64, 128)
    assert e.value.status == -1
    with pytest.raises(moe_lib.MoeError) as e:
        moe_lib.moe_plan_build([2**31 - 1, 5], 64, 128)
    assert e.value.status == -3
    assert b"2^31" in L.moe_last_error()
    blob = moe_lib.moe_plan_build([0, 0, 0], 64, 128)
    p = moe_lib.parse_plan_blob(blob)
    assert p["M"] == 0 and p["total"] == 0
    # total tiles overflow int32
    with pytest.raises(moe_lib.MoeError) as e:
        moe_lib.moe_plan_build([2**30] * 1, 64, 8 * 200000, bn=16)
    assert e.value.status == -3
    # status code of an all-empty build is MOE_OK_EMPTY
    c = np.zeros(3, dtype=np.int32)
    blob = np.zeros(4096, dtype=np.int32)
    n = ctypes.c_int64()
    st = L.moe_plan_build(c.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 3, 64, 128, 128, 256, 0,
                          blob.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), blob.size, ctypes.byref(n))
    assert st == moe_lib.MOE_OK_EMPTY


def test_suggest_tile_in_library():
    """moe_plan_suggest_tile (C ABI): the automatic rule applied to an even spread of the expected rows —
    pair tiles (256 x 512) for Mix / DS-sized batches, one-CTA 128 x 256 for decode batches."""
    assert moe_lib.suggest_tile(4096 * 2, 8, 4096, 14336) == (256, 512)
    assert moe_lib.suggest_tile(8192 * 6, 64, 2048, 1408) == (256, 512)
    assert moe_lib.suggest_tile(2, 8, 4096, 14336) == (128, 256)
    assert moe_lib.suggest_tile(32, 8, 4096, 14336) == (128, 256)
    # the same as building the even-spread plan by hand
    counts = np.zeros(8, dtype=np.int32)
    counts[:8] = 100
    b = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 4096, 14336, 0, 0))
    assert moe_lib.suggest_tile(800, 8, 4096, 14336) == (b["bm"], b["bn"])
    bm, bn = ctypes.c_int32(), ctypes.c_int32()
    assert moe_lib.lib().moe_plan_suggest_tile(-1, 8, 64, 64, ctypes.byref(bm), ctypes.byref(bn)) == -1


def test_plan_launch_option_flags():
    """Launch options live in the plan (no environment switches): accepted, recorded in the blob,
    mutually exclusive grid options rejected."""
    counts = [5, 0, 300]
    for f in (moe_lib.MOE_GRID_BALANCED, moe_lib.MOE_GRID_STATIC, moe_lib.MOE_A_GATHER4, moe_lib.MOE_EPI_REGISTER):
        p = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 64, 256, 128, 128, f))
        assert p["flags"] == f
    with pytest.raises(moe_lib.MoeError):
        moe_lib.moe_plan_build(counts, 64, 256, 128, 128, moe_lib.MOE_GRID_BALANCED | moe_lib.MOE_GRID_STATIC)


def test_planner_catalog_matches_oracle():
    """Per-task tiling strategies: random catalogs of up to two rules; the kind of
    each expert's last row tile equals the oracle's tail_kind, and the mapping is unchanged."""
    rng = random.Random(21)
    for _ in range(200):
        E = rng.randint(1, 200)
        counts = np.array([0 if rng.random() < 0.3 else rng.randint(1, 3000) for _ in range(E)])
        bn = rng.choice([256, 512])
        kinds = [0, 1, 2, 3] if bn == 512 else [0, 1]
        rules = [(k_, rng.randint(0, 4) if k_ == 2 else rng.randint(0, 32) if k_ == 3 else rng.randint(0, 256))
                 for k_ in (rng.choice(kinds) for _ in range(rng.randint(0, 2)))]
        if rng.random() < 0.3:
            counts = np.where(counts > 0, counts % 7, 0)                   # many 1-6 row experts
        elif rng.random() < 0.3:
            counts = np.where(counts > 0, 256 * rng.randint(1, 5) + counts % 40, 0)   # short tails on full tiles
        N = 8 * rng.randint(1, 3000) if rng.random() < 0.5 else 512 * rng.randint(1, 30)
        _compare(counts, N, 256, bn, rng.choice(["max", "repeat"]), catalog=rules,
                 order=rng.choice(["natural", "half_interval", "light_last"]))
        if all(k_ != 2 for k_, _ in rules):                                # swap / wide: mapping unchanged
            base = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 64, N, 256, bn, catalog=()))
            got = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 64, N, 256, bn, catalog=rules))
            assert np.array_equal(base["prefix"], got["prefix"]) and np.array_equal(base["sigma"], got["sigma"])
    # worked examples: tails 1 and 200 under {SWAP, 64}; 256-row experts have no tail
    p = moe_lib.parse_plan_blob(moe_lib.moe_plan_build([1, 456, 256, 0, 64, 65], 64, 1024, 256, 512, catalog=[(1, 64)]))
    assert p["params"][:, 3].tolist() == [1, 0, 0, 0, 1, 0]
    with pytest.raises(moe_lib.MoeError):                              # swap tiles need CTA-pair 256-column blocks
        moe_lib.moe_plan_build([5, 5], 64, 1024, 128, 256, catalog=[(1, 64)])
    with pytest.raises(moe_lib.MoeError):
        moe_lib.moe_plan_build([5, 5], 64, 1024, 256, 512, catalog=[(1, 64), (0, 9), (1, 200)])
    with pytest.raises(moe_lib.MoeError):
        moe_lib.moe_plan_build([5, 5], 64, 1024, 256, 512, catalog=[(7, 64)])
    # RIDE: tails of <= m_max rows on experts with a full row tile, 512-column tiles inside N
    cnt = [1029, 1009, 256, 300, 257, 20, 0]
    p = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(cnt, 64, 14336, 256, 512, catalog=[(2, 4), (3, 32)]))
    assert p["params"][:, 3].tolist() == [3, 0, 0, 0, 3, 0, 0]
    base = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(cnt, 64, 14336, 256, 512, catalog=()))
    assert np.array_equal(base["prefix"], p["prefix"]) and np.array_equal(base["params"][:, 6:], p["params"][:, 6:])
    p = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(cnt, 64, 1408, 256, 512, catalog=[(3, 32)]))
    assert p["params"][:, 3].tolist() == [0] * 7                       # N % 512 != 0: no ride
    for bad in ([(3, 33)],):
        with pytest.raises(moe_lib.MoeError):
            moe_lib.moe_plan_build(cnt, 64, 14336, 256, 512, catalog=bad)
    with pytest.raises(moe_lib.MoeError):
        moe_lib.moe_plan_build(cnt, 64, 14336, 256, 256, catalog=[(3, 32)])


def test_planner_gemv_strategy_by_hand():
    """MOE_KIND_GEMV (Alg. 3's per-task strategy for <= 4-row tasks): whole tasks of
    m <= m_max < 256 rows get kind 2 and no tiles — they leave TilePrefix and sigma; a 257-row expert's
    1-row tail stays a tile (GEMV covers whole tasks only); wide pair tiles only, m_max <= 4."""
    counts = [1, 456, 4, 0, 5, 257, 3]
    N = 16384                                                              # 32 column tiles of 512
    p = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 64, N, 256, 512, catalog=[(2, 4), (1, 64)]))
    assert p["params"][:, 3].tolist() == [2, 0, 2, 0, 1, 1, 2]
    assert p["M"] == 3 and p["sigma"][:3].tolist() == [1, 4, 5]           # experts 1, 4, 5 have tiles
    assert p["total"] == (2 + 1 + 2) * 32 >= 128                          # the other tasks' tiles cover GEMV
    # fewer than MOE_GEMV_MIN_TILES other tiles: the GEMV candidates fall through to the next rule
    q = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(counts, 64, 1024, 256, 512, catalog=[(2, 4), (1, 64)]))
    assert q["params"][:, 3].tolist() == [1, 0, 1, 0, 1, 1, 1] and q["M"] == 6
    q = moe_lib.parse_plan_blob(moe_lib.moe_plan_build([2, 0, 1], 64, 1024, 256, 512, catalog=[(2, 4)]))
    assert q["M"] == 2 and q["params"][:, 3].tolist() == [0, 0, 0]
    for bad in ([(2, 5)], [(2, 4)]):
        with pytest.raises(moe_lib.MoeError):
            moe_lib.moe_plan_build([1, 1], 64, 1024, 256, 256 if bad == [(2, 4)] else 512, catalog=bad)


def test_tile_catalog_env_override():
    """MOE_TILE_CATALOG overrides the catalog of plans built without an explicit one (read by the
    binding at import; the library reads no environment)."""
    import subprocess
    import sys
    M = moe_lib
    assert M.parse_catalog("default") is None and M.parse_catalog("none") == ()
    assert M.parse_catalog("2.4+1.64") == ((2, 4), (1, 64))
    with pytest.raises(ValueError):
        M.parse_catalog("1.16+1.32+2.4")
    code = ("import sys; sys.path.insert(0, %r); import paper_2501_16103_b200 as M; "
            "b = M.parse_plan_blob(M.moe_plan_build([1029, 1009, 1020, 1047, 1026, 1000, 1032, 1029], 4096, 14336, "
            "256, 512)); print(b['catalog'])") % ROOT
    out = {}
    for env in ("none", "1.64", ""):
        e = dict(os.environ, MOE_TILE_CATALOG=env)
        out[env] = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True,
                                  check=True).stdout.strip()
    assert out["none"] == "()"
    assert out["1.64"] == "((1, 64),)"
    assert out[""] == str(M.DEFAULT_CATALOG)


def test_ep_peer_create_rejects_decode_tiles_before_touching_the_device():
    """ADVICE (round 1, low): the peer step's GEMM stores through row pointers, which have no bm = 64 form —
    moe_ep_peer_create refuses it up front (argument checks run before any CUDA call, so this runs on CPU)."""
    L = moe_lib.lib()
    out = ctypes.c_void_p()
    blob = (ctypes.c_uint8 * 4096)()
    st = L.moe_ep_peer_create(0, 2, 8, 64, 256, 16, 2, 8192, 8192, ctypes.byref(out), blob)
    assert moe_lib.MOE_ERR[st] == "UNSUPPORTED" and not out.value
    assert b"bm = 64" in L.moe_last_error()


def test_gemv_share_rule():
    """MOE_GEMV_MIN_SHARE: a handful of <= 4-row experts next to a long launch stay tiles (their
    GEMV units' serial K streams outlast the launch: measured 223 -> 343 us on the DeepSeek shape with four such
    experts), many of them (the paper's worst case) become GEMV units; host planner = oracle."""
    ds = synth.CONFIGS["ds"]
    cnt = [int(x) for x in np.bincount(synth.route(ds, 0).ravel(), minlength=ds.E) if x > 0] + [1, 2, 3, 4]
    p = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(cnt, ds.H, ds.N, 256, 512))
    assert (p["params"][:, 3] == moe_lib.MOE_KIND_GEMV).sum() == 0
    assert [t["kind"] for t in omoe.plan(cnt, ds.N, 256, 512, catalog=moe_lib.DEFAULT_CATALOG)["tasks"]] == \
        p["params"][:, 3].tolist()
    pw = synth.CONFIGS["paper_worst"]
    cw = np.bincount(synth.route(pw, 0).ravel(), minlength=pw.E)
    q = moe_lib.parse_plan_blob(moe_lib.moe_plan_build(cw, pw.H, pw.N, 256, 512))
    assert (q["params"][:, 3] == moe_lib.MOE_KIND_GEMV).sum() == 56
