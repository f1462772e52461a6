"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bar (north star): mapping / indexing bit-exact; Y within
max|d| <= 1e-2 * (|ref| + 1) and relative Frobenius <= 2e-3 for bf16 inputs
with fp32 accumulation; integer-valued inputs with fp32 output bit-exact.
"""
import numpy as np
import pytest
import torch

import paper_2501_16103_b200 as M
import synth
from oracle import moe as omoe
from synth import workloads as wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def device():
    from paper_2501_16103_b200 import build
    build.build()
    n, ma, mi = M.moe_device_info()
    assert (ma, mi) == (10, 0), "needs sm_100"
    return n


def tol_check(Y, ref, tag=""):
    Y = Y.double()
    ref = torch.as_tensor(ref, dtype=torch.float64)
    d = (Y - ref).abs()
    bound = 1e-2 * (ref.abs() + 1)
    worst = (d / bound).max().item() if d.numel() else 0.0
    rel = ((Y - ref).norm() / ref.norm().clamp_min(1e-30)).item() if d.numel() else 0.0
    assert worst <= 1.0, f"{tag}: max |d| / (1e-2 (|ref|+1)) = {worst}"
    assert rel <= 2e-3, f"{tag}: rel Frobenius {rel}"
    return worst, rel


def _inputs(T, E, k, H, N, seed, mode="normal", routing=None):
    ids = routing if routing is not None else synth.route_gumbel(seed, T, E, k)
    X = synth.make_x(seed, T, H, mode)
    W = synth.make_w(seed, E, H, N, mode)
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    Wd = torch.from_numpy(W).to(torch.bfloat16).cuda()
    return ids, X, W, Xd, Wd


def run_path(ids, Xd, Wd, E, bn=256, out_dtype=torch.float32, pad=M.MOE_PAD_MAX, bm=128, flags=0):
    topk = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)).cuda()
    counts, row_off, tok, slot, status = M.moe_route(topk, E)
    counts_h = counts.cpu().numpy()
    plan = M.Plan(counts_h, Xd.shape[1], Wd.shape[2], bm, bn, pad | flags)
    Y = torch.full((tok.numel(), Wd.shape[2]), float("nan"), dtype=out_dtype, device="cuda")
    M.moe_gemm(plan, Xd, tok, Wd, Y=Y)
    torch.cuda.synchronize()
    return Y, counts_h, row_off, tok, slot, plan, status


# ---------------------------------------------------------------------------- gather4 probe
def _expected_swizzled(X, rows, col0, H):
    out = np.zeros((128, 64), dtype=np.uint16)
    xb = torch.from_numpy(X).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    for r in range(128):
        for c in range(64):
            if col0 + c < H:
                out[r, c] = xb[rows[r], col0 + c]
    # 16-byte chunk c of row r lands at chunk position c ^ (r % 8)
    sw = np.zeros_like(out)
    for r in range(128):
        for ch in range(8):
            sw[r, 8 * (ch ^ (r % 8)): 8 * (ch ^ (r % 8)) + 8] = out[r, 8 * ch: 8 * ch + 8]
    return sw.view(np.uint8).reshape(-1)


@pytest.mark.parametrize("H,col0", [(128, 0), (128, 64), (72, 64)])
def test_probe_gather4_swizzle(H, col0):
    T = 300
    X = synth.make_x(1, T, H)
    rng = np.random.default_rng(H + col0)
    rows = rng.integers(0, T, size=128).astype(np.int32)
    rows[5] = rows[4]                                             # repeated rows are legal
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    got = M.moe_probe_gather4(Xd, torch.from_numpy(rows).cuda(), col0).cpu().numpy()
    assert np.array_equal(got, _expected_swizzled(X, rows, col0, H))


# ---------------------------------------------------------------------------- decode (bit-exact)
def _decode_ref(counts, N, bn, pad="max"):
    pl = omoe.plan(counts, N, 128, bn, pad_mode=pad)
    row_off = np.concatenate([[0], np.cumsum(counts)])
    out = []
    for B in range(pl["total"]):
        d = omoe.decode(pl, row_off, B)
        out.append((d["h"], d["task"], d["l"], d["rt"], d["ct"]))
    return np.array(out, dtype=np.int64).reshape(-1, 5)


@pytest.mark.parametrize("case", ["tiny_a", "mix", "ds", "worst", "random_many"])
@pytest.mark.parametrize("pad", ["max", "repeat"])
def test_decode_debug_bit_exact(case, pad):
    if case == "tiny_a":
        counts, N, bn = np.array([11, 0, 11, 10]), 128, 128
    elif case == "random_many":
        rng = np.random.default_rng(7)
        counts = np.where(rng.random(300) < 0.3, 0, rng.integers(1, 700, size=300))
        N, bn = 1024, 64
    else:
        c = synth.CONFIGS[{"mix": "mix", "ds": "ds", "worst": "paper_worst"}[case]]
        counts = np.bincount(synth.route(c, 0).ravel(), minlength=c.E)
        N, bn = c.N, 256 if case != "ds" else 128
    plan = M.Plan(counts, 64, N, 128, bn, M.MOE_PAD_REPEAT if pad == "repeat" else 0)
    got = M.moe_decode_debug(plan).cpu().numpy()
    ref = _decode_ref(counts, N, bn, pad)
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)


def test_decode_large_total():
    """~10^6 virtual tiles across 3 chunks of TilePrefix."""
    rng = np.random.default_rng(8)
    counts = rng.integers(0, 40000, size=70)
    counts[::9] = 0
    plan = M.Plan(counts, 64, 4096, 128, 16)
    got = M.moe_decode_debug(plan).cpu().numpy()
    pl = M.parse_plan_blob(plan.blob())
    # independent enumeration of the lattice (sigma order, rt fastest)
    ref = []
    h = 0
    for e in range(70):
        if counts[e] == 0:
            continue
        R, C = -(-counts[e] // 128), 4096 // 16
        l = np.arange(R * C)
        ref.append(np.stack([np.full(R * C, h), np.full(R * C, e), l, l % R, l // R], axis=1))
        h += 1
    ref = np.concatenate(ref)
    assert pl["total"] == len(ref) and len(ref) > 900_000
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------------------- route (bit-exact)
@pytest.mark.parametrize("cfg", ["tiny", "mix", "ds", "paper_worst", "dec1", "dec16", "dec256", "ep"])
def test_route_bit_exact(cfg):
    c = synth.CONFIGS[cfg]
    ids = synth.route(c, 0)
    counts, row_off, tok, slot, status = M.moe_route(torch.from_numpy(ids).cuda(), c.E)
    rc, rr, rt, rs = omoe.buckets(ids, c.E)
    assert counts.cpu().numpy().tolist() == rc.tolist()
    assert row_off.cpu().numpy().tolist() == rr.tolist()
    assert tok.cpu().numpy().tolist() == rt.tolist()
    assert slot.cpu().numpy().tolist() == rs.tolist()
    assert status.item() == 0


def test_route_flags_bad_ids_and_empty():
    ids = np.array([[0, 1], [2, 2], [5, 1]], dtype=np.int32)          # duplicate and out-of-range
    counts, row_off, tok, slot, status = M.moe_route(torch.from_numpy(ids).cuda(), 4)
    assert status.item() == 1
    assert counts.cpu().tolist() == [1, 2, 1, 0]
    assert tok.cpu().tolist()[:4] == [0, 0, 2, 1]
    ids = np.zeros((0, 2), dtype=np.int32)
    counts, row_off, tok, slot, status = M.moe_route(torch.zeros((0, 2), dtype=torch.int32, device="cuda"), 4)
    assert counts.cpu().tolist() == [0, 0, 0, 0] and row_off.cpu().tolist() == [0] * 5


# ---------------------------------------------------------------------------- GEMM
@pytest.mark.parametrize("bm,bn,flags", [(128, 128, 0), (256, 128, 0), (256, 256, M.MOE_SPLIT_TAIL)])
def test_gemm_tiny_a_integer_bit_exact(bm, bn, flags):
    c = synth.CONFIGS["tiny"]
    ids = synth.route(c, 0)
    _, X, W, Xd, Wd = _inputs(c.T, c.E, c.k, c.H, c.N, 0, "int", routing=ids)
    Y, counts, row_off, tok, slot, plan, _ = run_path(ids, Xd, Wd, c.E, bn=bn, bm=bm, flags=flags)
    rc, rr, rt, rs = omoe.buckets(ids, c.E)
    ref = omoe.expert_gemm(X, W, rt, rr)
    assert counts.tolist() == [11, 0, 11, 10]
    assert np.array_equal(Y.cpu().double().numpy(), ref)


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_gemm_tiny_b_random(out_dtype):
    c = synth.CONFIGS["tiny_b"]
    ids = synth.route(c, 3)
    _, X, W, Xd, Wd = _inputs(c.T, c.E, c.k, c.H, c.N, 3, routing=ids)
    Y, *_ = run_path(ids, Xd, Wd, c.E, bn=128, out_dtype=out_dtype)
    rc, rr, rt, rs = omoe.buckets(ids, c.E)
    tol_check(Y.cpu(), omoe.expert_gemm(X, W, rt, rr), "tiny_b")


def test_gemm_identity_weights_bf16_exact():
    """W[e] = (e+1) I => Y row = (e+1) X[token] exactly, even with bf16 output."""
    T, E, k, H = 200, 4, 2, 128
    ids = synth.route_gumbel(2, T, E, k)
    X = synth.make_x(2, T, H, "int")
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    Wd = synth.make_w_torch(0, E, H, H, "identity", device="cuda")
    Y, counts, row_off, tok, *_ = run_path(ids, Xd, Wd, E, bn=128, out_dtype=torch.bfloat16)
    tok_h = tok.cpu().numpy()
    ro = row_off.cpu().numpy()
    exp = np.zeros((len(tok_h), H))
    for e in range(E):
        exp[ro[e]:ro[e + 1]] = (e + 1) * X[tok_h[ro[e]:ro[e + 1]]]
    assert np.array_equal(Y.cpu().double().numpy(), exp)


RAGGED = [
    (300, 5, 2, 200, 136, 128),     # K tail (200 = 3*64 + 8), N tail, ragged row tiles
    (513, 7, 3, 256, 512, 256),     # several row tiles per expert, exact N tiles
    (64, 16, 4, 128, 176, 176),     # bn not a multiple of 64 (3 W boxes, 176 used)
    (1, 8, 2, 4096, 1024, 256),     # decode: one token
    (2000, 3, 1, 64, 8, 16),        # smallest N tile
]
RAGGED_PAIR = [
    (300, 5, 2, 200, 136, 128),     # pair tiles: second CTA often has no valid rows
    (700, 3, 2, 256, 512, 256),     # several pair row tiles per expert
    (64, 16, 4, 128, 352, 224),     # bn/2 = 112: N half not a multiple of 64
    (1, 8, 2, 4096, 1024, 256),
    (1500, 4, 1, 128, 200, 32),     # smallest pair N tile, N % 64 != 0 (3-D W map)
]


RAGGED_SPLIT = [                    # MOE_SPLIT_TAIL: 256-row pair body tiles + swap-AB tail tiles
    (300, 5, 2, 200, 136),          # tails only / N < 256
    (700, 3, 2, 256, 512),          # body + tails
    (64, 16, 4, 128, 352),          # tails of 1..31 rows, N tail
    (1, 8, 2, 4096, 1024),          # decode: one-token tails
    (1500, 4, 1, 128, 200),         # 3-D W map (N % 64 != 0)
    (2048, 4, 2, 64, 256),          # 1024 rows/expert on average, tails of all sizes
]


RAGGED_WIDE = [                     # bm = 256, bn = 512: two N = 256 MMA blocks per tile
    (300, 5, 2, 200, 136),          # N < 256: the second block lies wholly past N
    (700, 3, 2, 256, 1024),         # several row tiles, exact N tiles
    (64, 16, 4, 128, 1408),         # N = 2.75 x 512 (DeepSeek-V2-Lite width)
    (1, 8, 2, 4096, 1024),          # decode: one token
    (1500, 4, 1, 128, 200),         # 3-D W map (N % 64 != 0)
    (2048, 4, 2, 64, 1536),         # 1024 rows/expert on average
]
RAGGED_DECODE = [                   # bm = 64 decode tiles (swap-AB, one CTA): any rows, 64 per tile
    (1, 8, 2, 4096, 1024),          # one token
    (40, 8, 2, 200, 136),           # K tail, N tail (3-D W map), ~10 rows per expert
    (300, 5, 2, 256, 512),          # several 64-row tiles per expert
    (64, 16, 4, 128, 1408),
]
RAGGED_WIDE_BN = [                  # wide tiles narrower than 512: blocks of bn/2 (not a multiple of 32 / 64)
    (300, 5, 2, 200, 1408, 480),    # DS width: 3 x 480, block 240 = 7.5 epilogue chunks
    (513, 7, 3, 256, 1000, 352),    # block 176: 2.75 W chunks per CTA half-block
    (64, 16, 4, 128, 600, 320),
]


@pytest.mark.parametrize("T,E,k,H,N,bn,bm,a_path,flags",
                         [c + (128, "0", 0) for c in RAGGED] + [c + (128, "1", 0) for c in RAGGED]
                         + [c + (256, "1", 0) for c in RAGGED_PAIR]
                         + [c + (256, 256, "1", M.MOE_SPLIT_TAIL) for c in RAGGED_SPLIT]
                         + [c + (512, 256, a, 0) for c in RAGGED_WIDE for a in ("0", "1")]
                         + [c + (512, 256, "1", M.MOE_SPLIT_TAIL) for c in RAGGED_SPLIT]
                         + [c + (512, 256, "0", M.MOE_SPLIT_TAIL) for c in RAGGED_SPLIT]   # pair gather4 + swap tails
                         + [c + (512, 256, "0", M.MOE_SCHED_DYNAMIC | M.MOE_ORDER_HALF_INTERVAL) for c in RAGGED_WIDE]
                         + [c[:5] + (c[5], 256, "1", f) for c in RAGGED_WIDE_BN for f in (0, M.MOE_SPLIT_TAIL)]
                         + [c + (256, 64, "1", 0) for c in RAGGED_DECODE])
@pytest.mark.parametrize("mode", ["int", "int_bf16", "normal"])
def test_gemm_ragged(T, E, k, H, N, bn, bm, a_path, flags, mode):
    if a_path == "0":                                  # A staging path: gather4 (plan option) / cp.async
        flags |= M.MOE_A_GATHER4
    ids, X, W, Xd, Wd = _inputs(T, E, k, H, N, T + E, "int" if mode == "int_bf16" else mode)
    # int_bf16: bf16 output (the TMA-store epilogue for full 32-row quarters): the exact integer
    # accumulator rounded once to bf16, compared bit for bit with the fp64 reference so rounded.
    out = torch.bfloat16 if mode == "int_bf16" else torch.float32
    Y, counts, row_off, tok, *_ = run_path(ids, Xd, Wd, E, bn=bn, bm=bm, flags=flags, out_dtype=out)
    rc, rr, rt, rs = omoe.buckets(ids, E)
    ref = omoe.expert_gemm(X, W, rt, rr)
    Yh = Y.cpu().double().numpy()
    assert not np.isnan(Yh).any(), "some Y element was never written"
    if mode == "int_bf16":
        assert np.array_equal(Yh, torch.from_numpy(ref).to(torch.bfloat16).double().numpy())
    elif mode == "int":
        assert np.array_equal(Yh, ref)
    else:
        tol_check(torch.from_numpy(Yh), ref, f"ragged {T},{E},{k},{H},{N},{bn}")


def test_gemm_empty_plan_no_launch():
    Xd = torch.zeros((4, 64), dtype=torch.bfloat16, device="cuda")
    Wd = torch.zeros((3, 64, 128), dtype=torch.bfloat16, device="cuda")
    plan = M.Plan([0, 0, 0], 64, 128, 128, 128)
    assert plan.status == M.MOE_OK_EMPTY
    tok = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = M.lib().moe_gemm(plan.handle, Xd.data_ptr(), 4, tok.data_ptr(), Wd.data_ptr(), Xd.data_ptr(), 0,
                          M._stream())
    assert st == M.MOE_OK_EMPTY


def test_gemm_misaligned_rejected():
    Xd = torch.zeros((4, 72), dtype=torch.bfloat16, device="cuda")
    Wd = torch.zeros((3, 64, 128), dtype=torch.bfloat16, device="cuda")
    plan = M.Plan([1, 0, 0], 64, 128, 128, 128)
    tok = torch.zeros(1, dtype=torch.int32, device="cuda")
    Y = torch.zeros((1, 129), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(M.MoeError):
        M.moe_gemm(plan, Xd[:, 1:].contiguous()[:, :64].contiguous(), tok, Wd, Y=Y[:, 1:])


# ---------------------------------------------------------------------------- full-size sampled parity
def _sample_rows(row_off, counts, rng, per_expert=6):
    rows = []
    for e in range(len(counts)):
        if counts[e] == 0:
            continue
        a, b = int(row_off[e]), int(row_off[e + 1])
        cand = {a, b - 1, min(a + 127, b - 1), min(a + 128, b - 1)}
        cand |= set(rng.integers(a, b, size=per_expert).tolist())
        rows += sorted(cand)
    return np.array(rows)


@pytest.mark.parametrize("cfg,bn,bm,flags", [("mix", 256, 128, 0), ("mix", 256, 256, 0), ("mix", 0, 0, 0),
                                             ("mix", 512, 256, 0), ("ds", 512, 256, 0), ("paper_balanced", 0, 0, 0),
                                             ("dec16", 512, 256, 0), ("paper_worst", 512, 256, 0),
                                             ("mix", 512, 256, 2), ("ds", 512, 256, 2), ("paper_worst", 512, 256, 2),
                                             ("ds", 0, 0, 0), ("ds", 480, 256, 2),
                                             ("dec16", 256, 64, 0), ("dec256", 256, 64, 0), ("dec1", 256, 64, 0),
                                             ("mix", 256, 256, 2), ("ds", 128, 128, 0), ("ds", 256, 256, 0),
                                             ("ds", 256, 256, 2), ("dec16", 256, 128, 0), ("dec16", 256, 0, 0),
                                             ("dec16", 256, 256, 2), ("paper_worst", 256, 256, 0),
                                             ("paper_worst", 256, 256, 2)])
def test_gemm_full_size_sampled(cfg, bn, bm, flags):
    """BASELINE.json sizes, the launch configuration bench.py times; sampled outputs vs fp64."""
    c = synth.CONFIGS[cfg]
    seed = 0
    ids = synth.route(c, seed)
    Xd = synth.make_x_torch(seed, c.T, c.H, device="cuda")
    Wd = synth.make_w_torch(seed, c.E, c.H, c.N, device="cuda")
    Y, counts, row_off, tok, *_ = run_path(ids, Xd, Wd, c.E, bn=bn, out_dtype=torch.bfloat16, bm=bm, flags=flags)
    rc, rr, rt, rs = omoe.buckets(ids, c.E)
    assert np.array_equal(tok.cpu().numpy(), rt)
    rng = np.random.default_rng(1)
    rows = _sample_rows(rr, rc, rng)
    cols = np.unique(np.concatenate([rng.integers(0, c.N, 40), [0, c.N - 1, 255, 256, 511, 512]]))
    cols = cols[cols < c.N]
    ref = omoe.expert_gemm_entries(lambda t: wl.x_rows(seed, c.T, c.H, [t])[0],
                                   lambda e, cs: wl.w_columns(seed, c.E, c.H, c.N, e, cs),
                                   rt, rr, rows, cols)
    got = Y[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu()
    tol_check(got, ref, cfg)
    # every row written (NaN sentinel) — the exactly-once cover follows from the bit-exact decode
    assert not torch.isnan(Y.float()).any().item()


# ---------------------------------------------------------------------------- device-side planner
ORDER_FLAG = {"natural": 0, "alternating": M.MOE_ORDER_ALTERNATING, "half_interval": M.MOE_ORDER_HALF_INTERVAL,
              "light_last": M.MOE_ORDER_LIGHT_LAST}


def _device_plan_blob(counts, N, bm, bn, pad, H=64, split=0, order="natural"):
    E = len(counts)
    plan = M.Plan(None, H, N, bm, bn, (M.MOE_PAD_REPEAT if pad == "repeat" else 0) | (M.MOE_SPLIT_TAIL if split else 0)
                  | ORDER_FLAG[order], E=E)
    plan.update_device(torch.tensor(np.asarray(counts), dtype=torch.int32, device="cuda"))
    st = plan.sync()
    return plan, st, M.parse_plan_blob(plan.blob())


@pytest.mark.parametrize("pad", ["max", "repeat"])
@pytest.mark.parametrize("bm,bn,split,order", [(128, 256, 0, "natural"), (256, 256, 0, "natural"), (128, 48, 0, "natural"),
                                               (256, 96, 0, "natural"), (256, 256, 1, "natural"),
                                               (256, 512, 0, "natural"), (256, 512, 0, "half_interval"),
                                               (256, 512, 1, "natural"),
                                               (128, 256, 0, "alternating"), (256, 256, 0, "half_interval"),
                                               (256, 512, 0, "light_last"), (128, 256, 0, "light_last")])
def test_plan_device_bit_exact(pad, bm, bn, split, order):
    rng = np.random.default_rng(bm + bn)
    cases = [np.array([11, 0, 11, 10]), np.zeros(5, dtype=np.int64), np.array([1]), np.array([256, 512, 5, 0, 300]),
             np.where(rng.random(1024) < 0.3, 0, rng.integers(1, 3000, size=1024)),
             np.bincount(synth.route(synth.CONFIGS["ds"], 0).ravel(), minlength=64)]
    for counts in cases:
        N = 1408
        plan, st, b = _device_plan_blob(counts, N, bm, bn, pad, split=split, order=order)
        # the library's built-in catalog, stated independently: {GEMV, 4} on wide pair plans
        catalog = ((2, 4),) if (bm == 256 and bn > 256) else ()
        ref = omoe.plan(counts, N, bm, bn, pad_mode=pad, split_tail=bool(split), order=order, catalog=catalog)
        E = len(counts)
        nt = E
        assert b["M"] == ref["M"] and b["total"] == ref["total"]
        assert st == (M.MOE_OK_EMPTY if ref["M"] == 0 else M.MOE_OK)
        assert b["M_pad"] == (32 if nt <= 32 else -(-nt // 32) * 32)
        assert b["prefix"][: ref["M"]].tolist() == ref["prefix"]
        padv = (ref["prefix"][-1] if ref["M"] else 2**31 - 1) if pad == "repeat" else 2**31 - 1
        assert (b["prefix"][ref["M"]:] == padv).all()
        assert b["sigma"][: ref["M"]].tolist() == ref["sigma"]
        assert b["row_off"].tolist() == np.concatenate([[0], np.cumsum(counts)]).tolist()
        host = M.parse_plan_blob(M.moe_plan_build(counts, 64, N, bm, bn, (M.MOE_PAD_REPEAT if pad == "repeat" else 0)
                                                  | (M.MOE_SPLIT_TAIL if split else 0) | ORDER_FLAG[order]))
        assert np.array_equal(b["params"], host["params"])


def test_plan_device_overflow_reported():
    plan, _, _ = None, None, None
    p = M.Plan(None, 64, 1 << 20, 128, 16, E=3)
    p.update_device(torch.tensor([2**30, 2**30, 5], dtype=torch.int32, device="cuda"))
    with pytest.raises(M.MoeError) as e:
        p.sync()
    assert e.value.status == -3


@pytest.mark.parametrize("bm", [128, 256, 0])
@pytest.mark.parametrize("T,E,k,H,N,bn", [(300, 5, 2, 200, 136, 128), (513, 7, 3, 256, 512, 256), (1, 8, 2, 4096, 1024, 256)])
def test_gemm_device_planned(T, E, k, H, N, bn, bm):
    ids, X, W, Xd, Wd = _inputs(T, E, k, H, N, T + E + 1, "int")
    topk = torch.from_numpy(ids).cuda()
    Yout = torch.full((T * k, N), float("nan"), dtype=torch.float32, device="cuda")
    Y, counts, row_off, tok, slot, plan = M.moe_forward(topk, Xd, Wd, E, bm=bm, bn=bn, Y=Yout, device_plan=True)
    torch.cuda.synchronize()
    rc, rr, rt, rs = omoe.buckets(ids, E)
    assert np.array_equal(Y.cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr))
    # a second step on the same plan object with different routing
    ids2 = synth.route_gumbel(99, T, E, k)
    Y2, *_ = M.moe_forward(torch.from_numpy(ids2).cuda(), Xd, Wd, E, plan=plan, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rc, rr, rt, rs = omoe.buckets(ids2, E)
    assert np.array_equal(Y2.cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr))


@pytest.mark.parametrize("bm,bn", [(256, 512), (0, 0)])
@pytest.mark.parametrize("T,E,k,H,N", [(300, 5, 2, 200, 136), (513, 7, 3, 256, 1024), (2048, 6, 2, 128, 1408)])
def test_gemm_device_planned_wide(T, E, k, H, N, bm, bn):
    """Device plan (M_pad = pad32(E), tile count read in-kernel) with wide tiles and bf16 output
    (TMA-store epilogue over a 2^31-row Y map): exact integers rounded once to bf16."""
    ids, X, W, Xd, Wd = _inputs(T, E, k, H, N, T + E + 2, "int")
    topk = torch.from_numpy(ids).cuda()
    Yout = torch.full((T * k, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    Y, counts, row_off, tok, slot, plan = M.moe_forward(topk, Xd, Wd, E, bm=bm, bn=bn, Y=Yout, device_plan=True)
    torch.cuda.synchronize()
    assert (plan.bm, plan.bn) == ((bm, bn) if bn else M.suggest_tile(T * k, E, H, N))
    rc, rr, rt, rs = omoe.buckets(ids, E)
    ref = torch.from_numpy(omoe.expert_gemm(X, W, rt, rr)).to(torch.bfloat16).double().numpy()
    assert np.array_equal(Y.cpu().double().numpy(), ref)


@pytest.mark.parametrize("order", ["alternating", "half_interval", "light_last"])
def test_gemm_ordering_invariance(order):
    """Y is bit-identical under every §4.2 ordering (paper worst case, integer data)."""
    c = synth.CONFIGS["paper_worst"]
    ids = synth.route(c)
    T, H, N = 512, 256, 512                                  # the routing pattern at a smaller width
    ids = np.ascontiguousarray(ids[:T])
    X = synth.make_x(4, T, H, "int")
    W = synth.make_w(4, c.E, H, N, "int")
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    Wd = torch.from_numpy(W).to(torch.bfloat16).cuda()
    Y0, *_ = run_path(ids, Xd, Wd, c.E, bn=256, bm=256)
    Y1, *_ = run_path(ids, Xd, Wd, c.E, bn=256, bm=256, flags=ORDER_FLAG[order])
    assert torch.equal(Y0, Y1)
    rc, rr, rt, rs = omoe.buckets(ids, c.E)
    assert np.array_equal(Y1.cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr))


def test_gemm_device_planned_all_empty():
    """A rank that receives no rows: the device plan has total 0 and the launch does nothing."""
    Xd = torch.zeros((4, 64), dtype=torch.bfloat16, device="cuda")
    Wd = torch.zeros((3, 64, 128), dtype=torch.bfloat16, device="cuda")
    plan = M.Plan(None, 64, 128, 128, 128, E=3)
    plan.update_device(torch.zeros(3, dtype=torch.int32, device="cuda"))
    tok = torch.zeros(1, dtype=torch.int32, device="cuda")
    Y = torch.full((1, 128), 7.0, dtype=torch.float32, device="cuda")
    M.moe_gemm(plan, Xd, tok, Wd, Y=Y)
    torch.cuda.synchronize()
    assert (Y == 7.0).all()


@pytest.mark.parametrize("cfg", ["tiny", "mix", "ds", "paper_worst", "dec1", "dec16", "dec256", "ep"])
def test_route_plan_fused_matches_separate(cfg):
    """moe_route_plan = moe_route + moe_plan_device, bit for bit (and both = the oracle)."""
    c = synth.CONFIGS[cfg]
    ids = torch.from_numpy(synth.route(c, 0)).cuda()
    plan_a = M.Plan(None, c.H, c.N, 0, 256, E=c.E)
    counts_a, row_off_a, tok_a, slot_a, st_a = M.moe_route(ids, c.E, plan=plan_a)
    counts_b, row_off_b, tok_b, slot_b, st_b = M.moe_route(ids, c.E)
    plan_b = M.Plan(None, c.H, c.N, 0, 256, E=c.E)
    plan_b.update_device(counts_b)
    plan_a.sync()
    plan_b.sync()
    assert torch.equal(counts_a, counts_b) and torch.equal(tok_a, tok_b) and torch.equal(slot_a, slot_b)
    assert np.array_equal(plan_a.blob(), plan_b.blob())
    rc, rr, rt, rs = omoe.buckets(synth.route(c, 0), c.E)
    assert tok_a.cpu().numpy().tolist() == rt.tolist()
    ref = omoe.plan(rc, c.N, plan_a.bm, 256)
    b = M.parse_plan_blob(plan_a.blob())
    assert b["total"] == ref["total"] and b["prefix"][: ref["M"]].tolist() == ref["prefix"]


def test_route_many_chunks_and_masked_slots():
    """> 1 chunk per expert, masked (negative) slots skipped, status only for real errors."""
    rng = np.random.default_rng(5)
    T, E, k = 5000, 37, 4
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    ids[rng.random((T, k)) < 0.2] = -1
    counts, row_off, tok, slot, status = M.moe_route(torch.from_numpy(ids).cuda(), E)
    assert status.item() == 0
    n = int(counts.sum().item())
    for e in range(E):
        a, b = int(row_off[e]), int(row_off[e + 1])
        got = tok[a:b].cpu().numpy().tolist()
        assert got == [t for t in range(T) if e in ids[t]]
    assert n == int((ids >= 0).sum())


@pytest.mark.parametrize("T,k,E,skew,small", [(20000, 3, 1024, 0.0, "1"), (8192, 6, 64, 1.2, "1"),
                                              (40000, 2, 64, 1.2, "1"), (32768, 2, 8, 0.0, "1"),
                                              (32769, 2, 8, 0.0, "1"), (3, 1, 1, 0.0, "1"), (3, 1, 1, 0.0, "0"),
                                              (1024, 2, 8, 0.0, "1"), (1024, 2, 8, 0.0, "0"), (1000, 8, 16, 1.2, "1"),
                                              (1, 2, 8, 0.0, "1"), (77, 3, 5, 0.0, "1"), (1025, 2, 8, 0.0, "1")])
def test_route_place_and_split_paths(T, k, E, skew, small):
    """chunks x experts <= 16K: histogram + fused scan/placement kernels (match_any groups);
    larger (20 chunks x 1024 experts): histogram + single-block scan + chunk x expert compaction;
    T <= 1024, E <= 16, k <= 8: the single-block small-batch kernel (MOE_ROUTE_NO_SMALL forces the
    multi-kernel path).  All must give the oracle's buckets exactly, with masked slots and invalid
    entries (out of range, repeated in a token's row) dropped and reported."""
    rng = np.random.default_rng(T + E)
    if skew > 0:
        ids = synth.route_gumbel(T, T, E, k, s=skew)
    else:
        ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    ids = ids.astype(np.int32)
    mask = rng.random((T, k)) < 0.1
    ids[mask] = -1                                           # masked slots: skipped silently
    bad_t = rng.integers(0, T, size=3)
    if k >= 2:
        ids[bad_t, 1] = np.where(ids[bad_t, 0] >= 0, ids[bad_t, 0], E)   # repeat or out of range
    counts, row_off, tok, slot, status = M.moe_route(torch.from_numpy(ids).cuda(), E,
                                                     route_flags=0 if small == "1" else M.MOE_ROUTE_NO_SMALL)
    # reference: drop masked, out-of-range and repeated entries; tokens ascending per expert
    lists = [[] for _ in range(E)]
    for t in range(T):
        seen = set()
        for j in range(k):
            e = int(ids[t, j])
            if e < 0 or e >= E or e in seen:
                continue
            seen.add(e)
            lists[e].append((t, j))
    assert counts.cpu().numpy().tolist() == [len(b) for b in lists]
    rt = [t for b in lists for (t, _) in b]
    rs = [j for b in lists for (_, j) in b]
    n = len(rt)
    assert tok.cpu().numpy()[:n].tolist() == rt
    assert slot.cpu().numpy()[:n].tolist() == rs
    assert row_off.cpu().numpy().tolist() == np.concatenate([[0], np.cumsum([len(b) for b in lists])]).tolist()
    assert status.item() == (1 if k >= 2 else 0)


@pytest.mark.parametrize("bm,bn,flags", [(128, 256, 0), (256, 256, 0), (256, 512, 0), (256, 512, M.MOE_SPLIT_TAIL),
                                         (256, 256, M.MOE_SPLIT_TAIL)])
@pytest.mark.parametrize("T,E,k,H,N", [(300, 5, 2, 200, 136), (700, 3, 2, 256, 1024), (1, 8, 2, 512, 640)])
def test_gemm_contiguous_rows_token_idx_null(T, E, k, H, N, bm, bn, flags):
    """token_idx NULL: X already in CSR row order (one tile TMA per stage) — the same Y, bit for
    bit, as gathering the same rows through the token-index array; exact vs the oracle (integers)."""
    ids, X, W, Xd, Wd = _inputs(T, E, k, H, N, T + N, "int")
    counts, row_off, tok, _, _ = M.moe_route(torch.from_numpy(ids).cuda(), E)
    plan = M.Plan(counts.cpu().numpy(), H, N, bm, bn, flags)
    Xc = Xd.index_select(0, tok.long()).contiguous()            # rows in CSR order
    Yc = M.moe_gemm(plan, Xc, None, Wd, out_dtype=torch.float32)
    Yg = M.moe_gemm(plan, Xd, tok, Wd, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(Yc, Yg)
    rc, rr, rt, rs = omoe.buckets(ids, E)
    assert np.array_equal(Yc.cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr))


@pytest.mark.parametrize("bm,bn", [(128, 256), (256, 512)])
def test_gemm_1024_experts(bm, bn):
    """M_pad = 1024 (32 warp-vote chunks per decode), most experts with 0-3 rows."""
    T, E, k, H, N = 1024, 1024, 4, 128, 256
    ids, X, W, Xd, Wd = _inputs(T, E, k, H, N, 1234, "int")
    Y, counts, row_off, tok, *_ = run_path(ids, Xd, Wd, E, bn=bn, bm=bm)
    rc, rr, rt, rs = omoe.buckets(ids, E)
    assert np.array_equal(Y.cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr))


TILE_VARIANTS = [(128, 256, 0), (128, 112, 0), (256, 256, 0), (256, 256, M.MOE_SPLIT_TAIL), (256, 512, 0),
                 (256, 512, M.MOE_SPLIT_TAIL), (256, 384, 0), (256, 480, M.MOE_SPLIT_TAIL), (64, 256, 0),
                 (256, 512, M.MOE_ORDER_HALF_INTERVAL), (128, 256, M.MOE_PAD_REPEAT | M.MOE_ORDER_ALTERNATING)]


@pytest.mark.parametrize("case", range(88))
def test_gemm_fuzz_tile_variants(case):
    """Random shapes (ragged K, N, rows; empty experts; a skewed or uniform routing) through a
    random tile variant: exact integers, fp32 and bf16 (TMA-store) outputs, gathered or
    CSR-ordered (token_idx NULL) rows — all bit-exact against the oracle."""
    rng = np.random.default_rng(1000 + case)
    E = int(rng.integers(1, 24))
    k = int(rng.integers(1, min(E, 6) + 1))
    T = int(rng.choice([1, 7, 64, 200, 513, 1500]))
    H = int(8 * rng.integers(1, 80))
    N = int(8 * rng.integers(1, 200))
    bm, bn, flags = TILE_VARIANTS[case % len(TILE_VARIANTS)]
    s = float(rng.choice([0.0, 1.2]))
    n_empty = int(rng.integers(0, max(1, E - k)))
    ids = synth.route_gumbel(case, T, E, k, s=s, n_empty=min(n_empty, E - k))
    X = synth.make_x(case, T, H, "int")
    W = synth.make_w(case, E, H, N, "int")
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    Wd = torch.from_numpy(W).to(torch.bfloat16).cuda()
    counts, row_off, tok, _, _ = M.moe_route(torch.from_numpy(ids).cuda(), E)
    plan = M.Plan(counts.cpu().numpy(), H, N, bm, bn, flags)
    rc, rr, rt, rs = omoe.buckets(ids, E)
    ref = omoe.expert_gemm(X, W, rt, rr)
    out = torch.float32 if case % 2 == 0 else torch.bfloat16
    contiguous = case % 3 == 0
    Xin = Xd.index_select(0, tok.long()).contiguous() if contiguous else Xd
    Y = torch.full((tok.numel(), N), float("nan"), dtype=out, device="cuda")
    if plan.total_tiles:
        M.moe_gemm(plan, Xin, None if contiguous else tok, Wd, Y=Y)
    torch.cuda.synchronize()
    got = Y.cpu().double().numpy()
    exp = ref if out == torch.float32 else torch.from_numpy(ref).to(torch.bfloat16).double().numpy()
    assert np.array_equal(got, exp), f"case {case}: T={T} E={E} k={k} H={H} N={N} tile={bm}x{bn} flags={flags}"


@pytest.mark.parametrize("case", range(24))
def test_forward_device_plan_fuzz(case):
    """moe_forward with the plan built on the device inside the routing kernels (M_pad = pad32(E),
    tile count read in-kernel), random shapes and tile variants, two steps on one plan."""
    rng = np.random.default_rng(5000 + case)
    E = int(rng.integers(1, 40))
    k = int(rng.integers(1, min(E, 4) + 1))
    T = int(rng.choice([1, 33, 300, 1100]))
    H = int(8 * rng.integers(1, 64))
    N = int(8 * rng.integers(1, 160))
    bm, bn, flags = TILE_VARIANTS[case % len(TILE_VARIANTS)]
    X = synth.make_x(case, T, H, "int")
    W = synth.make_w(case, E, H, N, "int")
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    Wd = torch.from_numpy(W).to(torch.bfloat16).cuda()
    plan = M.Plan(None, H, N, bm, bn, flags, E=E)
    for step in range(2):
        ids = synth.route_gumbel(case * 7 + step, T, E, k, s=1.2 if step else 0.0)
        Y, *_ = M.moe_forward(torch.from_numpy(ids).cuda(), Xd, Wd, E, plan=plan, out_dtype=torch.float32)
        torch.cuda.synchronize()
        rc, rr, rt, rs = omoe.buckets(ids, E)
        assert np.array_equal(Y.cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr)), f"case {case} step {step}"


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("bn", [512, 480])
def test_split_tail_consecutive_tail_tiles(out_dtype, bn):
    """Regression: with MOE_SPLIT_TAIL, a CTA pair running two swap-AB tail tiles in a row (here
    every expert has 300 rows = one body + one tail row tile, 80 tiles on 74 pairs, so pairs 1, 3
    and 5 take tail tiles v and v + 74) — the non-transposing epilogue warps used to run ahead
    into the next tile's tmem-empty barrier with fp32 output and corrupt block 1."""
    T, E, k, H, N = 1200, 8, 2, 64, 2560
    ids = synth.route_balanced(T, E, k)
    X, W = synth.make_x(5, T, H, "int"), synth.make_w(5, E, H, N, "int")
    Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    Y, counts, row_off, tok, *_ = run_path(ids, Xd, Wd, E, bn=bn, bm=256, flags=M.MOE_SPLIT_TAIL, out_dtype=out_dtype)
    rc, rr, rt, rs = omoe.buckets(ids, E)
    ref = omoe.expert_gemm(X, W, rt, rr)
    exp = ref if out_dtype == torch.float32 else torch.from_numpy(ref).to(torch.bfloat16).double().numpy()
    assert np.array_equal(Y.cpu().double().numpy(), exp)


# ---------------------------------------------------------------------------- per-task strategies + tile order
@pytest.mark.parametrize("case", range(40))
def test_catalog_and_dynamic_order_fuzz(case):
    """Mixed-kind plans (the catalog's WIDE / SWAP strategies for each expert's last row tile, P:213,
    P:251-253) under the static and the dynamic tile order: bit-exact on integer data, fp32 and bf16
    out, host and device plans, three launches on one plan (the dynamic counter resets each time)."""
    rng = np.random.default_rng(1000 + case)
    E = int(rng.integers(1, 24))
    k = int(rng.integers(1, min(E, 4) + 1))
    T = int(rng.integers(1, 1500))
    H = int(rng.choice([64, 128, 200, 512]))
    N = int(rng.choice([256, 512, 640, 1024, 1408]))
    bn = int(rng.choice([256, 512]))
    rules = [(int(rng.integers(0, 2)), int(rng.integers(0, 257))) for _ in range(int(rng.integers(0, 3)))]
    flags = int(rng.choice([0, M.MOE_SCHED_DYNAMIC])) | int(rng.choice([0, M.MOE_ORDER_HALF_INTERVAL]))
    out = torch.float32 if case % 2 else torch.bfloat16
    ids = synth.route_gumbel(case, T, E, k, s=float(rng.choice([0.0, 1.5])), n_empty=int(rng.integers(0, E - k + 1)))
    X, W = synth.make_x(case, T, H, "int"), synth.make_w(case, E, H, N, "int")
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    Wd = torch.from_numpy(W).to(torch.bfloat16).cuda()
    topk = torch.from_numpy(ids).cuda()
    rc, rr, rt, _ = omoe.buckets(ids, E)
    ref = omoe.expert_gemm(X, W, rt, rr)
    ref_t = torch.from_numpy(ref).to(out).double().numpy()
    device_plan = bool(case % 3 == 0)
    if device_plan:
        plan = M.Plan(None, H, N, 256, bn, flags, E=E, catalog=rules)
    else:
        counts, _, _, _, _ = M.moe_route(topk, E)
        plan = M.Plan(counts.cpu().numpy(), H, N, 256, bn, flags, catalog=rules)
        kinds = M.parse_plan_blob(plan.blob())["params"][:, 3]
        assert kinds.tolist() == [omoe.tail_kind(m, 256, rules) for m in rc]
    for rep in range(3):
        _, _, tok, _, _ = M.moe_route(topk, E, plan=plan if device_plan else None)
        Y = torch.full((T * k, N), float("nan"), dtype=out, device="cuda")
        M.moe_gemm(plan, Xd, tok, Wd, Y=Y)
        torch.cuda.synchronize()
        assert np.array_equal(Y.cpu().double().numpy(), ref_t), (rep, rules, flags, bn)


@pytest.mark.parametrize("cfg", ["paper_worst", "ds", "mix"])
def test_dynamic_order_full_size_graph(cfg):
    """The dynamic tile order at full size inside a CUDA graph replayed three times (device plan fused
    into the route, built-in catalog): sampled entries against the fp64 oracle, identical replays."""
    c = synth.CONFIGS[cfg]
    ids = synth.route(c, 0)
    topk = torch.from_numpy(ids).cuda()
    Xd = synth.make_x_torch(0, c.T, c.H, device="cuda")
    Wd = synth.make_w_torch(0, c.E, c.H, c.N, device="cuda")
    plan = M.Plan(None, c.H, c.N, 256, 512, M.MOE_SCHED_DYNAMIC, E=c.E)
    Y = torch.empty((c.T * c.k, c.N), dtype=torch.bfloat16, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        _, _, tok, _, _ = M.moe_route(topk, c.E, with_slot=False, plan=plan)
        M.moe_gemm(plan, Xd, tok, Wd, Y=Y)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        _, _, tok_g, _, _ = M.moe_route(topk, c.E, with_slot=False, plan=plan)
        M.moe_gemm(plan, Xd, tok_g, Wd, Y=Y)
    outs = []
    for _ in range(3):
        Y.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        outs.append(Y.clone())
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
    rc, rr, rt, _ = omoe.buckets(ids, c.E)
    rng = np.random.default_rng(2)
    rows = _sample_rows(rr, rc, rng, 3)
    cols = np.unique(np.concatenate([rng.integers(0, c.N, 16), [0, c.N - 1]]))
    ref = omoe.expert_gemm_entries(lambda t: wl.x_rows(0, c.T, c.H, [t])[0],
                                   lambda e, cs: wl.w_columns(0, c.E, c.H, c.N, e, cs), rt, rr, rows, cols)
    tol_check(outs[0][torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu(), ref, cfg)


@pytest.mark.parametrize("shape", [(700, 9, 3, 256, 1408), (2000, 16, 2, 128, 2560), (300, 5, 2, 512, 640),
                                   (4096, 64, 6, 128, 1408)])
@pytest.mark.parametrize("device_plan", [False, True])
def test_half_tiles_last_order_is_invisible(shape, device_plan):
    """The dynamic fetch orders of wide tiles — MOE_SCHED_HALF_LAST (each task's <= 128-row
    last row tile after every full tile), the default narrow-column-block-last order (N % 512 != 0 here for
    two shapes) and MOE_SCHED_PLAN_ORDER — give bit-identical, exact Y."""
    T, E, k, H, N = shape
    ids = synth.route_gumbel(T, T, E, k, s=1.1, n_empty=1)
    X, W = synth.make_x(T, T, H, "int"), synth.make_w(T, E, H, N, "int")
    Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    topk = torch.from_numpy(ids).cuda()
    outs = []
    for flags in (M.MOE_SCHED_HALF_LAST, 0, M.MOE_SCHED_PLAN_ORDER):       # 0: narrow column block last
        if device_plan:
            plan = M.Plan(None, H, N, 256, 512, flags, E=E)
            counts, row_off, tok, _, _ = M.moe_route(topk, E, plan=plan)
        else:
            counts, row_off, tok, _, _ = M.moe_route(topk, E)
            plan = M.Plan(counts.cpu().numpy(), H, N, 256, 512, flags)
        Y = torch.full((tok.numel(), N), float("nan"), device="cuda")
        for _ in range(2):
            M.moe_gemm(plan, Xd, tok, Wd, Y=Y)
        outs.append(Y)
    torch.cuda.synchronize()
    rc, rr, rt, _ = omoe.buckets(ids, E)
    assert np.array_equal(outs[0].cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr))
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
