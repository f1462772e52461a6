"""GPU parity of the FP8 E4M3 expert GEMM (moe_gemm_fp8, include/moe_sm100_fp8.h) against the fp64
oracle (oracle/fp8.py) on the same seeded E4M3 codes (synth/fp8.py).

Bar: integer-valued codes with fp32 output and power-of-two scales are bit-exact (|partial sums|
<= 16 H < 2^24); the "normal" codes meet the north-star tolerance max|d| <= 1e-2 (|ref| + 1),
relative Frobenius <= 2e-3 (fp32 accumulation of exact E4M3 products).
"""
import numpy as np
import pytest
import torch

import paper_2501_16103_b200 as M
import synth
from oracle import fp8 as ofp8
from oracle import moe as omoe
from synth import fp8 as sfp8

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def device():
    from paper_2501_16103_b200 import build
    build.build()
    n, ma, mi = M.moe_device_info()
    assert (ma, mi) == (10, 0), "needs sm_100"
    return n


def tol_check(Y, ref, tag=""):
    Y = torch.as_tensor(Y, dtype=torch.float64)
    ref = torch.as_tensor(ref, dtype=torch.float64)
    d = (Y - ref).abs()
    worst = (d / (1e-2 * (ref.abs() + 1))).max().item() if d.numel() else 0.0
    rel = ((Y - ref).norm() / ref.norm().clamp_min(1e-30)).item() if d.numel() else 0.0
    assert worst <= 1.0, f"{tag}: max |d| / (1e-2 (|ref|+1)) = {worst}"
    assert rel <= 2e-3, f"{tag}: rel Frobenius {rel}"


def _run(ids, Xc, Wc, E, bm, bn, scale, out_dtype, device_plan=False, csr_rows=False):
    topk = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)).cuda()
    H, N = Xc.shape[1], Wc.shape[2]
    Xd, Wd = torch.from_numpy(Xc).cuda(), torch.from_numpy(Wc).cuda()
    sc = torch.from_numpy(scale).cuda() if scale is not None else None
    if device_plan:
        plan = M.Plan(None, H, N, bm, bn, E=E)
        counts, row_off, tok, slot, _ = M.moe_route(topk, E, plan=plan)
    else:
        counts, row_off, tok, slot, _ = M.moe_route(topk, E)
        plan = M.Plan(counts.cpu().numpy(), H, N, bm, bn)
    Y = torch.full((tok.numel(), N), float("nan"), dtype=out_dtype, device="cuda")
    if csr_rows:                                   # token_idx NULL: X rows already in CSR order
        Xg = Xd[tok.long()].contiguous()
        M.moe_gemm_fp8(plan, Xg, None, Wd, sc, Y=Y)
    else:
        M.moe_gemm_fp8(plan, Xd, tok, Wd, sc, Y=Y)
    torch.cuda.synchronize()
    return Y.cpu().double().numpy()


CASES = [   # T, E, k, H, N
    (16, 4, 2, 128, 128),           # tiny, K = one block
    (300, 5, 2, 208, 256),          # K tail (208 = 128 + 80), several row tiles
    (64, 16, 4, 144, 1408),         # DeepSeek width: N = 2.75 x 512, tails of 1..31 rows
    (1, 8, 2, 4096, 1024),          # decode: one token, long K
    (700, 3, 2, 256, 1024),         # several 256-row tiles per expert
    (2048, 4, 2, 64, 640),          # K < one block, ragged column tile
]
TILES = [(128, 128), (128, 256), (256, 256), (256, 512)]


@pytest.mark.parametrize("T,E,k,H,N", CASES)
@pytest.mark.parametrize("bm,bn", TILES)
@pytest.mark.parametrize("mode", ["int", "int_bf16", "normal"])
def test_fp8_gemm_ragged(T, E, k, H, N, bm, bn, mode):
    gen = "int" if mode.startswith("int") else "normal"
    ids = synth.route_gumbel(T + E, T, E, k)
    Xc, Wc = sfp8.make_x_fp8(T + E, T, H, gen), sfp8.make_w_fp8(T + E, E, H, N, gen)
    # power-of-two scales (exact); "normal" carries W's 1/sqrt(H) magnitude in the scale
    scale = sfp8.w_scale(E, H, gen) * (2.0 ** (np.arange(E) % 3 - 1)).astype(np.float32)
    out = torch.bfloat16 if mode == "int_bf16" else torch.float32
    Y = _run(ids, Xc, Wc, E, bm, bn, scale, out)
    rc, rr, rt, rs = omoe.buckets(ids, E)
    ref = ofp8.expert_gemm_fp8(Xc, Wc, rt, rr, scale)
    assert not np.isnan(Y).any(), "some Y element was never written"
    if mode == "int":
        assert np.array_equal(Y, ref)
    elif mode == "int_bf16":
        assert np.array_equal(Y, torch.from_numpy(ref).to(torch.bfloat16).double().numpy())
    else:
        tol_check(Y, ref, f"fp8 {T},{E},{k},{H},{N} {bm}x{bn}")


@pytest.mark.parametrize("bm,bn", [(0, 0), (256, 512), (128, 256)])
@pytest.mark.parametrize("csr_rows", [False, True])
def test_fp8_device_planned_and_csr_rows(bm, bn, csr_rows):
    T, E, k, H, N = 777, 8, 2, 384, 1024
    ids = synth.route_gumbel(5, T, E, k, s=1.0, n_empty=2)
    Xc, Wc = sfp8.make_x_fp8(5, T, H, "int"), sfp8.make_w_fp8(5, E, H, N, "int")
    Y = _run(ids, Xc, Wc, E, bm, bn, None, torch.float32, device_plan=True, csr_rows=csr_rows)
    rc, rr, rt, rs = omoe.buckets(ids, E)
    assert np.array_equal(Y, ofp8.expert_gemm_fp8(Xc, Wc, rt, rr))


def test_fp8_unsupported_shapes_rejected():
    Xd = torch.zeros((4, 128), dtype=torch.uint8, device="cuda")
    tok = torch.zeros(1, dtype=torch.int32, device="cuda")
    Wd = torch.zeros((2, 128, 200), dtype=torch.uint8, device="cuda")
    with pytest.raises(M.MoeError):                # N % 128 != 0
        M.moe_gemm_fp8(M.Plan([1, 0], 128, 200, 128, 128), Xd, tok, Wd)
    Wd = torch.zeros((2, 128, 256), dtype=torch.uint8, device="cuda")
    for bm, bn, flags in ((64, 256, 0), (128, 64, 0), (256, 384, 0)):
        with pytest.raises(M.MoeError):
            M.moe_gemm_fp8(M.Plan([1, 0], 128, 256, bm, bn, flags), Xd, tok, Wd)


def test_fp8_ignores_swap_catalog():
    """The FP8 kernel runs every tile as MOE_KIND_WIDE: a plan whose catalog asks for swap-AB tails
    (built-in catalog, MOE_SPLIT_TAIL) still gives the exact result (same tile partition)."""
    T, E, k, H, N = 300, 5, 2, 256, 512
    ids = synth.route_gumbel(3, T, E, k)
    X8, W8 = sfp8.make_x_fp8(3, T, H, "int"), sfp8.make_w_fp8(3, E, H, N, "int")
    rc, rr, rt, rs = omoe.buckets(ids, E)
    ref = ofp8.expert_gemm_fp8(X8, W8, rt, rr)
    topk = torch.from_numpy(ids).cuda()
    counts, _, tok, _, _ = M.moe_route(topk, E)
    for flags, cat in ((M.MOE_SPLIT_TAIL, None), (0, None), (0, ((1, 256),))):
        plan = M.Plan(counts.cpu().numpy(), H, N, 256, 512, flags, catalog=cat)
        assert plan.catalog
        Y = M.moe_gemm_fp8(plan, torch.from_numpy(X8).cuda(), tok, torch.from_numpy(W8).cuda(), out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert np.array_equal(Y.cpu().double().numpy(), ref)


@pytest.mark.parametrize("cfg,bm,bn", [("mix", 0, 0), ("ds", 0, 0), ("dec16", 0, 0), ("dec1", 128, 256)])
def test_fp8_full_size_sampled(cfg, bm, bn):
    """BASELINE.json sizes in the launch configuration bench.py --dtype fp8 times; sampled outputs vs fp64."""
    c = synth.CONFIGS[cfg]
    ids = synth.route(c, 0)
    Xd = sfp8.make_x_fp8_torch(0, c.T, c.H, device="cuda")
    Wd = sfp8.make_w_fp8_torch(0, c.E, c.H, c.N, device="cuda")
    scale = sfp8.w_scale(c.E, c.H)
    topk = torch.from_numpy(ids).cuda()
    if bm == 0:
        bm, bn = M.suggest_tile(c.T * c.k, c.E, c.H, c.N)
    plan = M.Plan(None, c.H, c.N, bm, bn, E=c.E)
    counts, row_off, tok, slot, _ = M.moe_route(topk, c.E, plan=plan)
    Y = torch.full((tok.numel(), c.N), float("nan"), dtype=torch.bfloat16, device="cuda")
    M.moe_gemm_fp8(plan, Xd, tok, Wd, torch.from_numpy(scale).cuda(), Y=Y)
    torch.cuda.synchronize()
    rc, rr, rt, rs = omoe.buckets(ids, c.E)
    assert np.array_equal(tok.cpu().numpy(), rt)
    rng = np.random.default_rng(1)
    rows = []
    for e in range(c.E):
        a, b = int(rr[e]), int(rr[e + 1])
        if b > a:
            rows += sorted({a, b - 1, min(a + 127, b - 1), min(a + 128, b - 1)} | set(rng.integers(a, b, 4).tolist()))
    rows = np.array(rows)
    cols = np.unique(np.concatenate([rng.integers(0, c.N, 24), [0, c.N - 1, 255, 256, 511, 512]]))
    cols = cols[cols < c.N]
    ref = np.zeros((len(rows), len(cols)))
    for i, r in enumerate(rows):
        e = int(np.searchsorted(rr, r, side="right") - 1)
        ref[i] = ofp8.expert_gemm_fp8_entries(sfp8.x_fp8_rows(0, c.T, c.H, [rt[r]]),
                                              sfp8.w_fp8_columns(0, c.E, c.H, c.N, e, cols), scale[e])[0]
    got = Y[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu()
    tol_check(got, ref, cfg)
    assert not torch.isnan(Y.float()).any().item()


FP8_TILES = [(128, 128, 0), (128, 256, 0), (128, 128, 1), (256, 256, 0), (256, 512, 0),
             (256, 512, 8), (128, 256, 1 | 4)]          # 8 = MOE_ORDER_HALF_INTERVAL, 1 | 4 = PAD_REPEAT | ALTERNATING


@pytest.mark.parametrize("case", range(42))
def test_fp8_fuzz_tile_variants(case):
    """Random shapes (ragged K in 16-byte steps, N in 128-column steps, rows; empty experts; skewed or
    uniform routing), random FP8 tile variant, host- or device-built plan, gathered or CSR-ordered
    rows, fp32 / bf16 output, random power-of-two scales: bit-exact against the oracle."""
    rng = np.random.default_rng(7000 + case)
    E = int(rng.integers(1, 24))
    k = int(rng.integers(1, min(E, 6) + 1))
    T = int(rng.choice([1, 7, 64, 200, 513, 1500]))
    H = int(16 * rng.integers(1, 60))
    N = int(128 * rng.integers(1, 14))
    bm, bn, flags = FP8_TILES[case % len(FP8_TILES)]
    s = float(rng.choice([0.0, 1.2]))
    n_empty = int(rng.integers(0, max(1, E - k)))
    ids = synth.route_gumbel(case, T, E, k, s=s, n_empty=min(n_empty, E - k))
    Xc, Wc = sfp8.make_x_fp8(case, T, H, "int"), sfp8.make_w_fp8(case, E, H, N, "int")
    scale = (2.0 ** rng.integers(-3, 4, size=E)).astype(np.float32)
    topk = torch.from_numpy(ids).cuda()
    Xd, Wd = torch.from_numpy(Xc).cuda(), torch.from_numpy(Wc).cuda()
    device_plan = case % 4 == 1
    if device_plan:
        plan = M.Plan(None, H, N, bm, bn, flags, E=E)
        counts, row_off, tok, _, _ = M.moe_route(topk, E, plan=plan)
        launch = True
    else:
        counts, row_off, tok, _, _ = M.moe_route(topk, E)
        plan = M.Plan(counts.cpu().numpy(), H, N, bm, bn, flags)
        launch = plan.total_tiles > 0
    rc, rr, rt, rs = omoe.buckets(ids, E)
    ref = ofp8.expert_gemm_fp8(Xc, Wc, rt, rr, scale)
    out = torch.float32 if case % 2 == 0 else torch.bfloat16
    contiguous = case % 3 == 0
    Xin = Xd.index_select(0, tok.long()).contiguous() if contiguous else Xd
    Y = torch.full((tok.numel(), N), float("nan"), dtype=out, device="cuda")
    if launch:
        M.moe_gemm_fp8(plan, Xin, None if contiguous else tok, Wd, torch.from_numpy(scale).cuda(), Y=Y)
    torch.cuda.synchronize()
    got = Y.cpu().double().numpy()
    exp = ref if out == torch.float32 else torch.from_numpy(ref).to(torch.bfloat16).double().numpy()
    assert np.array_equal(got, exp), f"case {case}: T={T} E={E} k={k} H={H} N={N} tile={bm}x{bn} flags={flags}"
