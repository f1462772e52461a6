"""GPU parity of MOE_KIND_GEMV tasks (Alg. 3's per-task strategy for <= 4-row tasks): tasks
of at most m_max rows have no tiles; the epilogue warps of the wide pair kernel compute them as CUDA-core
GEMVs between their accumulator drains, from a global unit queue.

Checks against the fp64 oracle: integer inputs bit-exact (host- and device-planned, bf16 and
fp32 Y, with swap-AB tails and whole tiles in the same launch, a plan of GEMV tasks only, three launches on
one plan: the unit queue resets), FP8 codes bit-exact, the paper's §5 worst case at full size sampled within
the north-star tolerance, and the EP row-pointer epilogue."""
import numpy as np
import pytest
import torch

import paper_2501_16103_b200 as M
import synth
from oracle import fp8 as ofp8
from oracle import moe as omoe
from synth import fp8 as sfp8
from synth import workloads as wl

pytestmark = pytest.mark.gpu
GEMV = ((2, 4), (1, 64))


def _worst_like(T, E, k, seed):
    """P:375-shaped routing at a small size: the first k experts take most tokens, the rest get 1-4."""
    rng = np.random.default_rng(seed)
    ids = np.zeros((T, k), dtype=np.int32)
    light = list(range(k, E))
    n_light = [int(rng.integers(1, 5)) if 8 * len(light) <= T else 1 for _ in light]
    assert sum(n_light) <= T
    t = 0
    for e, n in zip(light, n_light):
        for _ in range(n):
            row = [e] + [j for j in range(k) if j != e][: k - 1]
            ids[t] = row
            t += 1
    for tt in range(t, T):
        ids[tt] = rng.permutation(k)
    return ids


def _run(ids, Xd, Wd, E, device_plan, out_dtype=torch.float32, catalog=GEMV, flags=0, reps=1):
    topk = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)).cuda()
    H, N = Xd.shape[1], Wd.shape[2]
    if device_plan:
        plan = M.Plan(None, H, N, 256, 512, flags, E=E, catalog=catalog)
        counts, row_off, tok, _, _ = M.moe_route(topk, E, plan=plan)
    else:
        counts, row_off, tok, _, _ = M.moe_route(topk, E)
        plan = M.Plan(counts.cpu().numpy(), H, N, 256, 512, flags, catalog=catalog)
    outs = []
    for _ in range(reps):
        Y = torch.full((tok.numel(), N), float("nan"), dtype=out_dtype, device="cuda")
        M.moe_gemm(plan, Xd, tok, Wd, Y=Y)
        outs.append(Y)
    torch.cuda.synchronize()
    return outs, plan, counts.cpu().numpy()


@pytest.mark.parametrize("device_plan", [False, True])
@pytest.mark.parametrize("shape", [(600, 24, 2, 256, 16384), (1200, 40, 3, 512, 8192), (400, 64, 8, 128, 5120)])
def test_gemv_integer_bit_exact(shape, device_plan):
    T, E, k, H, N = shape
    ids = _worst_like(T, E, k, T)
    X, W = synth.make_x(T, T, H, "int"), synth.make_w(T, E, H, N, "int")
    Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    outs, plan, counts = _run(ids, Xd, Wd, E, device_plan, reps=3)
    assert ((counts > 0) & (counts <= 4)).sum() >= E - k - 1              # GEMV tasks present
    rc, rr, rt, _ = omoe.buckets(ids, E)
    ref = omoe.expert_gemm(X, W, rt, rr)
    for Y in outs:                                                      # the unit queue resets per launch
        assert np.array_equal(Y.cpu().double().numpy(), ref)
    (Yb,), _, _ = _run(ids, Xd, Wd, E, device_plan, out_dtype=torch.bfloat16)
    assert torch.equal(Yb, torch.from_numpy(ref).float().to(torch.bfloat16).cuda())


def test_gemv_below_min_tiles_falls_through():
    """Every expert has 1-4 rows: no tiles would cover the GEMV streams (< MOE_GEMV_MIN_TILES), so the
    GEMV rule does not apply and the tasks run as tiles; exact either way."""
    T, E, k, H, N = 20, 16, 1, 256, 768
    ids = (np.arange(T, dtype=np.int32) % E)[:, None]
    X, W = synth.make_x(3, T, H, "int"), synth.make_w(3, E, H, N, "int")
    Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    (Y,), plan, counts = _run(ids, Xd, Wd, E, False)
    assert plan.total_tiles > 0 and counts.max() <= 4
    rc, rr, rt, _ = omoe.buckets(ids, E)
    assert np.array_equal(Y.cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr))


def test_gemv_fp8_codes_bit_exact():
    T, E, k, H, N = 600, 32, 2, 256, 16384
    ids = _worst_like(T, E, k, 9)
    X8, W8 = sfp8.make_x_fp8(9, T, H, "int"), sfp8.make_w_fp8(9, E, H, N, "int")
    sc = np.array([2.0 ** (e % 3 - 1) for e in range(E)], dtype=np.float32)
    topk = torch.from_numpy(ids).cuda()
    counts, row_off, tok, _, _ = M.moe_route(topk, E)
    plan = M.Plan(counts.cpu().numpy(), H, N, 256, 512, catalog=GEMV)
    Y = M.moe_gemm_fp8(plan, torch.from_numpy(X8).cuda(), tok, torch.from_numpy(W8).cuda(), torch.from_numpy(sc).cuda(),
                       out_dtype=torch.float32)
    torch.cuda.synchronize()
    rc, rr, rt, _ = omoe.buckets(ids, E)
    assert np.array_equal(Y.cpu().double().numpy(), ofp8.expert_gemm_fp8(X8, W8, rt, rr, sc))


def test_gemv_generic_tolerance_paper_worst_full_size():
    """The paper's §5 worst case at full size, full-mantissa inputs, device plan with the GEMV
    rule: the 56 one-token experts through the GEMV strategy, sampled rows / columns against the oracle."""
    c = synth.CONFIGS["paper_worst"]
    ids = synth.route(c, 0)
    Xd = synth.make_x_torch(0, c.T, c.H, "generic", device="cuda")
    Wd = synth.make_w_torch(0, c.E, c.H, c.N, "generic", device="cuda")
    (Y,), plan, counts = _run(ids, Xd, Wd, c.E, True)
    rc, rr, rt, _ = omoe.buckets(ids, c.E)
    rng = np.random.default_rng(1)
    light = [e for e in range(c.E) if 0 < rc[e] <= 4]
    heavy = [e for e in range(c.E) if rc[e] > 4]
    assert len(light) == c.E - c.k
    rows = [int(rr[e]) for e in light[:6]] + [int(rr[e]) + int(rng.integers(0, rc[e])) for e in heavy]
    cols = np.unique(np.concatenate([[0, 127, 128, c.N - 1], rng.integers(0, c.N, 20)]))
    got = Y[torch.tensor(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().double().numpy()
    ref = np.zeros_like(got)
    for i, r in enumerate(rows):
        e = int(np.searchsorted(rr, r, side="right") - 1)
        ref[i] = wl.x_rows(0, c.T, c.H, [int(rt[r])], "generic")[0] @ wl.w_columns(0, c.E, c.H, c.N, e, cols, "generic")
    d = np.abs(got - ref)
    assert (d <= 1e-2 * (np.abs(ref) + 1)).all(), d.max()
    assert np.linalg.norm(got - ref) <= 2e-3 * np.linalg.norm(ref)


def test_gemv_through_ep_peer_rowptr():
    """The EP step's row-pointer epilogue (results stored at the token owners) carries GEMV rows too:
    G = 2 virtual ranks, wide pair tiles, rank 0's plan has one-token experts next to two busy ones."""
    G, E, k, T_l, H, N = 2, 8, 2, 512, 128, 16384
    T = G * T_l
    ids = _worst_like(T, E, k, 5)
    X, W = synth.make_x(5, T, H, "int"), synth.make_w(5, E, H, N, "int")
    El = E // G
    Ws = [torch.from_numpy(W[r * El:(r + 1) * El]).to(torch.bfloat16).cuda() for r in range(G)]
    Xs = [torch.from_numpy(X[r * T_l:(r + 1) * T_l]).to(torch.bfloat16).cuda() for r in range(G)]
    tks = [torch.from_numpy(np.ascontiguousarray(ids[r * T_l:(r + 1) * T_l])).cuda() for r in range(G)]
    eps = M.PeerExpertParallel.group(G, E, Ws, max_tokens=T_l, k=k, bm=256, bn=512)
    for ep in eps:
        ep.set_timeout(20.0)
    outs = [torch.full((T_l * k, N), float("nan"), device="cuda") for _ in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    torch.cuda.synchronize()
    for r in range(G):
        with torch.cuda.stream(streams[r]):
            eps[r].forward(tks[r], Xs[r], out=outs[r])
    torch.cuda.synchronize()
    assert [ep.status() for ep in eps] == [0] * G
    got = torch.cat([o.cpu() for o in outs]).double().numpy()
    assert np.array_equal(got, omoe.per_slot_outputs(ids, X, W))
