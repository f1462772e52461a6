"""MOE_KIND_RIDE: an expert's short tail rides on the two 256-column halves of its last full
row tile — one more swap-AB MMA on the same staged W.  Compared with the fp64 oracle (oracle/moe.py):
bit-exact on integer data (fp32 sums exact), the north-star tolerance on full-mantissa
data at the Mixtral shape; the same plan on kernels without the strategy (FP8, contiguous-row A) runs the ride
slots as plain wide tiles."""
import numpy as np
import pytest
import torch

import paper_2501_16103_b200 as M
import synth
from oracle import moe as omoe

pytestmark = pytest.mark.gpu

RIDE = ((M.MOE_KIND_GEMV, 4), (M.MOE_KIND_RIDE, 32))


def _ids_from_counts(counts, k, rng):
    """top-k ids whose per-expert counts are exactly `counts` (sum divisible by k; each token's k experts
    distinct when possible)."""
    slots = np.repeat(np.arange(len(counts), dtype=np.int32), counts)
    rng.shuffle(slots)
    T = len(slots) // k
    return np.ascontiguousarray(slots[:T * k].reshape(T, k))


def _counts(rng, E):
    out = []
    for _ in range(E):
        u = rng.random()
        if u < 0.15:
            out.append(0)
        elif u < 0.7:
            out.append(256 * int(rng.integers(1, 5)) + int(rng.integers(1, 33)))   # ride tails 1..32
        else:
            out.append(int(rng.integers(1, 1100)))
    return out


@pytest.mark.parametrize("case", range(24))
def test_ride_fuzz_integer_bit_exact(case):
    rng = np.random.default_rng(5000 + case)
    E = int(rng.integers(1, 9))
    counts = _counts(rng, E)
    if sum(counts) == 0:
        counts[0] = 300
    ids = _ids_from_counts(counts, 1, rng)
    T = ids.shape[0]
    rc, rr, rt, _ = omoe.buckets(ids, E)
    H = int(rng.choice([64, 128, 256, 512]))
    N = int(rng.choice([512, 1024, 1536]))
    catalog = [RIDE, ((M.MOE_KIND_RIDE, 32),), ((M.MOE_KIND_RIDE, 16),)][case % 3]
    flags = int(rng.choice([0, M.MOE_SCHED_DYNAMIC, M.MOE_GRID_STATIC]))
    out = torch.float32 if case % 2 else torch.bfloat16
    X, W = synth.make_x(case, T, H, "int"), synth.make_w(case, E, H, N, "int")
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    Wd = torch.from_numpy(W).to(torch.bfloat16).cuda()
    topk = torch.from_numpy(ids).cuda()
    ref = omoe.expert_gemm(X, W, rt, rr)
    ref_t = torch.from_numpy(ref).to(out).double().numpy()
    device_plan = case % 4 == 0
    if device_plan:
        plan = M.Plan(None, H, N, 256, 512, flags, E=E, catalog=catalog)
    else:
        plan = M.Plan(rc, H, N, 256, 512, flags, catalog=catalog)
        kinds = M.parse_plan_blob(plan.blob())["params"][:, 3]
        assert kinds.tolist() == [omoe.tail_kind(m, 256, catalog, 512, N) for m in rc]
        assert (kinds == M.MOE_KIND_RIDE).any() == any(m > 256 and 0 < m % 256 <= catalog[-1][1] for m in rc)
    for rep in range(2):
        _, _, tok, _, _ = M.moe_route(topk, E, plan=plan if device_plan else None)
        Y = torch.full((T, N), float("nan"), dtype=out, device="cuda")
        M.moe_gemm(plan, Xd, tok, Wd, Y=Y)
        torch.cuda.synchronize()
        assert np.array_equal(Y.cpu().double().numpy(), ref_t), (rep, counts, catalog, flags, H, N)


@pytest.mark.parametrize("tail", [1, 5, 16, 17, 31, 32])
def test_ride_every_tail_height(tail):
    """Tails of 1-32 rows (swap N = 16 or 32) on experts of 1-3 full row tiles, row map output."""
    rng = np.random.default_rng(tail)
    counts = [256 + tail, 512 + tail, 768 + tail, 256]
    ids = _ids_from_counts(counts, 1, rng)
    T, E, H, N = ids.shape[0], len(counts), 192, 1024
    rc, rr, rt, _ = omoe.buckets(ids, E)
    X, W = synth.make_x(tail, T, H, "int"), synth.make_w(tail, E, H, N, "int")
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    Wd = torch.from_numpy(W).to(torch.bfloat16).cuda()
    _, _, tok, _, _ = M.moe_route(torch.from_numpy(ids).cuda(), E)
    plan = M.Plan(rc, H, N, 256, 512, 0, catalog=((M.MOE_KIND_RIDE, 32),))
    assert M.parse_plan_blob(plan.blob())["params"][:, 3].tolist() == [3, 3, 3, 0]
    ref = omoe.expert_gemm(X, W, rt, rr)
    perm = torch.from_numpy(rng.permutation(T).astype(np.int32)).cuda()     # Y row of CSR row i
    Y = torch.full((T, N), float("nan"), dtype=torch.float32, device="cuda")
    M.moe_gemm(plan, Xd, tok, Wd, Y=Y, row_map=perm)
    torch.cuda.synchronize()
    got = Y.cpu().double().numpy()[perm.cpu().numpy()]
    assert np.array_equal(got, ref)


def test_ride_plan_on_kernels_without_the_strategy():
    """FP8 and contiguous-row A (token_idx NULL) run a ride plan's slots as the plain wide tiles: same Y."""
    from synth import fp8 as sfp8
    from oracle import fp8 as ofp8
    rng = np.random.default_rng(3)
    counts = [261, 520, 300, 777, 0, 259]
    ids = _ids_from_counts(counts, 1, rng)
    T, E, H, N = ids.shape[0], len(counts), 256, 1024
    rc, rr, rt, _ = omoe.buckets(ids, E)
    plan = M.Plan(rc, H, N, 256, 512, 0, catalog=RIDE)
    assert (M.parse_plan_blob(plan.blob())["params"][:, 3] == M.MOE_KIND_RIDE).sum() == 4     # 261, 520, 777, 259
    _, _, tok, _, _ = M.moe_route(torch.from_numpy(ids).cuda(), E)
    # contiguous rows: X already in CSR order
    X = synth.make_x(9, T, H, "int")
    W = synth.make_w(9, E, H, N, "int")
    Xc = torch.from_numpy(X[rt]).to(torch.bfloat16).cuda()
    Y = M.moe_gemm(plan, Xc, None, torch.from_numpy(W).to(torch.bfloat16).cuda(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr))
    # FP8 E4M3 operands
    Xq = sfp8.make_x_fp8(1, T, H)
    Wq = sfp8.make_w_fp8(1, E, H, N)
    Y8 = M.moe_gemm_fp8(plan, torch.from_numpy(Xq).cuda(), tok, torch.from_numpy(Wq).cuda(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref8 = ofp8.expert_gemm_fp8(Xq, Wq, rt, rr)
    assert np.array_equal(Y8.cpu().double().numpy(), ref8)


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_ride_full_size_mixtral_generic(out_dtype):
    """The bench shape (Mixtral 8x7B, uniform routing seed 0: tails 5 / 23 / 8 / 5 ride) on full-mantissa data:
    every tail row and a sample of body rows against the fp64 oracle, north-star tolerance."""
    c = synth.CONFIGS["mix"]
    ids = synth.route(c, 0)
    rc, rr, rt, _ = omoe.buckets(ids, c.E)
    Xd = synth.make_x_torch(0, c.T, c.H, device="cuda", mode="generic")
    Wd = synth.make_w_torch(0, c.E, c.H, c.N, device="cuda", mode="generic")
    plan = M.Plan(rc, c.H, c.N, 256, 512, 0, catalog=RIDE)
    kinds = M.parse_plan_blob(plan.blob())["params"][:, 3]
    assert (kinds == M.MOE_KIND_RIDE).sum() >= 3
    _, _, tok, _, _ = M.moe_route(torch.from_numpy(ids).cuda(), c.E)
    Y = M.moe_gemm(plan, Xd, tok, Wd, out_dtype=out_dtype)
    torch.cuda.synchronize()
    rows = []
    for e in range(c.E):
        m = int(rc[e])
        if kinds[e] == M.MOE_KIND_RIDE:
            R = m // 256
            rows += list(range(rr[e] + (R - 1) * 256 - 3, rr[e] + m))        # the body row tile's end + the tail
        rows += [int(rr[e]), int(rr[e]) + m // 2]
    rows = np.array(sorted(set(rows)))
    cols = np.arange(0, c.N, 7)
    colt = torch.from_numpy(cols).cuda()
    X = Xd.float().cpu().double().numpy()
    expert_of = np.searchsorted(rr, rows, side="right") - 1
    ref = np.zeros((len(rows), len(cols)))
    for e in np.unique(expert_of):
        We = Wd[int(e)][:, colt].float().cpu().double().numpy()
        sel = expert_of == e
        ref[sel] = X[rt[rows[sel]]] @ We
    got = Y[torch.from_numpy(rows).cuda()][:, colt].cpu().double().numpy()
    d = np.abs(got - ref)
    assert (d <= 1e-2 * (np.abs(ref) + 1)).all(), d.max()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 2e-3


@pytest.mark.parametrize("flags", [0, M.MOE_A_GATHER4])
def test_ride_with_gemv_tasks_fp32_and_row_map(flags):
    """A plan holding GEMV tasks (one-row experts), ride tasks and plain tasks in one launch; gather4 A makes
    the ride slots run as wide tiles (ride needs the cp.async rows): the same exact Y either way."""
    rng = np.random.default_rng(77)
    counts = [1, 2, 300, 1, 513, 777, 256, 4, 280, 3] + [600] * 8         # >= 128 other tiles: GEMV applies
    ids = _ids_from_counts(counts, 1, rng)
    T, E, H, N = ids.shape[0], len(counts), 128, 2048
    rc, rr, rt, _ = omoe.buckets(ids, E)
    plan = M.Plan(rc, H, N, 256, 512, flags, catalog=RIDE)
    kinds = M.parse_plan_blob(plan.blob())["params"][:, 3].tolist()
    assert kinds.count(M.MOE_KIND_GEMV) == 5 and kinds.count(M.MOE_KIND_RIDE) == 3
    X, W = synth.make_x(77, T, H, "int"), synth.make_w(77, E, H, N, "int")
    _, _, tok, _, _ = M.moe_route(torch.from_numpy(ids).cuda(), E)
    perm = torch.from_numpy(rng.permutation(T).astype(np.int32)).cuda()
    Y = torch.full((T, N), float("nan"), dtype=torch.float32, device="cuda")
    M.moe_gemm(plan, torch.from_numpy(X).to(torch.bfloat16).cuda(), tok, torch.from_numpy(W).to(torch.bfloat16).cuda(),
               Y=Y, row_map=perm)
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().double().numpy()[perm.cpu().numpy()], omoe.expert_gemm(X, W, rt, rr))
