"""GPU parity of split-K one-CTA tiles (MOE_SPLIT_K, opt-in): when whole 128 x bn tiles
would leave SMs idle and every task has <= 16 rows (decode batches), the kernel splits every tile's K blocks
into S equal parts spread over one CTA per SM; the CTA finishing a tile's last part sums the parts in K
order.

Checks: integer inputs bit-exact against the fp64 oracle and against the whole-tile path
(no MOE_SPLIT_K) — host- and device-planned, bf16 and fp32 Y, short K (units spanning several tiles
and tiles split over three CTAs), repeated launches on one plan (the arrival counters reset), FP8 codes;
full-mantissa inputs within the north-star tolerance."""
import numpy as np
import pytest
import torch

import paper_2501_16103_b200 as M
import synth
from oracle import fp8 as ofp8
from oracle import moe as omoe
from synth import fp8 as sfp8

pytestmark = pytest.mark.gpu

CASES = [  # T, E, k, H, N: tiles < SMs, <= 16 rows per expert (the 20-row case keeps whole tiles)
    (1, 8, 2, 4096, 14336),    # the dec1 shape: 112 tiles of 64 K blocks over 148 CTAs
    (3, 8, 2, 256, 1024),      # 4 K blocks per tile: a CTA's share spans several tiles
    (5, 16, 3, 512, 640),      # ragged last column tile (640 = 2.5 x 256)
    (16, 4, 2, 1024, 2048),    # 8 rows per expert
    (40, 2, 1, 2048, 512),     # ~20 rows per expert, few tiles
    (1, 64, 8, 3584, 2560),    # paper §5 shape, one token
]


def _run(ids, Xd, Wd, E, flags=M.MOE_SPLIT_K, device_plan=False, out_dtype=torch.float32, reps=1):
    topk = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)).cuda()
    if device_plan:
        plan = M.Plan(None, Xd.shape[1], Wd.shape[2], 128, 256, flags, E=E)
        counts, row_off, tok, slot, _ = M.moe_route(topk, E, plan=plan)
    else:
        counts, row_off, tok, slot, _ = M.moe_route(topk, E)
        plan = M.Plan(counts.cpu().numpy(), Xd.shape[1], Wd.shape[2], 128, 256, flags)
    outs = []
    for _ in range(reps):
        Y = torch.full((tok.numel(), Wd.shape[2]), float("nan"), dtype=out_dtype, device="cuda")
        M.moe_gemm(plan, Xd, tok, Wd, Y=Y)
        outs.append(Y)
    torch.cuda.synchronize()
    return outs, counts.cpu().numpy()


@pytest.mark.parametrize("device_plan", [False, True])
@pytest.mark.parametrize("case", CASES)
def test_streamk_integer_bit_exact(case, device_plan):
    T, E, k, H, N = case
    ids = synth.route_gumbel(T + H, T, E, k)
    X, W = synth.make_x(T, T, H, "int"), synth.make_w(T, E, H, N, "int")
    Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    outs, counts = _run(ids, Xd, Wd, E, device_plan=device_plan, reps=3)
    whole, _ = _run(ids, Xd, Wd, E, flags=0, device_plan=device_plan)
    rc, rr, rt, _ = omoe.buckets(ids, E)
    ref = omoe.expert_gemm(X, W, rt, rr)
    for Y in outs:                                     # three launches on one plan: counters reset
        assert np.array_equal(Y.cpu().double().numpy(), ref)
    assert torch.equal(outs[0], whole[0])


@pytest.mark.parametrize("case", CASES[:3])
def test_streamk_bf16_out_matches_whole_tiles(case):
    """bf16 Y: the split sum of exact integer partials rounds exactly like the whole-tile accumulator."""
    T, E, k, H, N = case
    ids = synth.route_gumbel(T, T, E, k)
    X, W = synth.make_x(T + 1, T, H, "int"), synth.make_w(T + 1, E, H, N, "int")
    Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    (Y,), _ = _run(ids, Xd, Wd, E, out_dtype=torch.bfloat16, device_plan=True)
    (Yw,), _ = _run(ids, Xd, Wd, E, flags=0, out_dtype=torch.bfloat16, device_plan=True)
    assert torch.equal(Y, Yw)


@pytest.mark.parametrize("case", [CASES[0], CASES[1], CASES[5]])
def test_streamk_generic_tolerance(case):
    """Full-mantissa inputs (fp32 accumulation rounds): north-star tolerance against the fp64 oracle."""
    T, E, k, H, N = case
    ids = synth.route_gumbel(2 * T, T, E, k)
    X, W = synth.make_x(3, T, H, "generic"), synth.make_w(3, E, H, N, "generic")
    Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    (Y,), _ = _run(ids, Xd, Wd, E, device_plan=True)
    rc, rr, rt, _ = omoe.buckets(ids, E)
    ref = omoe.expert_gemm(X, W, rt, rr)
    got = Y.cpu().double().numpy()
    d = np.abs(got - ref)
    assert (d <= 1e-2 * (np.abs(ref) + 1)).all(), d.max()
    assert np.linalg.norm(got - ref) <= 2e-3 * np.linalg.norm(ref)


@pytest.mark.parametrize("case", [(1, 8, 2, 4096, 14336), (3, 8, 2, 256, 1024)])
def test_streamk_fp8_codes_bit_exact(case):
    T, E, k, H, N = case
    ids = synth.route_gumbel(T, T, E, k)
    X8, W8 = sfp8.make_x_fp8(T, T, H, "int"), sfp8.make_w_fp8(T, E, H, N, "int")
    sc = np.array([2.0 ** (e % 3 - 1) for e in range(E)], dtype=np.float32)
    topk = torch.from_numpy(ids).cuda()
    counts, row_off, tok, _, _ = M.moe_route(topk, E)
    plan = M.Plan(counts.cpu().numpy(), H, N, 128, 256, M.MOE_SPLIT_K)
    Y = M.moe_gemm_fp8(plan, torch.from_numpy(X8).cuda(), tok, torch.from_numpy(W8).cuda(), torch.from_numpy(sc).cuda(),
                       out_dtype=torch.float32)
    torch.cuda.synchronize()
    rc, rr, rt, _ = omoe.buckets(ids, E)
    assert np.array_equal(Y.cpu().double().numpy(), ofp8.expert_gemm_fp8(X8, W8, rt, rr, sc))


def test_streamk_not_used_above_16_rows():
    """Tasks of more than 16 rows keep whole tiles (the partial slots hold 16 rows): same bits either way."""
    T, E, k, H, N = 100, 2, 1, 512, 1024
    ids = synth.route_gumbel(5, T, E, k)
    X, W = synth.make_x(5, T, H, "int"), synth.make_w(5, E, H, N, "int")
    Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    (Y,), counts = _run(ids, Xd, Wd, E)
    assert counts.max() > 16
    rc, rr, rt, _ = omoe.buckets(ids, E)
    assert np.array_equal(Y.cpu().double().numpy(), omoe.expert_gemm(X, W, rt, rr))
