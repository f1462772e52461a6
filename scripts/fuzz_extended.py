"""Extended randomized parity sweep (GPU): random routings, shapes, tile shapes, catalogs (GEMV / SWAP / RIDE), plan
flags (dynamic / static order, expert orderings, gather4 A, register epilogue), host / device plans, bf16 / fp32
output, bf16 and FP8 operands — every case on integer data against the fp64 oracle, bit for bit.

    python scripts/fuzz_extended.py [n_cases] [seed] [int|generic]   (one JSON line per failure, then a summary)

generic: full-mantissa bf16 / full-range E4M3 operands (synth "generic" mode) whose fp32 sums round, checked
against the north-star tolerance (max |d| <= 1e-2 (|ref| + 1), relative Frobenius <= 2e-3); the summary carries
the worst max-|d| / bound ratio and relative Frobenius error seen.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2501_16103_b200 as M  # noqa: E402
import synth  # noqa: E402
from oracle import fp8 as ofp8  # noqa: E402
from oracle import moe as omoe  # noqa: E402
from synth import fp8 as sfp8  # noqa: E402


MODE = "int"
WORST = {"max_ratio": 0.0, "rel_fro": 0.0}


def one_case(rng, i):
    E = int(rng.integers(1, 33))
    k = int(rng.integers(1, min(E, 6) + 1))
    T = int(rng.integers(1, 2500))
    H = int(rng.choice([64, 128, 192, 320, 512, 1024]))
    fp8 = bool(rng.random() < 0.2)
    shape = [(128, 128), (128, 256), (256, 256), (256, 512), (0, 0)][int(rng.integers(0, 5))]
    bm, bn = shape
    N = int(rng.choice([128, 256, 512, 640, 1024, 1408, 2048])) if not fp8 else int(rng.choice([256, 512, 1024, 2048]))
    if fp8 and bm == 256 and bn == 256:
        bn = 512
    flags = 0
    if rng.random() < 0.3:
        flags |= int(rng.choice([M.MOE_SCHED_DYNAMIC, M.MOE_GRID_STATIC, M.MOE_GRID_BALANCED]))
    if rng.random() < 0.3:
        flags |= int(rng.choice([M.MOE_ORDER_ALTERNATING, M.MOE_ORDER_HALF_INTERVAL, M.MOE_ORDER_LIGHT_LAST]))
    if rng.random() < 0.2:
        flags |= M.MOE_A_GATHER4
    if rng.random() < 0.15:
        flags |= M.MOE_EPI_REGISTER
    if (flags & M.MOE_GRID_STATIC) and (flags & M.MOE_GRID_BALANCED):
        flags &= ~M.MOE_GRID_BALANCED
    catalog = None
    wide = bm == 256 and bn == 512
    if wide and not fp8 and rng.random() < 0.5:
        opts = [(M.MOE_KIND_GEMV, 4), (M.MOE_KIND_SWAP, int(rng.integers(1, 257))), (M.MOE_KIND_RIDE, int(rng.integers(1, 33)))]
        catalog = tuple(opts[j] for j in rng.choice(3, size=int(rng.integers(0, 3)), replace=False))
    skew = float(rng.choice([0.0, 1.2]))
    n_empty = int(rng.integers(0, max(1, E - k + 1)))
    ids = synth.route_gumbel(i, T, E, k, s=skew, n_empty=min(n_empty, E - k))
    rc, rr, rt, _ = omoe.buckets(ids, E)
    out = torch.float32 if rng.random() < 0.5 else torch.bfloat16
    if fp8:
        m8 = "full" if MODE == "generic" else MODE
        X, W = sfp8.make_x_fp8(i, T, H, m8), sfp8.make_w_fp8(i, E, H, N, m8)
        # full-range codes carry the per-expert scale that puts Y at O(1), as the tests do (synth.fp8.w_scale):
        # the tolerance's "+ 1" presumes values of that size
        sc = sfp8.w_scale(E, H, m8)
        ref = ofp8.expert_gemm_fp8(X, W, rt, rr, sc)
        Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
        scd = torch.from_numpy(sc).cuda()
    else:
        X, W = synth.make_x(i, T, H, MODE), synth.make_w(i, E, H, N, MODE)
        ref = omoe.expert_gemm(X, W, rt, rr)
        Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    device_plan = bool(rng.random() < 0.4)
    topk = torch.from_numpy(ids).cuda()
    try:
        if device_plan:
            plan = M.Plan(None, H, N, bm, bn, flags, E=E, catalog=catalog)
            _, _, tok, _, _ = M.moe_route(topk, E, plan=plan)
        else:
            counts, _, tok, _, _ = M.moe_route(topk, E)
            plan = M.Plan(counts.cpu().numpy(), H, N, bm, bn, flags, catalog=catalog)
    except M.MoeError as e:                                  # a combination the planner refuses up front
        return "refused", str(e)[:120]
    Y = torch.full((int(rc.sum()), N), float("nan"), dtype=out, device="cuda")
    for _ in range(2):
        if fp8:
            M.moe_gemm_fp8(plan, Xd, tok, Wd, scale=scd, Y=Y)
        else:
            M.moe_gemm(plan, Xd, tok, Wd, Y=Y)
    torch.cuda.synchronize()
    got = Y.cpu().double().numpy()
    if MODE == "int":
        ok = np.array_equal(got, torch.from_numpy(ref).to(out).double().numpy())
    else:
        d = np.abs(got - ref)
        ratio = float((d / (1e-2 * (np.abs(ref) + 1))).max()) if d.size else 0.0
        fro = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)) if d.size else 0.0
        WORST["max_ratio"] = max(WORST["max_ratio"], ratio)
        WORST["rel_fro"] = max(WORST["rel_fro"], fro)
        ok = ratio <= 1.0 and fro <= 2e-3 and not np.isnan(got).any()
    desc = dict(case=i, E=E, k=k, T=T, H=H, N=N, bm=bm, bn=bn, flags=flags, catalog=catalog, fp8=fp8,
                out=str(out), device_plan=device_plan)
    return ("ok" if ok else "FAIL"), desc


def main():
    global MODE
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    MODE = sys.argv[3] if len(sys.argv) > 3 else "int"
    rng = np.random.default_rng(seed)
    counts = {"ok": 0, "FAIL": 0, "refused": 0}
    t0 = time.time()
    for i in range(n):
        status, desc = one_case(rng, seed * 100000 + i)
        counts[status] += 1
        if status != "ok":
            print(json.dumps({"status": status, "case": desc}), flush=True)
    print(json.dumps({"summary": counts, "cases": n, "seed": seed, "mode": MODE, "seconds": round(time.time() - t0, 1),
                      **({"worst": WORST} if MODE != "int" else {})}), flush=True)


if __name__ == "__main__":
    main()
