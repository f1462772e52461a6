#!/usr/bin/env python
"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
route (small + multi-kernel), device plan, bf16 GEMM (1-CTA, pair, wide, split tail, decode tile,
CSR rows), FP8 GEMM (1-CTA, wide), the FFN layer's gated GEMM + combine, GEMV tasks, split-K decode tiles,
the light-last merge, the loopback and peer-memory EP steps, checked against the oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_16103_b200 as M  # noqa: E402
import synth  # noqa: E402
from oracle import fp8 as ofp8  # noqa: E402
from oracle import moe as omoe  # noqa: E402
from synth import fp8 as sfp8  # noqa: E402


def main():
    T, E, k, H, N = 300, 5, 2, 192, 640
    ids = synth.route_gumbel(1, T, E, k, s=1.0, n_empty=1)
    X, W = synth.make_x(1, T, H, "int"), synth.make_w(1, E, H, N, "int")
    Xd, Wd = torch.from_numpy(X).to(torch.bfloat16).cuda(), torch.from_numpy(W).to(torch.bfloat16).cuda()
    rc, rr, rt, rs = omoe.buckets(ids, E)
    ref = omoe.expert_gemm(X, W, rt, rr)
    topk = torch.from_numpy(ids).cuda()
    n = 0
    for bm, bn, fl in ((128, 256, 0), (256, 256, 0), (256, 512, 0), (256, 256, M.MOE_SPLIT_TAIL), (64, 256, 0)):
        plan = M.Plan(None, H, N, bm, bn, fl, E=E)
        Y, *_ = M.moe_forward(topk, Xd, Wd, E, plan=plan, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert np.array_equal(Y.cpu().double().numpy(), ref), (bm, bn, fl)
        n += 1
    counts, row_off, tok, slot, _ = M.moe_route(topk, E)
    plan = M.Plan(counts.cpu().numpy(), H, N, 256, 512)
    Yc = M.moe_gemm(plan, Xd.index_select(0, tok.long()).contiguous(), None, Wd, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert np.array_equal(Yc.cpu().double().numpy(), ref)
    c2, r2, t2, s2, _ = M.moe_route(topk, E, route_flags=M.MOE_ROUTE_NO_SMALL)
    assert torch.equal(t2, tok)
    X8, W8 = sfp8.make_x_fp8(1, T, H, "int"), sfp8.make_w_fp8(1, E, H, N, "int")
    ref8 = ofp8.expert_gemm_fp8(X8, W8, rt, rr)
    for bm, bn in ((128, 256), (256, 512)):
        Y8, *_ = M.moe_forward(topk, torch.from_numpy(X8).cuda(), torch.from_numpy(W8).cuda(), E, bm=bm, bn=bn,
                               out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert np.array_equal(Y8.cpu().double().numpy(), ref8), (bm, bn)
        n += 1
    Wg, Wu, Wdn = (torch.from_numpy(synth.make_w(s, E, H, 256, "int")).to(torch.bfloat16).cuda() for s in (2, 3, 4))
    layer = M.MoeFFN(Wg, Wu, torch.from_numpy(synth.make_w(5, E, 256, H, "int")).to(torch.bfloat16).cuda())
    w = torch.rand((T, k), device="cuda")
    layer.forward(Xd, topk, w)
    torch.cuda.synchronize()
    # decode tiles with the balanced grid (more tiles than SMs), and the library's EP step over the
    # loopback transport (2 virtual ranks, one thread each), combine fused into the epilogue
    Td, Hd, Nd = 16, 256, 14336
    idd = synth.route_gumbel(2, Td, 8, 2)
    Xq, Wq = synth.make_x(2, Td, Hd, "int"), synth.make_w(2, 8, Hd, Nd, "int")
    Yd, *_ = M.moe_forward(torch.from_numpy(idd).cuda(), torch.from_numpy(Xq).to(torch.bfloat16).cuda(),
                           torch.from_numpy(Wq).to(torch.bfloat16).cuda(), 8, bm=128, bn=256, out_dtype=torch.float32)
    torch.cuda.synchronize()
    c3, r3, t3, s3 = omoe.buckets(idd, 8)
    assert np.array_equal(Yd.cpu().double().numpy(), omoe.expert_gemm(Xq, Wq, t3, r3))
    import threading
    G, Tl = 2, 64
    ide = synth.route_gumbel(3, G * Tl, 8, 2)
    Xe, We = synth.make_x(3, G * Tl, 64, "int"), synth.make_w(3, 8, 64, 256, "int")
    eps = M.NativeExpertParallel.loopback_group(
        G, 8, [torch.from_numpy(We[4 * r:4 * r + 4]).to(torch.bfloat16).cuda() for r in range(G)], fused=True)
    outs = [None] * G

    def body(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            outs[r] = eps[r].forward(torch.from_numpy(np.ascontiguousarray(ide[r * Tl:(r + 1) * Tl])).cuda(),
                                     torch.from_numpy(Xe[r * Tl:(r + 1) * Tl]).to(torch.bfloat16).cuda(),
                                     out_dtype=torch.float32)
        s.synchronize()

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert np.array_equal(torch.cat([o.cpu() for o in outs]).double().numpy(), omoe.per_slot_outputs(ide, Xe, We))
    # round 2: GEMV tasks in a wide plan (>= 128 other tiles), split-K one-CTA tiles, light-last order
    # with the dynamic merge, the peer-memory EP step (2 virtual ranks, one thread)
    Tg, Eg, Hg, Ng = 300, 12, 128, 16384
    idg = np.zeros((Tg, 2), dtype=np.int32)
    for i, e in enumerate(range(2, Eg)):
        idg[i] = [e, 0]
    for t in range(Eg - 2, Tg):
        idg[t] = [0, 1] if t % 2 else [1, 0]
    Xg, Wg2 = synth.make_x(6, Tg, Hg, "int"), synth.make_w(6, Eg, Hg, Ng, "int")
    cg, rg, tg_, _ = omoe.buckets(idg, Eg)
    for fl in (0, M.MOE_ORDER_LIGHT_LAST):
        Yg, *_ = M.moe_forward(torch.from_numpy(idg).cuda(), torch.from_numpy(Xg).to(torch.bfloat16).cuda(),
                               torch.from_numpy(Wg2).to(torch.bfloat16).cuda(), Eg,
                               plan=M.Plan(None, Hg, Ng, 256, 512, fl, E=Eg), out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert np.array_equal(Yg.cpu().double().numpy(), omoe.expert_gemm(Xg, Wg2, tg_, rg)), fl
    Ys, *_ = M.moe_forward(torch.from_numpy(idd).cuda(), torch.from_numpy(Xq).to(torch.bfloat16).cuda(),
                           torch.from_numpy(Wq).to(torch.bfloat16).cuda(), 8,
                           plan=M.Plan(None, Hd, Nd, 128, 256, M.MOE_SPLIT_K, E=8), out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert np.array_equal(Ys.cpu().double().numpy(), omoe.expert_gemm(Xq, Wq, t3, r3))
    peers = M.PeerExpertParallel.group(G, 8, [torch.from_numpy(We[4 * r:4 * r + 4]).to(torch.bfloat16).cuda()
                                              for r in range(G)], max_tokens=Tl, k=2)
    pouts = [torch.empty((Tl * 2, 256), device="cuda") for _ in range(G)]
    pst = [torch.cuda.Stream() for _ in range(G)]
    torch.cuda.synchronize()
    for r in range(G):
        with torch.cuda.stream(pst[r]):
            peers[r].forward(torch.from_numpy(np.ascontiguousarray(ide[r * Tl:(r + 1) * Tl])).cuda(),
                             torch.from_numpy(Xe[r * Tl:(r + 1) * Tl]).to(torch.bfloat16).cuda(), out=pouts[r])
    torch.cuda.synchronize()
    assert [p_.status() for p_ in peers] == [0] * G
    assert np.array_equal(torch.cat([o.cpu() for o in pouts]).double().numpy(), omoe.per_slot_outputs(ide, Xe, We))
    # round 2, late: ride tiles (tails on the last full row tile) and the pair gather4 A path
    rng = np.random.default_rng(8)
    cr = [261, 520, 300, 280, 0, 259]
    idr = np.repeat(np.arange(len(cr), dtype=np.int32), cr)[:, None]
    rng.shuffle(idr)
    Xr, Wr = synth.make_x(8, idr.shape[0], 128, "int"), synth.make_w(8, len(cr), 128, 1024, "int")
    crr, rrr, trr, _ = omoe.buckets(idr, len(cr))
    for cat, fl in ((((M.MOE_KIND_RIDE, 32),), 0), (None, M.MOE_A_GATHER4)):
        Yr, *_ = M.moe_forward(torch.from_numpy(idr).cuda(), torch.from_numpy(Xr).to(torch.bfloat16).cuda(),
                               torch.from_numpy(Wr).to(torch.bfloat16).cuda(), len(cr),
                               plan=M.Plan(None, 128, 1024, 256, 512, fl, E=len(cr), catalog=cat), out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert np.array_equal(Yr.cpu().double().numpy(), omoe.expert_gemm(Xr, Wr, trr, rrr)), (cat, fl)
    print(f"sanitize workload ok: {n} GEMM variants + ride tiles + pair gather4 + CSR rows + both route paths + FFN layer + balanced decode "
          f"grid + EP step (loopback, fused combine) + GEMV tasks (natural, light-last) + split-K decode tiles + "
          f"peer-memory EP step")


if __name__ == "__main__":
    main()
