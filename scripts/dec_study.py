#!/usr/bin/env python
"""Decode-regime timing study (run on the GPU box): where does the T = 1 kernel's time go?

1. moe_gemm with the dec1 routing (2 experts x 1 row, N = 14336) at H = 64 .. 4096: the
   intercept of time vs bytes is the fixed cost (launch, prologue, first refill, drain), the
   slope the streaming rate.
2. torch copy / sum over the same byte counts: what a plain HBM stream reaches at that size.
Every launch follows an L2 flush (256 MiB memset); median of 30, CUDA events.
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_16103_b200 as M  # noqa: E402


def timeit(fn, flush, reps=30):
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    E, N = 8, 14336
    out = {"gemm": [], "copy": [], "sum": []}
    bm, bn = int(os.environ.get("BM", "128")), int(os.environ.get("BN", "256"))
    for T, counts in ((1, [0, 0, 0, 0, 1, 0, 0, 1]), (16, [4, 7, 2, 5, 7, 3, 0, 4])):
        rows = sum(counts)
        for H in (64, 256, 1024, 2048, 4096, 8192):
            X = torch.randn(T, H, device="cuda").to(torch.bfloat16)
            W = torch.randn(E, H, N, device="cuda").to(torch.bfloat16)
            tok = torch.tensor([t % T for t in range(rows)], dtype=torch.int32, device="cuda")
            plan = M.Plan(np.array(counts, np.int32), H, N, bm=bm, bn=bn)
            Y = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
            us = timeit(lambda: M.moe_gemm(plan, X, tok, W, Y=Y), flush)
            active = sum(1 for c in counts if c)
            byts = active * H * N * 2
            out["gemm"].append({"T": T, "H": H, "us": us, "w_bytes": byts, "gbs": byts / us / 1e3,
                                "tile": f"{plan.bm}x{plan.bn}"})
            print(json.dumps(out["gemm"][-1]), flush=True)
            del W
    for mb in (16, 64, 117, 235, 470, 940):
        n = mb * (1 << 20) // 2
        a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        b = torch.empty_like(a)
        us = timeit(lambda: b.copy_(a), flush)
        out["copy"].append({"MiB": mb, "us": us, "gbs": 2 * n * 2 / us / 1e3})
        us = timeit(lambda: a.sum(), flush)
        out["sum"].append({"MiB": mb, "us": us, "gbs": n * 2 / us / 1e3})
        print(json.dumps(out["copy"][-1]), json.dumps(out["sum"][-1]), flush=True)
    tiny = torch.zeros(1, device="cuda")
    out["empty_us"] = timeit(lambda: tiny.add_(1), flush)
    print(json.dumps({"empty_us": out["empty_us"]}))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/dec_study.json", "w"), indent=1)


if __name__ == "__main__":
    main()
