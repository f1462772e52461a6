"""Same-box comparators for the MoE expert GEMM (context for DESIGN.md §7; not on our path).

* ours           : moe_gemm (one launch, gathered rows, device-planned), kernel time
* cublas_loop    : the naive per-expert loop: gather X rows per expert, torch.matmul each
* grouped_mm     : the grouped-GEMM prior art: index_select gather into a
                   contiguous buffer + torch._grouped_mm (one launch, dynamic tile scheduling)
* dense_cublas   : one dense torch.matmul with the same FLOPs and N, K (a ceiling for the shape)

All timed with CUDA events, L2 flushed before every launch, median of 20.

    python scripts/comparators.py [config ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_16103_b200 as M  # noqa: E402
import synth  # noqa: E402



class CleanFlush:
    """256 MiB memset then a 256 MiB read: L2 is cold for the timed op and holds no dirty lines
    whose write-back would be charged to it (as bench.py)."""

    def __init__(self):
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(32 << 20, dtype=torch.int64, device="cuda")

    def __call__(self):
        self.w.zero_()
        self.r.sum()

def timed(fn, flush, reps=20):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(4_000_000)               # the host enqueues the timed launches first (device time only)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms))


def main():
    names = sys.argv[1:] or ["mix", "ds", "paper_balanced", "dec16"]
    flush = CleanFlush()
    for name in names:
        c = synth.CONFIGS[name]
        ids = torch.from_numpy(synth.route(c, 0)).cuda()
        X = synth.make_x_torch(0, c.T, c.H, device="cuda")
        W = synth.make_w_torch(0, c.E, c.H, c.N, device="cuda")
        counts, row_off, tok, _, _ = M.moe_route(ids, c.E)
        counts_h = counts.cpu().numpy()
        ro = row_off.cpu().numpy()
        tok_l = tok.long()
        plan = M.Plan(counts_h, c.H, c.N, 0, 0)
        Y = torch.empty((tok.numel(), c.N), dtype=torch.bfloat16, device="cuda")
        res = {"config": name, "flops": c.flops}
        res["ours_ms"] = timed(lambda: M.moe_gemm(plan, X, tok, W, Y=Y), flush)

        def loop():
            for e in range(c.E):
                a, b = int(ro[e]), int(ro[e + 1])
                if b > a:
                    torch.matmul(X.index_select(0, tok_l[a:b]), W[e], out=Y[a:b])
        res["cublas_loop_ms"] = timed(loop, flush)
        offs = torch.from_numpy(ro[1:].astype(np.int32)).cuda()
        Xg = torch.empty((tok.numel(), c.H), dtype=torch.bfloat16, device="cuda")

        def grouped():
            torch.index_select(X, 0, tok_l, out=Xg)
            return torch._grouped_mm(Xg, W, offs=offs)
        try:
            res["grouped_mm_ms"] = timed(grouped, flush)
            ref = grouped().float()
            res["grouped_mm_matches_ours"] = bool(torch.allclose(ref, Y.float(), rtol=2e-2, atol=2e-2))
        except Exception as e:  # pragma: no cover
            res["grouped_mm_error"] = repr(e)[:200]
        rows = int(tok.numel())
        A = torch.randn((rows, c.H), dtype=torch.bfloat16, device="cuda")
        B = torch.randn((c.H, c.N), dtype=torch.bfloat16, device="cuda")
        res["dense_cublas_ms"] = timed(lambda: torch.matmul(A, B), flush)
        for k in list(res):
            if k.endswith("_ms"):
                res[k.replace("_ms", "_tflops")] = c.flops / (res[k] * 1e-3) / 1e12
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
