"""The paper's own §5 evaluation (Table 1) on one B200: T=4096 tokens, E=64 experts,
top-8, expert weight [3584, 2560] (H=3584, N=2560 — the FLOP count is the same either way),
balanced / best / worst routing, under the §4.2 expert orderings.  Reports moe_gemm kernel
TFLOP/s (useful flops, L2 flushed before each launch) and % of the measured B200 peak, beside
the paper's H20 / H800 percentages (context, other hardware).

    python scripts/paper_table1.py [--out profiles/r01/paper_table1.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_16103_b200 as M  # noqa: E402
import synth  # noqa: E402

PAPER = {"balanced": {"H20": 94.67, "H800": 84.82}, "best": {"H20": 94.89, "H800": 90.70},
         "worst": {"H20": 90.11, "H800": 59.37}}
ORDER = {"natural": 0, "alternating": M.MOE_ORDER_ALTERNATING, "half_interval": M.MOE_ORDER_HALF_INTERVAL}



class CleanFlush:
    """256 MiB memset then a 256 MiB read: L2 is cold for the timed op and holds no dirty lines
    whose write-back would be charged to it (as bench.py)."""

    def __init__(self):
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(32 << 20, dtype=torch.int64, device="cuda")

    def __call__(self):
        self.w.zero_()
        self.r.sum()

def time_gemm(plan, X, tok, W, Y, flush, reps=20):
    for _ in range(3):
        M.moe_gemm(plan, X, tok, W, Y=Y)
    ms = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(4_000_000)               # the host enqueues the timed launches first (device time only)
        a.record()
        M.moe_gemm(plan, X, tok, W, Y=Y)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    peak = float(peaks["bf16_tflops"])
    flush = CleanFlush()
    c0 = synth.CONFIGS["paper_balanced"]
    X = synth.make_x_torch(0, c0.T, c0.H, device="cuda")
    W = synth.make_w_torch(0, c0.E, c0.H, c0.N, device="cuda")
    rows = []
    for case in ("balanced", "best", "worst"):
        c = synth.CONFIGS[f"paper_{case}"]
        ids = torch.from_numpy(synth.route(c)).cuda()
        counts, row_off, tok, _, _ = M.moe_route(ids, c.E)
        counts_h = counts.cpu().numpy()
        Y = torch.empty((tok.numel(), c.N), dtype=torch.bfloat16, device="cuda")
        for bm, bn in ((128, 256), (256, 256), (256, 512)):
            for order, fl in ORDER.items():
                plan = M.Plan(counts_h, c.H, c.N, bm, bn, fl)
                ms = time_gemm(plan, X, tok, W, Y, flush)
                tf = c.flops / (ms * 1e-3) / 1e12
                rows.append({"case": case, "tile": f"{bm}x{bn}", "order": order, "ms": ms, "tflops": tf,
                             "pct_of_measured_peak": 100 * tf / peak, "paper_pct": PAPER[case]})
                print(json.dumps(rows[-1]), flush=True)
    if args.out:
        json.dump({"peak_tflops": peak, "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
