"""Same-box timing of moe_gemm launch variants (tile shape, plan flags, sigma order) on named configs.

    python scripts/tile_probe.py --cases paper_worst:256:512:0:natural,paper_worst:256:512:2:half_interval
        [--reps 20] [--out gpurun_out/probe.jsonl]

A case is cfg:bm:bn:flags:order[:catalog]; flags is the integer moe_plan flag word (2 = MOE_SPLIT_TAIL,
...); catalog is "default", "none", or rules "kind.m_max+kind.m_max" (e.g. 1.64 = swap tails <= 64 rows).
Kernel time = CUDA events around one moe_gemm launch after a clean-L2 flush (bench.py's method),
median over reps.  Prints one JSON line per case with TFLOP/s and the fraction of the measured peak.
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

ORDER = {"natural": 0, "alternating": M.MOE_ORDER_ALTERNATING, "half_interval": M.MOE_ORDER_HALF_INTERVAL,
         "light_last": M.MOE_ORDER_LIGHT_LAST}


class CleanFlush:
    def __init__(self):
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(32 << 20, dtype=torch.int64, device="cuda")

    def __call__(self):
        self.w.zero_()
        self.r.sum()


def time_gemm(plan, X, tok, W, Y, flush, reps):
    for _ in range(3):
        M.moe_gemm(plan, X, tok, W, Y=Y)
    ms = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(4_000_000)
        a.record()
        M.moe_gemm(plan, X, tok, W, Y=Y)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms)), float(np.min(ms))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", required=True)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak = float(json.load(open(p))["bf16_tflops"]) if os.path.exists(p) else 1590.0
    flush = CleanFlush()
    cache = {}
    out = open(args.out, "a") if args.out else None
    for case in args.cases.split(","):
        parts = case.split(":")
        cfg, bm, bn, flags, order = parts[:5]
        seed = 0
        if "@" in cfg:                              # cfg@seed: another routing draw of the same config
            cfg, seed = cfg.split("@")[0], int(cfg.split("@")[1])
        cat = parts[5] if len(parts) > 5 else "default"
        catalog = None if cat == "default" else () if cat == "none" else tuple(
            tuple(int(x) for x in r.split(".")) for r in cat.split("+"))
        if cfg.startswith("counts"):                # counts[H<h>N<n>_]A-B-C...: one expert per count (k = 1)
            body, hh, nn = cfg[6:], 4096, 14336     # (default: Mixtral H / N)
            if body.startswith("H"):
                dims, body = body.split("_", 1)
                hh, nn = (int(x) for x in dims[1:].split("N"))
            cnt = [int(x) for x in body.split("-")]
            c = synth.Config(cfg, E=len(cnt), k=1, T=sum(cnt), H=hh, N=nn, routing="custom")
            ids_np = np.repeat(np.arange(len(cnt), dtype=np.int32), cnt)[:, None]
        elif cfg.startswith("rows"):                  # rowsR_E: E experts of R rows each, Mixtral H / N (tile-kind cost)
            r_, e_ = (int(x) for x in cfg[4:].split("_"))
            c = synth.Config(cfg, E=e_, k=1, T=r_ * e_, H=4096, N=14336, routing="custom")
            ids_np = (np.arange(r_ * e_, dtype=np.int32) // r_)[:, None]
        elif cfg.startswith("light"):               # lightN: N experts of the paper §5 shape, one token each
            n = int(cfg[5:])
            c = synth.Config(cfg, E=64, k=1, T=n, H=3584, N=2560, routing="custom")
            ids_np = np.arange(n, dtype=np.int32)[:, None]
        else:
            c = synth.CONFIGS[cfg]
            ids_np = None
        if (cfg, seed) not in cache:
            cache.clear()
            ids = torch.from_numpy(synth.route(c, seed) if ids_np is None else ids_np).cuda()
            counts, row_off, tok, _, _ = M.moe_route(ids, c.E)
            X = synth.make_x_torch(0, c.T, c.H, device="cuda")
            W = synth.make_w_torch(0, c.E, c.H, c.N, device="cuda")
            Y = torch.empty((tok.numel(), c.N), dtype=torch.bfloat16, device="cuda")
            cache[(cfg, seed)] = (counts.cpu().numpy(), tok, X, W, Y)
        counts_h, tok, X, W, Y = cache[(cfg, seed)]
        plan = M.Plan(counts_h, c.H, c.N, int(bm), int(bn), int(flags) | ORDER[order], catalog=catalog)
        ms, mn = time_gemm(plan, X, tok, W, Y, flush, args.reps)
        tf = c.flops / (ms * 1e-3) / 1e12
        kinds = M.parse_plan_blob(plan.blob())["params"][:, 3]
        line = {"case": case, "tile": f"{plan.bm}x{plan.bn}", "catalog": plan.catalog, "swap_tasks": int(kinds.sum()),
                "tiles": plan.total_tiles, "ms": ms, "ms_min": mn,
                "tflops": tf, "frac": tf / peak}
        print(json.dumps(line), flush=True)
        if out:
            out.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
