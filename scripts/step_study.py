#!/usr/bin/env python
"""Where a step's time goes (run on the GPU box): CUDA-graph replays of route(+device plan) alone,
of route + GEMM, and the GEMM alone, each after a clean L2 flush (memset + read), device time."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_16103_b200 as M  # noqa: E402
import synth  # noqa: E402


def graph_of(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def timed(fn, reps=30):
    w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    r = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
    out = []
    for i in range(reps + 3):
        w.zero_()
        r.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i >= 3:
            out.append(a.elapsed_time(b) * 1e3)
    return statistics.median(out)


def main():
    res = []
    for name in sys.argv[1:] or ["dec1", "dec16", "dec256", "mix", "ds"]:
        c = synth.CONFIGS[name]
        topk = torch.from_numpy(synth.route(c, 0)).cuda()
        X = synth.make_x_torch(0, c.T, c.H, device="cuda")
        W = synth.make_w_torch(0, c.E, c.H, c.N, device="cuda")
        bm, bn = M.suggest_tile(c.T * c.k, c.E, c.H, c.N)
        plan = M.Plan(None, c.H, c.N, bm, bn, E=c.E)
        _, _, tok, _, _ = M.moe_route(topk, c.E, with_slot=False, plan=plan)
        Y = M.moe_gemm(plan, X, tok, W)
        g_route = graph_of(lambda: M.moe_route(topk, c.E, with_slot=False, plan=plan))
        g_step = graph_of(lambda: M.moe_gemm(plan, X, M.moe_route(topk, c.E, with_slot=False, plan=plan)[2], W, Y=Y))
        out = {"config": name, "tile": f"{bm}x{bn}",
               "route_graph_us": timed(g_route.replay), "step_graph_us": timed(g_step.replay),
               "gemm_eager_us": timed(lambda: M.moe_gemm(plan, X, tok, W, Y=Y)),
               "empty_graph_us": timed(graph_of(lambda: torch.cuda._sleep(1)).replay)}
        print(json.dumps(out), flush=True)
        res.append(out)
        del W
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/step_study.json", "w"), indent=1)


if __name__ == "__main__":
    main()
