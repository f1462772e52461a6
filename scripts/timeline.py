"""Kernel phase timeline of moe_gemm: %globaltimer stamps per CTA from a study build
    scripts/ab_build.sh WORKTREE tl "-DMOE_TIMELINE=1"; MOE_LIB=build_ab/tl/libmoe_sm100.so python scripts/timeline.py
Stamps: 0 entry, 1 after the PDL wait, 2 prologue done, 3 first stage landed, 4 last MMA issued, 5 epilogue done,
6 stores complete; printed as min / median / max over CTAs in us from the first entry."""
import ctypes
import json
import os
import sys

import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_16103_b200 as M, synth
from scripts.tile_probe import CleanFlush
L = M.lib()
L.moe_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
flush = CleanFlush()
def case(name, counts, H, N):
    E = len(counts); T = int(sum(counts))
    ids = np.repeat(np.arange(E, dtype=np.int32), counts)[:, None]
    X = synth.make_x_torch(0, T, H, device="cuda"); W = synth.make_w_torch(0, E, H, N, device="cuda")
    _, _, tok, _, _ = M.moe_route(torch.from_numpy(ids).cuda(), E)
    plan = M.Plan(np.array(counts, np.int32), H, N, 0, 0)
    Y = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
    for _ in range(3): M.moe_gemm(plan, X, tok, W, Y=Y)
    res = []
    for rep in range(5):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        a.record(); M.moe_gemm(plan, X, tok, W, Y=Y); b.record(); b.synchronize()
        buf = np.zeros(1024 * 8, np.uint64)
        L.moe_debug_timeline(buf.ctypes.data, buf.size)
        n = plan.total_tiles if plan.total_tiles < 148 else 148
        tl = buf.reshape(1024, 8)[:n].astype(np.int64)
        base = tl[:, 0].min()
        rel = (tl - base) / 1000.0
        q = {f"s{i}": [round(float(np.min(rel[:, i])), 2), round(float(np.median(rel[:, i])), 2), round(float(np.max(rel[:, i])), 2)] for i in range(8)}
        res.append((a.elapsed_time(b) * 1e3, q))
    ev, q = sorted(res, key=lambda r: r[0])[len(res) // 2]
    print(json.dumps({"case": name, "tiles": plan.total_tiles, "event_us": round(ev, 2), "stamps_us_min_med_max": q}))
case("dec1", [0, 0, 0, 0, 1, 0, 0, 1], 4096, 14336)
case("one_tile_H64", [1], 64, 256)
case("dec1_H64", [0, 0, 0, 0, 1, 0, 0, 1], 64, 14336)
case("dec16", [4, 7, 2, 5, 7, 3, 0, 4], 4096, 14336)
