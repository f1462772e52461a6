"""One moe_gemm launch (after two warm-up launches) of a named config with given plan flags, for an ncu
capture of exactly that launch:  ncu -k regex:moe_gemm_kernel -s 2 -c 1 python scripts/ncu_one.py cfg bm bn flags"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2501_16103_b200 as M  # noqa: E402
import synth  # noqa: E402

cfg, bm, bn, flags = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
c = synth.CONFIGS[cfg]
ids = torch.from_numpy(synth.route(c)).cuda()
X = synth.make_x_torch(0, c.T, c.H, device="cuda")
W = synth.make_w_torch(0, c.E, c.H, c.N, device="cuda")
plan = M.Plan(None, c.H, c.N, bm, bn, flags, E=c.E)
counts, row_off, tok, _, _ = M.moe_route(ids, c.E, plan=plan)
Y = torch.empty((c.T * c.k, c.N), dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    M.moe_gemm(plan, X, tok, W, Y=Y)
torch.cuda.synchronize()
print("ok", cfg, bm, bn, flags)
