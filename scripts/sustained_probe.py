"""Sustained back-to-back moe_gemm launches (no flush) with the SM clock sampled by NVML: cp.async vs pair gather4 A
staging under the power cap; profiles/r02/sustained_gather4.txt."""
import sys, json, threading, time, numpy as np, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_16103_b200 as M, synth
import pynvml
pynvml.nvmlInit(); hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
def run(cfg, flags, n):
    c = synth.CONFIGS[cfg]
    ids = torch.from_numpy(synth.route(c, 0)).cuda()
    X = synth.make_x_torch(0, c.T, c.H, device="cuda"); W = synth.make_w_torch(0, c.E, c.H, c.N, device="cuda")
    counts, _, tok, _, _ = M.moe_route(ids, c.E)
    plan = M.Plan(counts.cpu().numpy(), c.H, c.N, 256, 512, flags)
    Y = torch.empty((tok.numel(), c.N), dtype=torch.bfloat16, device="cuda")
    for _ in range(5): M.moe_gemm(plan, X, tok, W, Y=Y)
    torch.cuda.synchronize()
    clk = []
    stop = [False]
    def samp():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)); time.sleep(0.01)
    th = threading.Thread(target=samp); th.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): M.moe_gemm(plan, X, tok, W, Y=Y)
    b.record(); b.synchronize(); stop[0] = True; th.join()
    ms = a.elapsed_time(b) / n
    return ms, c.flops / (ms * 1e-3) / 1e12, float(np.median(clk)) if clk else None
for rep in range(2):
    for cfg, n in (("mix", 400), ("ds", 1200), ("ep", 40)):
        for fl in (0, M.MOE_A_GATHER4):
            ms, tf, mhz = run(cfg, fl, n)
            print(json.dumps({"cfg": cfg, "flags": fl, "ms": round(ms * 1e3, 1), "tflops": round(tf, 1), "sm_mhz": mhz}), flush=True)
