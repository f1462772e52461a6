"""Per-role cycle breakdown of moe_gemm from the instrumented build (moe_gemm_profile).

    python scripts/gemm_breakdown.py [config] [bn]
Prints one JSON line: fractions of the MMA warp's loop time spent waiting for TMA
bytes vs for a free TMEM accumulator, producer / epilogue figures, and the
kernel time of the plain build for comparison."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2501_16103_b200 as M  # noqa: E402
import synth  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "mix"
    bn = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    bm = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    flags = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    catalog = () if len(sys.argv) > 5 and sys.argv[5] == "none" else None   # "none": one strategy per launch
    fp8 = os.environ.get("FP8", "0") == "1"          # FP8 E4M3 operands (moe_gemm_fp8)
    c = synth.CONFIGS[name]
    ids = torch.from_numpy(synth.route(c, 0)).cuda()
    if fp8:
        from synth import fp8 as sfp8
        X = sfp8.make_x_fp8_torch(0, c.T, c.H, device="cuda")
        W = sfp8.make_w_fp8_torch(0, c.E, c.H, c.N, device="cuda")
        gemm = M.moe_gemm_fp8
    else:
        X = synth.make_x_torch(0, c.T, c.H, device="cuda")
        W = synth.make_w_torch(0, c.E, c.H, c.N, device="cuda")
        gemm = M.moe_gemm
    counts, row_off, tok, _, _ = M.moe_route(ids, c.E)
    plan = M.Plan(counts.cpu().numpy(), c.H, c.N, bm, bn, flags, catalog=catalog)
    Y = torch.empty((tok.numel(), c.N), dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        gemm(plan, X, tok, W, Y=Y)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        gemm(plan, X, tok, W, Y=Y)
    ev[1].record()
    torch.cuda.synchronize()
    t_plain = ev[0].elapsed_time(ev[1]) / 10
    # SM clock under this load: NVML sample in the middle of ~300 ms of back-to-back launches.
    sm_mhz = None
    try:
        import threading
        import time
        import pynvml
        pynvml.nvmlInit()
        hnd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        samples = []

        def sample():
            time.sleep(0.15)
            for _ in range(5):
                samples.append(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM))
                time.sleep(0.02)
        n_launch = max(1, int(300 / max(t_plain, 1e-3)))
        th = threading.Thread(target=sample)
        th.start()
        for _ in range(n_launch):
            gemm(plan, X, tok, W, Y=Y)
        torch.cuda.synchronize()
        th.join()
        sm_mhz = sorted(samples)[len(samples) // 2] if samples else None
    except Exception:  # pragma: no cover - NVML missing
        pass
    Y2 = torch.empty_like(Y)
    M.moe_gemm_profile(plan, X, tok, W, Y2)
    ev[0].record()
    _, prof = M.moe_gemm_profile(plan, X, tok, W, Y2)
    ev[1].record()
    torch.cuda.synchronize()
    t_prof = ev[0].elapsed_time(ev[1])
    pall = prof.double()
    p = pall[0::2] if bm == 256 else pall           # MMA counters live in the pair leaders
    busy = p[:, 6] > 0                              # CTAs (pairs) that processed tiles
    p = p[busy]
    if bm == 256:
        pall = torch.stack([pall[0::2][busy], pall[1::2][busy]], 1).reshape(-1, pall.shape[1])
    tot = p[:, 2]
    out = {
        "config": name, "fp8": fp8, "bn": bn, "bm": bm, "flags": flags, "catalog": plan.catalog, "tiles": plan.total_tiles, "ms_plain": t_plain, "ms_instrumented": t_prof,
        "tflops_plain": c.flops / t_plain / 1e9, "sm_mhz_plain": sm_mhz,
        "tensor_frac_at_clock": (c.flops / t_plain / 1e9) / (148 * 8192 * sm_mhz * 1e-6) if sm_mhz else None,
        "identical_Y": bool(torch.equal(Y, Y2)),
        "mma_wait_full_frac": float((p[:, 1] / tot).mean()),
        "mma_wait_tmem_frac": float((p[:, 0] / tot).mean()),
        "prod_wait_empty_frac": float((p[:, 3] / p[:, 7]).mean()),
        "epi_work_per_tile_cycles": float((p[:, 5] / p[:, 6]).mean()),
        "mma_cycles_per_tile": float((tot / p[:, 6]).mean()),
        "mma_loop_cycles_max": float(tot.max()), "mma_loop_cycles_min": float(tot.min()),
        "tiles_per_cta_min": int(p[:, 6].min()), "tiles_per_cta_max": int(p[:, 6].max()),
        "mma_issue_frac": float((p[:, 8] / tot).mean()),
        "mma_tile_gap_frac": float((p[:, 9] / tot).mean()),
        "b_wait_empty_frac": float((pall[:, 10] / pall[:, 11]).mean()),
        "fill_latency_b_cycles": float((p[:, 12] / p[:, 15]).mean()),
        "fill_latency_a_cycles": float((p[:, 13] / p[:, 15]).mean()),
        "release_to_reissue_cycles": float((p[:, 14] / p[:, 15]).mean()),
        "mma_cycles_per_stage": float((tot / p[:, 15]).mean()),
        # finish spread of the persistent CTA pairs (the launch ends with the slowest one)
        "mma_loop_cycles_quantiles": [float(torch.quantile(tot, q_)) for q_ in (0.0, 0.1, 0.5, 0.9, 1.0)],
        "mma_loop_cycles_mean": float(tot.mean()),
        "tiles_per_cta_hist": {int(k_): int(v_) for k_, v_ in zip(*torch.unique(p[:, 6], return_counts=True))},
    }
    if bm == 256:
        q = pall[1::2]
        out["peer_a_wait_empty_frac"] = float((q[:, 3] / q[:, 7]).mean())
        out["peer_b_wait_empty_frac"] = float((q[:, 10] / q[:, 11]).mean())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
