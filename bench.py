#!/usr/bin/env python
"""Benchmark of the statically batched MoE expert GEMM (arXiv 2501.16103) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config mix]
                    [--dtype bf16|fp8] [--ffn] [--ep] [--host-plan] [--order natural|...]

A step = one pass of the whole hot path over one batch of synthetic input:
moe_route_plan (device buckets + the device-built compressed mapping, Alg. 1 + sigma) ->
moe_gemm (one tcgen05 launch over every expert tile), replayed as one CUDA graph; --host-plan
plans on the host instead (counts D2H, blob H2D).  `value` = useful FLOPs (2 * sum m_e * H * N)
/ device step time, inputs resident in HBM; `e2e` = the same metric through the public API with
X / top-k ids copied from pinned host memory and Y copied back inside the timed region.  L2 is
flushed (256 MiB memset, then a 256 MiB read so no dirty line is left to write back) before
every timed step.  `--impl reference` times the fp64 CPU oracle on a bounded sample of the same
workload (the tier's reference arm).

Multi-GPU (torchrun, N > 1) or --ep: the expert-parallel step in the library (moe_ep_forward,
NCCL from C++; --ep-python: the torch.distributed orchestration) — weak scaling on the Mix shape,
strong scaling on the 8x22B `ep` shape.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "MoE GEMM TFLOPS and % of B200 BF16 tensor peak at 1/2/4/8 GPUs"
ORDER_FLAGS = {"natural": 0, "alternating": 4, "half_interval": 8, "light_last": 4096}   # MOE_ORDER_* (include/moe_sm100.h)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_traffic(workload: str):
    """dram bytes per launch of moe_gemm_kernel from the committed ncu --set full summary."""
    v = load_ncu(workload)
    return (v.get("dram_bytes_per_launch"), v.get("source")) if v else (None, None)


def load_ncu(workload: str) -> dict:
    """The committed ncu --set full summary of moe_gemm_kernel for this workload (profiles/traffic.json:
    DRAM bytes, tensor-pipe and DRAM-throughput % of peak, ncu's own duration and SM clock)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(workload) or {}
    return {}


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg / reference arm)
# ---------------------------------------------------------------------------
def oracle_sample(cfg, seed: int, budget_s: float, cache: dict | None = None, fp8: bool = False):
    """Times oracle.moe.expert_gemm (fp8: oracle.fp8.expert_gemm_fp8 on E4M3 codes) expert by expert
    on the workload until budget_s of CPU work has been spent (input generation excluded).
    Returns (flops, seconds, sample, cores)."""
    from oracle import fp8 as ofp8
    from oracle import moe as omoe
    from synth import fp8 as sfp8
    try:
        from threadpoolctl import threadpool_info
        cores = sum(int(i.get("num_threads", 1)) for i in threadpool_info() if i.get("user_api") == "blas") or 1
    except Exception:  # pragma: no cover
        cores = os.cpu_count()
    cache = {} if cache is None else cache
    if "inputs" not in cache:
        ids = synth.route(cfg, seed)
        cache["inputs"] = (omoe.buckets(ids, cfg.E),
                           sfp8.make_x_fp8(seed, cfg.T, cfg.H) if fp8 else synth.make_x(seed, cfg.T, cfg.H))
    (counts, row_off, tok, _), X = cache["inputs"]
    flops, secs, done = 0, 0.0, []
    for e in range(cfg.E):
        if counts[e] == 0:
            continue
        if e not in cache:                                               # generation is not timed
            cache[e] = (sfp8.w_fp8_columns(seed, cfg.E, cfg.H, cfg.N, e, np.arange(cfg.N))[None] if fp8
                        else synth.make_w(seed, cfg.E, cfg.H, cfg.N, experts=[e]))   # [1, H, N]
        W = cache[e]
        a, b = int(row_off[e]), int(row_off[e + 1])
        sub_tok = tok[a:b]
        t0 = time.perf_counter()
        if fp8:
            ofp8.expert_gemm_fp8(X, W, sub_tok, np.array([0, b - a]), [2.0 ** -synth.w_scale_exp(cfg.H)])
        else:
            omoe.expert_gemm(X, W, sub_tok, np.array([0, b - a]))
        secs += time.perf_counter() - t0
        flops += 2 * (b - a) * cfg.H * cfg.N
        done.append(e)
        if secs >= budget_s:
            break
    sample = (f"{cfg.name} seed {seed}: experts {done} ({int(sum(counts[e] for e in done))} of "
              f"{int(counts.sum())} rows, full H x N), fp64 numpy/OpenBLAS" + (" on decoded E4M3 codes" if fp8 else ""))
    return flops, secs, sample, cores


def ref_config(cfg, args, ws: int) -> dict:
    """The reference arm reports the `config` our arm prints for the same command (the tile label is the
    planner's host rule, moe_plan_suggest_tile; nothing of our engine runs in this arm)."""
    if ws > 1 or args.ep:
        return ep_config(cfg, ws, args)
    import paper_2501_16103_b200 as M
    if not (args.bm or args.bn):
        args.bm_resolved, args.bn_resolved = M.suggest_tile(cfg.T * cfg.k, cfg.E, cfg.H, cfg.N)
    return config_dict(cfg, args)


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    # warm-up: one small expert product so BLAS threads exist
    from oracle import moe as omoe
    omoe.expert_gemm(np.ones((8, 64)), np.ones((1, 64, 64)), np.arange(8), np.array([0, 8]))
    per_step = max(1.0, 60.0 / max(args.steps + args.warmup, 1))
    vals, ms = [], []
    info = None
    cache = {}
    for i in range(args.warmup + args.steps):
        f, s, sample, cores = oracle_sample(cfg, args.seed, per_step, cache)
        if i >= args.warmup:
            vals.append(f / s / 1e12)
            ms.append(s * 1e3)
            info = (sample, cores)
    v = float(statistics.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(statistics.mean(ms)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": ref_config(cfg, args, ws),
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": info[1], "kind": "oracle", "sample": info[0]},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class L2Flush:
    """Between timed steps: write a 256 MiB buffer (evicts everything), then read another 256 MiB
    one, so L2 holds only clean lines of the flush buffer.  The timed kernel then misses in L2 for
    all its inputs and does not pay the HBM write-back of the flush's own dirty lines (the state
    ncu's --cache-control all gives a replayed kernel).  `write_only()` is the plain memset flush."""

    def __init__(self, torch, dev):
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        self.r = torch.ones(32 << 20, dtype=torch.int64, device=dev)

    def write_only(self):
        self.w.zero_()

    def __call__(self):
        self.w.zero_()
        self.r.sum()


def host_pad(torch, ms: float = 2.0):
    """Queue a GPU sleep so the host enqueues the timed launches before the device reaches them:
    events then bracket device time only, not the Python/ctypes launch latency of an eager call."""
    torch.cuda._sleep(int(ms * 2.0e6))             # ~2e6 cycles per ms at the 1.9-2.0 GHz boost clock


def route_launches(T: int, E: int, k: int = 2) -> int:
    """Kernels one moe_route(_plan) call launches (route.cu): the single-block small-batch kernel
    when T <= 1024, E <= 16, k <= 8; else histogram + fused scan/compaction while chunks x experts
    <= 16384, else histogram + scan + compaction."""
    if T <= 1024 and E <= 16 and k <= 8:
        return 1
    chunks = max(1, -(-T // 1024))
    return 2 if chunks * E <= 16384 else 3


def run_ffn(args, cfg):
    """--ffn: the full MoE FFN layer on the config's shape, N = the FFN width I:
    route + device plans -> moe_gemm_swiglu (gate/up, SwiGLU epilogue) -> moe_gemm (down, H_out = H)
    -> moe_combine, one CUDA graph per step.  Useful flops = 6 * sum(m_e) * H * I."""
    import torch

    import paper_2501_16103_b200 as M

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    M.moe_device_info()
    peaks, peak_src = load_peaks()
    H, I, E = cfg.H, cfg.N, cfg.E
    ids = synth.route(cfg, args.seed)
    topk_d = torch.from_numpy(ids).to(dev)
    rng = np.random.default_rng(args.seed)
    w = rng.random((cfg.T, cfg.k)).astype(np.float32)
    w /= w.sum(axis=1, keepdims=True)
    w_d = torch.from_numpy(w).to(dev)
    Xd = synth.make_x_torch(args.seed, cfg.T, H, device=dev)
    Wg = synth.make_w_torch(args.seed, E, H, I, device=dev)
    Wu = synth.make_w_torch(args.seed + 1, E, H, I, device=dev)
    Wdn = synth.make_w_torch(args.seed + 2, E, I, H, device=dev)
    layer = M.MoeFFN(Wg, Wu, Wdn)
    out = torch.empty((cfg.T, H), dtype=torch.bfloat16, device=dev)
    flush = L2Flush(torch, dev)
    stream = torch.cuda.current_stream()
    rows = int((ids >= 0).sum())
    flops = 6.0 * rows * H * I
    for _ in range(args.warmup):
        layer.forward(Xd, topk_d, w_d, out=out)
    torch.cuda.synchronize()
    # per-stage times (eager, events on the launching stream)
    stages = {"route_plans": [], "swiglu_gemm": [], "down_gemm": [], "combine": []}
    for _ in range(max(3, min(args.steps, 10))):
        flush()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        host_pad(torch)
        ev[0].record(stream)
        counts, row_off, tok, slot, _ = M.moe_route(topk_d, E, plan=layer.plan_gu)
        layer.plan_dn.update_device(counts)
        ev[1].record(stream)
        h = M.moe_gemm_swiglu(layer.plan_gu, Xd, tok, Wg, Wu)
        ev[2].record(stream)
        y = M.moe_gemm(layer.plan_dn, h, None, Wdn, out_dtype=torch.float32)
        ev[3].record(stream)
        M.moe_combine(y, tok, slot, row_off, w_d, out=out)
        ev[4].record(stream)
        ev[4].synchronize()
        for i, k in enumerate(stages):
            stages[k].append(ev[i].elapsed_time(ev[i + 1]))
    st = {k: statistics.mean(v) for k, v in stages.items()}
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        layer.forward(Xd, topk_d, w_d, out=out)
    stream.wait_stream(side)
    with torch.cuda.graph(graph):
        layer.forward(Xd, topk_d, w_d, out=out)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    step_ms = []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            flush()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            host_pad(torch, 0.5)
            s0.record(stream)
            graph.replay()
            s1.record(stream)
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
    ms = statistics.mean(step_ms)
    peak = float(peaks["bf16_tflops"])
    gu = 4.0 * rows * H * I / (st["swiglu_gemm"] * 1e-3) / 1e12
    dn = 2.0 * rows * H * I / (st["down_gemm"] * 1e-3) / 1e12
    comb_bytes = rows * H * 4 + cfg.T * H * 2 + cfg.T * cfg.k * 8      # fp32 expert rows in, bf16 out
    line = {
        "metric": "MoE FFN layer TFLOP/s (SwiGLU gate/up + down + weighted combine)", "value": flops / (ms * 1e-3) / 1e12,
        "unit": "TFLOP/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "cuda_graph": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name} FFN: E={E} top-{cfg.k} T={cfg.T} H={H} I={I} routing={cfg.routing} "
                               f"seed={args.seed}", "tiles": f"gate/up {layer.plan_gu.bm}x{layer.plan_gu.bn} (x2 "
                               f"accumulators), down {layer.plan_dn.bm}x{layer.plan_dn.bn}",
                   "l2": "flushed before every timed step (256 MiB memset + 256 MiB read: clean L2)"},
        "stages_ms": st,
        "kernels": {"swiglu_gemm_tflops": gu, "down_gemm_tflops": dn,
                    "combine_gbs": comb_bytes / (st["combine"] * 1e-3) / 1e9},
        "roofline": {"bound": "tensor", "achieved": gu, "peak": peak, "unit": "TFLOP/s", "frac": gu / peak,
                     "traffic": None, "kernel": "moe_gemm_kernel (gated)", "peak_source": peak_src},
        "gpu_launches": (route_launches(cfg.T, E, cfg.k) + 1 + 1 + 1 + 2) * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def ep_workload(base, ws: int):
    """The expert-parallel workload at ws ranks: strong scaling on the 8x22B `ep` shape (total T fixed),
    weak scaling otherwise (T per rank fixed).  Returns (config, strong, T per rank, experts per rank)."""
    strong = base.name == "ep"
    T_total = base.T if strong else base.T * ws
    if base.E % ws or T_total % ws:
        raise SystemExit(f"E={base.E} and T={T_total} must be divisible by {ws} ranks")
    cfg = synth.Config(f"{base.name}-ep{ws}", E=base.E, k=base.k, T=T_total, H=base.H, N=base.N,
                       routing=base.routing, zipf_s=base.zipf_s, n_empty=base.n_empty)
    return cfg, strong, T_total // ws, base.E // ws


def ep_config(base, ws: int, args) -> dict:
    """`config` of an N > 1 line (both arms print the same one)."""
    import paper_2501_16103_b200 as M
    cfg, _, T_l, El = ep_workload(base, ws)
    bm, bn = (args.bm, args.bn) if args.bm or args.bn else M.suggest_tile(T_l * cfg.k, El, cfg.H, cfg.N)
    return {"workload": f"{cfg.name}: E={cfg.E} top-{cfg.k} T={cfg.T} ({T_l}/rank) H={cfg.H} N={cfg.N} "
                        f"routing={cfg.routing} seed={args.seed}",
            "tile": f"{bm}x{bn}", "out_dtype": args.out_dtype,
            "operands": "FP8 E4M3 X and W, per-expert fp32 scale" if getattr(args, "dtype", "bf16") == "fp8" else "bf16",
            "global_batch": cfg.T, "parallelism": f"ep{ws}",
            "l2": "flushed before every timed step (memset + read: clean L2)"}


def config_dict(cfg, args):
    return {"workload": f"{cfg.name}: E={cfg.E} top-{cfg.k} T={cfg.T} H={cfg.H} N={cfg.N} "
                        f"routing={cfg.routing} seed={args.seed}",
            "tile": f"{getattr(args, 'bm_resolved', args.bm) or 'auto'}x{getattr(args, 'bn_resolved', args.bn) or 'auto'}", "out_dtype": args.out_dtype,
            "planner": "host (counts D2H + moe_plan_update)" if args.host_plan else "device (moe_plan_device)", "global_batch": cfg.T,
            "operands": "FP8 E4M3 X and W, per-expert fp32 scale" if getattr(args, "dtype", "bf16") == "fp8" else "bf16",
            "task_order": getattr(args, "order", "natural"),
            "l2": "flushed before every timed step (256 MiB memset + 256 MiB read: clean L2); W alone exceeds L2",
            "timing": "CUDA events on the launching stream; a GPU sleep queued ahead of each timed step "
                      "keeps host launch latency out of the device time (e2e includes it)",
            "parallelism": f"ep{args.gpus}" if args.gpus > 1 else "1 GPU"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch

    import paper_2501_16103_b200 as M

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    M.moe_device_info()
    peaks, peak_src = load_peaks()
    out_dtype = torch.bfloat16 if args.out_dtype == "bf16" else torch.float32

    ids = synth.route(cfg, args.seed)
    topk_d = torch.from_numpy(ids).to(dev)
    fp8 = args.dtype == "fp8"
    if fp8:                                        # FP8 E4M3 codes + per-expert scale (synth/fp8.py)
        from synth import fp8 as sfp8
        Xd = sfp8.make_x_fp8_torch(args.seed, cfg.T, cfg.H, device=dev)
        Wd = sfp8.make_w_fp8_torch(args.seed, cfg.E, cfg.H, cfg.N, device=dev)
        w_scale = torch.from_numpy(sfp8.w_scale(cfg.E, cfg.H)).to(dev)
    else:
        Xd = synth.make_x_torch(args.seed, cfg.T, cfg.H, device=dev)
        Wd = synth.make_w_torch(args.seed, cfg.E, cfg.H, cfg.N, device=dev)
        w_scale = None
    esz = 1 if fp8 else 2

    def gemm(plan, X, tok, W, Y=None):
        if fp8:
            return M.moe_gemm_fp8(plan, X, tok, W, w_scale, Y=Y, out_dtype=out_dtype)
        return M.moe_gemm(plan, X, tok, W, Y=Y, out_dtype=out_dtype)
    flush = L2Flush(torch, dev)
    flops = cfg.flops
    stream = torch.cuda.current_stream()

    plan = None

    def step(Y=None, pad_gemm=False):
        nonlocal plan
        if args.host_plan:                         # P:142 option 1: counts D2H, plan on the host
            counts, row_off, tok, slot, _ = M.moe_route(topk_d, cfg.E, with_slot=False)
            counts_h = counts.cpu().numpy()
            if plan is None:
                plan = M.Plan(counts_h, cfg.H, cfg.N, args.bm, args.bn, ORDER_FLAGS[args.order])
            else:
                plan.update(counts_h)
        else:                                      # P:142 option 2: plan generated on the device,
            if plan is None:                       # fused into the routing scan (moe_route_plan)
                bm, bn = (args.bm, args.bn) if args.bm or args.bn else M.suggest_tile(cfg.T * cfg.k, cfg.E, cfg.H, cfg.N)
                plan = M.Plan(None, cfg.H, cfg.N, bm, bn, ORDER_FLAGS[args.order], E=cfg.E)
            counts, row_off, tok, slot, _ = M.moe_route(topk_d, cfg.E, with_slot=False, plan=plan)
        if pad_gemm:                               # host-planned: the host synchronised above; let it
            host_pad(torch, 0.2)                   # enqueue the GEMM before the device reaches g0
        g0 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        Y = gemm(plan, Xd, tok, Wd, Y=Y)
        return Y, g0

    Y0, _ = step()
    Ybuf = torch.empty_like(Y0)
    for _ in range(args.warmup):
        step(Ybuf)
    torch.cuda.synchronize()

    # (1) eager steps: per-launch GEMM time on the launching stream (the roofline's kernel time).
    # A GPU sleep ahead of each step lets the host enqueue it first, so the events see device time
    # only (the host-planned mode still synchronises inside the step, before the GEMM launch).
    step_ms_eager, gemm_ms = [], []
    for _ in range(args.steps):
        flush()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        host_pad(torch)
        s0.record(stream)
        _, g0 = step(Ybuf, pad_gemm=args.host_plan)
        s1.record(stream)
        s1.synchronize()
        step_ms_eager.append(s0.elapsed_time(s1))
        gemm_ms.append(g0.elapsed_time(s1))
    # the same launches after a write-only (memset) flush: the kernel also pays the HBM write-back of
    # the flush's dirty lines (reported beside the clean-L2 time, not used for the roofline)
    gemm_ms_dirty = []
    for _ in range(min(args.steps, 10)):
        flush.write_only()
        s1 = torch.cuda.Event(enable_timing=True)
        host_pad(torch)
        _, g0 = step(Ybuf, pad_gemm=args.host_plan)
        s1.record(stream)
        s1.synchronize()
        gemm_ms_dirty.append(g0.elapsed_time(s1))
    # the same launches back to back, one event pair around all of them, no flush in between (every BASELINE
    # shape's W is larger than the 126 MB L2): the per-launch event bracket above carries a fixed ~6 us (an
    # empty kernel measures 6.1 us that way) that this average does not (reported beside the
    # roofline's clean-L2 per-launch time, not used for it)
    _, _, tok_b, _, _ = M.moe_route(topk_d, cfg.E, with_slot=False, plan=plan) if not args.host_plan else \
        M.moe_route(topk_d, cfg.E, with_slot=False)
    gemm(plan, Xd, tok_b, Wd, Y=Ybuf)
    torch.cuda.synchronize()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host_pad(torch)
    b0.record(stream)
    for _ in range(args.steps):
        gemm(plan, Xd, tok_b, Wd, Y=Ybuf)
    b1.record(stream)
    b1.synchronize()
    gemm_ms_b2b = b0.elapsed_time(b1) / args.steps
    # (2) the step as one CUDA graph (route + device plan + GEMM, no host synchronisation inside)
    graph = None
    if args.graph and not args.host_plan:
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step(Ybuf)                                   # warm the capture stream
        stream.wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            _, _, tok_g, _, _ = M.moe_route(topk_d, cfg.E, with_slot=False, plan=plan)
            gemm(plan, Xd, tok_g, Wd, Y=Ybuf)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
    step_ms = []
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            host_pad(torch, 0.5)
            s0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                step(Ybuf)
            s1.record(stream)
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    t_total = sum(step_ms)
    if ws > 1:
        t = torch.tensor([t_total], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_total = float(t.item())
    value = flops * ws * args.steps / (t_total * 1e-3) / 1e12
    gemm_avg = statistics.mean(gemm_ms)
    achieved = flops / (gemm_avg * 1e-3) / 1e12
    # FP8 contractions take the bf16 measured peak x the nominal FP8 / BF16 ratio (4.5 / 2.25 PF).
    peak = float(peaks["bf16_tflops"]) * (2.0 if fp8 else 1.0)
    # Algorithmic HBM bytes of one moe_gemm launch: W of active experts, the token
    # rows routed anywhere, Y (out dtype) and the token-index array.
    counts_np = np.bincount(ids.ravel(), minlength=cfg.E)
    ybytes = 2 if out_dtype == torch.bfloat16 else 4
    n_tokens = int((ids >= 0).any(axis=1).sum())   # distinct tokens routed anywhere: each X row is read once
    alg_bytes = (int((counts_np > 0).sum()) * cfg.H * cfg.N * esz + n_tokens * cfg.H * esz
                 + int(counts_np.sum()) * (cfg.N * ybytes + 4) + (4 * cfg.E if fp8 else 0))
    hbm = float(peaks["hbm_gbs"])
    mem_bound = flops / alg_bytes < peak * 1e12 / (hbm * 1e9)
    traffic, tsrc = load_traffic(("fp8_" if fp8 else "") + cfg.name)
    ncu = load_ncu(("fp8_" if fp8 else "") + cfg.name)

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        X_h = (sfp8.make_x_fp8_torch(args.seed, cfg.T, cfg.H) if fp8
               else synth.make_x_torch(args.seed, cfg.T, cfg.H)).pin_memory()
        ids_h = torch.from_numpy(ids).pin_memory()
        Y_h = torch.empty(Y0.shape, dtype=Y0.dtype).pin_memory()
        Xe = torch.empty_like(Xd)
        te = torch.empty_like(topk_d)

        def e2e_step():
            if graph is not None:                  # the captured step reads Xd / topk_d
                Xd.copy_(X_h, non_blocking=True)
                topk_d.copy_(ids_h, non_blocking=True)
                graph.replay()
                Y_h.copy_(Ybuf, non_blocking=True)
                return None
            Xe.copy_(X_h, non_blocking=True)
            te.copy_(ids_h, non_blocking=True)
            Y, counts, _, _, _, _ = M.moe_forward(te, Xe, Wd, cfg.E, bm=args.bm, bn=args.bn, out_dtype=out_dtype,
                                                  plan=plan, device_plan=not args.host_plan, Y=Ybuf, scale=w_scale)
            Y_h.copy_(Y, non_blocking=True)
            return counts

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        e_ms = []
        for _ in range(max(3, min(args.steps, 10))):
            flush()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            e2e_step()
            s1.record(stream)
            s1.synchronize()
            e_ms.append(s0.elapsed_time(s1))
        h2d = X_h.numel() * X_h.element_size() + ids_h.numel() * 4
        d2h = Y_h.numel() * Y_h.element_size()
        if args.host_plan:
            h2d += 4 * plan.blob().size            # plan blob upload
            d2h += 4 * cfg.E                       # counts read back for the host planner
        serial_ms = statistics.mean(e_ms)
        # Pipelined serving loop through the same public API: step i's H2D, step i-1's compute and
        # step i-2's D2H overlap on three streams (inputs and outputs double-buffered); the timed
        # region covers every step's copies.  The PCIe read-back of Y bounds it.
        pipe_ms = None
        if not args.host_plan:
            s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
            Xb = [torch.empty_like(Xd) for _ in range(2)]
            tb = [torch.empty_like(topk_d) for _ in range(2)]
            Yb = [torch.empty_like(Ybuf) for _ in range(2)]
            Yh = [Y_h, torch.empty(Y0.shape, dtype=Y0.dtype).pin_memory()]
            ev_in = [torch.cuda.Event() for _ in range(2)]
            ev_comp = [torch.cuda.Event() for _ in range(2)]
            ev_out = [torch.cuda.Event() for _ in range(2)]
            n_pipe = max(4, min(args.steps, 12))

            def run_pipe(n):
                for i in range(n):
                    b = i % 2
                    with torch.cuda.stream(s_in):
                        if i >= 2:
                            s_in.wait_event(ev_comp[b])          # step i-2 has consumed Xb[b], tb[b]
                        Xb[b].copy_(X_h, non_blocking=True)
                        tb[b].copy_(ids_h, non_blocking=True)
                        ev_in[b].record(s_in)
                    stream.wait_event(ev_in[b])
                    if i >= 2:
                        stream.wait_event(ev_out[b])             # step i-2's D2H has read Yb[b]
                    M.moe_forward(tb[b], Xb[b], Wd, cfg.E, bm=args.bm, bn=args.bn, out_dtype=out_dtype, plan=plan,
                                  Y=Yb[b], scale=w_scale)
                    ev_comp[b].record(stream)
                    with torch.cuda.stream(s_out):
                        s_out.wait_event(ev_comp[b])
                        Yh[b].copy_(Yb[b], non_blocking=True)
                        ev_out[b].record(s_out)
                stream.wait_stream(s_in)
                stream.wait_stream(s_out)

            run_pipe(2)
            torch.cuda.synchronize()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            s_in.wait_stream(stream)
            run_pipe(n_pipe)
            p1.record(stream)
            p1.synchronize()
            pipe_ms = p0.elapsed_time(p1) / n_pipe
        e_best = pipe_ms if pipe_ms is not None else serial_ms
        e2e = {"value": flops / (e_best * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e_best, "mode": "pipelined: H2D / compute / D2H on three streams, double-buffered"
               if pipe_ms is not None else "serial", "serial_ms_per_step": serial_ms}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        f, s, sample, cores = oracle_sample(cfg, args.seed, args.cpu_budget, fp8=fp8)
        cpu = {"value": f / s / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample,
               "seconds": s}

    args.bm_resolved, args.bn_resolved = plan.bm, plan.bn
    # Host planner time (Alg. 1 + sigma + task table for this step's counts; SURVEY §8(d) reports it
    # apart from the kernel), median of 50 calls of moe_plan_build.
    hp = []
    for _ in range(50):
        t0 = time.perf_counter()
        M.moe_plan_build(counts_np.astype(np.int32), cfg.H, cfg.N, plan.bm, plan.bn)
        hp.append((time.perf_counter() - t0) * 1e6)
    host_plan_us = statistics.median(hp)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.mean(step_ms), "higher_is_better": True,
            "ms_per_step_eager": None if args.host_plan else statistics.mean(step_ms_eager),
            "cuda_graph": graph is not None,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp8_e4m3" if fp8 else "bf16", "data": "synthetic",
            "config": config_dict(cfg, args),
            "pct_of_peak": value / peak,
            "step_ms_median": statistics.median(step_ms), "step_ms_min": min(step_ms),
            "host_plan_us": host_plan_us,
            "kernel": {"name": "moe_gemm_kernel", "ms_per_launch": gemm_avg, "tflops": achieved,
                       "ms_per_launch_median": statistics.median(gemm_ms), "ms_per_launch_min": min(gemm_ms),
                       "ms_per_launch_after_memset_flush": statistics.mean(gemm_ms_dirty),
                       "ms_per_launch_back_to_back": gemm_ms_b2b,
                       "pct_of_measured_burst_peak": achieved / peak,
                       "pct_of_measured_sustained_peak": achieved / (float(peaks["bf16_tflops_sustained"])
                                                                     * (2.0 if fp8 else 1.0)),
                       "pct_of_datasheet_2250": achieved / (4500.0 if fp8 else 2250.0)},
            "roofline": ({"bound": "hbm", "achieved": alg_bytes / (gemm_avg * 1e-3) / 1e9, "peak": hbm,
                          "unit": "GB/s", "frac": alg_bytes / (gemm_avg * 1e-3) / 1e9 / hbm, "traffic": traffic,
                          "peak_source": f"{peak_src} hbm_gbs", "algorithmic_bytes_per_launch": alg_bytes,
                          "algorithmic_flops_per_launch": flops, "traffic_source": tsrc}
                         if mem_bound else
                         {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                          "frac": achieved / peak, "traffic": traffic,
                          "peak_source": f"{peak_src} bf16_tflops (burst; kernel timed per launch)"
                                         + (" x 2 (nominal FP8 / BF16 dense ratio, 4.5 / 2.25 PF)" if fp8 else ""),
                          "algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": alg_bytes,
                          "traffic_source": tsrc}),
            "ncu": ({"tensor_pipe_pct": ncu.get("tensor_pipe_pct"), "dram_throughput_pct": ncu.get("dram_throughput_pct"),
                     "traffic_over_algorithmic": traffic / alg_bytes if traffic else None,
                     "ncu_us": ncu.get("ncu_us"), "ncu_sm_mhz": ncu.get("sm_mhz"), "source": ncu.get("source")}
                    if ncu else None),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": (route_launches(cfg.T, cfg.E, cfg.k) + 1) * args.steps,   # route (+plan), GEMM
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------
# multi-GPU: expert parallelism (one process per GPU, NCCL all-to-all dispatch / combine)
# ---------------------------------------------------------------------------
def run_ep(args, base):
    import torch
    import torch.distributed as dist

    import paper_2501_16103_b200 as M
    from paper_2501_16103_b200.ep import ExpertParallelMoE, TorchComm

    for k_, v_ in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531"), ("RANK", "0"), ("WORLD_SIZE", "1")):
        os.environ.setdefault(k_, v_)                 # `--ep` on one GPU without torchrun
    ws, rank, local = dist_env()
    # More ranks than GPUs (a functional run of the multi-rank path on a smaller box): ranks share
    # devices, the process group is gloo (NCCL refuses two ranks on one GPU), the peer transport maps
    # regions with CUDA IPC on the same device.  The line says so; it is not a scaling number.
    n_dev = torch.cuda.device_count()
    shared = n_dev < ws
    local = local % n_dev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    cdev = torch.device("cpu") if shared else dev    # where the bench's own small collectives run
    M.moe_device_info()
    peaks, peak_src = load_peaks()
    out_dtype = torch.bfloat16 if args.out_dtype == "bf16" else torch.float32
    cfg, strong, T_l, El = ep_workload(base, ws)
    T_total = cfg.T
    ids = synth.route(cfg, args.seed)               # the global batch (identical on every rank)
    topk_l = torch.from_numpy(np.ascontiguousarray(ids[rank * T_l:(rank + 1) * T_l])).to(dev)
    fp8 = args.dtype == "fp8"
    if fp8:                                          # FP8 E4M3 rows and weights (synth/fp8.py, R15)
        from synth import fp8 as sfp8
        X_l = sfp8.make_x_fp8_torch(args.seed, T_l, cfg.H, device=dev, row0=rank * T_l)
        W_l = sfp8.make_w_fp8_torch(args.seed, cfg.E, cfg.H, cfg.N, device=dev, experts=range(rank * El, (rank + 1) * El))
        w_scale = torch.from_numpy(sfp8.w_scale(El, cfg.H)).to(dev)
    else:
        X_l = synth.counter_values_torch(args.seed, synth.workloads.STREAM_X, rank * T_l * cfg.H, T_l * cfg.H,
                                         "normal", 6, dev).reshape(T_l, cfg.H)
        W_l = synth.make_w_torch(args.seed, cfg.E, cfg.H, cfg.N, device=dev, experts=range(rank * El, (rank + 1) * El))
        w_scale = None
    native = None
    peer = not args.ep_python and args.ep_transport == "peer"
    out_view = None
    peer_fallback = None
    if peer:                                         # the library's moe_ep_* step over symmetric peer memory
        y_bytes = cfg.N * (2 if out_dtype == torch.bfloat16 else 4)
        native, err = None, None
        try:
            native = M.PeerExpertParallel(rank, ws, cfg.E, W_l, max_tokens=T_l, k=cfg.k, w_scale=w_scale,
                                          bm=args.bm, bn=args.bn, max_out_bytes=y_bytes, connect=False)
        except Exception as e:  # pragma: no cover - region allocation failed
            err = repr(e)[:200]
        blobs = [None] * ws
        dist.all_gather_object(blobs, native.blob if native is not None else None)
        if native is not None and all(b is not None for b in blobs):
            try:
                native.connect(blobs)                # CUDA IPC mappings of every peer's region
            except Exception as e:  # pragma: no cover - e.g. no P2P / IPC between these GPUs
                err = repr(e)[:200]
        ok = [None] * ws
        dist.all_gather_object(ok, err)
        if any(o is not None for o in ok) or any(b is None for b in blobs):
            # every rank falls back together: the NCCL transport of the same library step
            peer_fallback = next(o for o in ok if o is not None) if any(o is not None for o in ok) else "no blob"
            native, peer = None, False
            dist.barrier()
        else:
            out_view = native.output(T_l, cfg.N, out_dtype)      # zero copy: the rows stay in the output buffer
    if not peer and not args.ep_python:              # the library's moe_ep_* step (NCCL from C++)
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(M.moe_ep_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        native = M.NativeExpertParallel(bytes(uid.cpu().numpy().tobytes()), rank, ws, cfg.E, W_l, w_scale=w_scale,
                                        bm=args.bm, bn=args.bn)
    moe = ExpertParallelMoE(cfg.E, W_l, TorchComm(), bm=args.bm, bn=args.bn, out_dtype=out_dtype, w_scale=w_scale)
    flush = L2Flush(torch, dev)
    stream = torch.cuda.current_stream()
    if peer:
        fwd = lambda t, x: native.forward(t, x, out=out_view)            # noqa: E731
    elif native is not None:
        fwd = lambda t, x: native.forward(t, x, out_dtype=out_dtype)     # noqa: E731
    else:
        fwd = moe.forward
    for _ in range(args.warmup):
        fwd(topk_l, X_l)
    torch.cuda.synchronize()
    moe.time_gemm = True
    step_ms, gemm_ms, local_rows = [], [], []
    dist.barrier()
    torch.cuda.synchronize()

    def aligned_start():
        # every rank's device reaches the step together: flush, drain, host barrier, then a GPU sleep
        # queued ahead of the step so the host enqueues it before the device gets there
        flush()
        torch.cuda.synchronize()
        dist.barrier()
        host_pad(torch)

    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            aligned_start()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            fwd(topk_l, X_l)
            s1.record(stream)
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            if native is None:
                gemm_ms.append(moe.gemm_events[0].elapsed_time(moe.gemm_events[1]))
                local_rows.append(moe.last["local_rows"])
            else:                                    # events the library records around its GEMM launch
                gemm_ms.append(native.last_gemm_ms())
                local_rows.append(native.last_rows()["local_rows"])
        # The peer-memory step has no host synchronisation inside: replay it as one CUDA graph (the
        # eager steps above give the GEMM's own launch time).
        graph, graph_err = None, None
        if peer and args.graph:
            try:
                side = torch.cuda.Stream()
                side.wait_stream(stream)
                with torch.cuda.stream(side):
                    fwd(topk_l, X_l)
                stream.wait_stream(side)
                torch.cuda.synchronize()
                dist.barrier()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    fwd(topk_l, X_l)
                torch.cuda.synchronize()
                dist.barrier()
                graph.replay()                       # one untimed replay (every rank replays in lockstep)
                torch.cuda.synchronize()
            except Exception as e:  # pragma: no cover
                graph, graph_err = None, repr(e)[:200]
        step_ms_eager = list(step_ms)
        if graph is not None:
            step_ms = []
            for _ in range(args.steps):
                aligned_start()
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record(stream)
                graph.replay()
                s1.record(stream)
                s1.synchronize()
                step_ms.append(s0.elapsed_time(s1))
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([sum(step_ms)], device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    value = cfg.flops * args.steps / (float(t.item()) * 1e-3) / 1e12
    gemm_avg = statistics.mean(gemm_ms)
    flops_l = 2 * local_rows[-1] * cfg.H * cfg.N
    achieved = flops_l / (gemm_avg * 1e-3) / 1e12
    peak = float(peaks["bf16_tflops"]) * (2.0 if fp8 else 1.0)
    per_rank = torch.tensor([statistics.mean(step_ms), gemm_avg, achieved], device=cdev)
    gathered = [torch.zeros_like(per_rank) for _ in range(ws)]
    dist.all_gather(gathered, per_rank)
    # e2e: the rank's X / top-k ids from pinned host memory, result rows back to the host
    e2e = None
    if not args.no_e2e:
        X_h = X_l.cpu().pin_memory()
        ids_h = topk_l.cpu().pin_memory()
        out0 = fwd(topk_l, X_l)
        out_h = torch.empty(out0.shape, dtype=out0.dtype).pin_memory()
        Xe, te = torch.empty_like(X_l), torch.empty_like(topk_l)
        e_ms = []
        for i in range(2 + max(3, min(args.steps, 10))):
            flush()
            dist.barrier()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            Xe.copy_(X_h, non_blocking=True)
            te.copy_(ids_h, non_blocking=True)
            out_h.copy_(fwd(te, Xe), non_blocking=True)
            s1.record(stream)
            s1.synchronize()
            if i >= 2:
                e_ms.append(s0.elapsed_time(s1))
        te_max = torch.tensor([sum(e_ms)], device=cdev)
        dist.all_reduce(te_max, op=dist.ReduceOp.MAX)
        e2e = {"value": cfg.flops * len(e_ms) / (float(te_max.item()) * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(X_h.numel() * X_h.element_size() + ids_h.numel() * 4) * ws,
               "d2h_bytes_per_step": int(out_h.numel() * out_h.element_size()) * ws}
    # rank 0's exchange traffic per step (rows out / in for dispatch and return, incl. its own share)
    if native is not None:
        lr = native.last_rows()
        x_b = cfg.H * (1 if fp8 else 2)
        y_b = cfg.N * (2 if out_dtype == torch.bfloat16 else 4)
        exch_bytes = {"dispatch_rows_sent": lr["sent"], "dispatch_rows_received": lr["received"],
                      "dispatch_bytes": (lr["sent"] + lr["received"]) * x_b,
                      "combine_rows": lr["local_rows"], "combine_bytes": lr["local_rows"] * y_b}
    else:
        exch_bytes = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(t.item()) / args.steps, "higher_is_better": True,
            "cuda_graph": graph is not None, **({"cuda_graph_error": graph_err} if graph_err else {}),
            "ms_per_step_eager_rank0": statistics.mean(step_ms_eager),
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "fp8_e4m3" if fp8 else "bf16",
            "data": "synthetic",
            "config": {**ep_config(base, ws, args),
                       **({"oversubscribed": f"{ws} ranks on {n_dev} GPU(s): functional run, not a scaling number"}
                          if shared else {}),
                       **({"peer_transport_unavailable": peer_fallback} if peer_fallback else {}),
                       "collectives": ("none: symmetric peer memory (CUDA IPC) — dispatch rows stored into the "
                                       "owners' receive buffers, the GEMM epilogue storing result rows into the "
                                       "token owners' outputs, device-side epoch flags (moe_ep_peer_*)") if peer else
                                      ("NCCL grouped send/recv from the library (moe_ep_forward): counts, "
                                       "dispatch rows, combine rows") if native is not None else
                                      ("NCCL all_to_all_single (torch.distributed): counts, dispatch rows, "
                                       "combine rows")},
            "pct_of_peak": value / (peak * ws),
            "exchange_bytes_per_step_rank0": exch_bytes,
            # exchange rate per GPU against NVLink's ~900 GB/s per direction.  The combine rides in
            # the GEMM's epilogue, so the step's time outside the GEMM bounds the dispatch side: this is its rate
            # over that time (a lower bound; oversubscribed shared-GPU runs say nothing about NVLink)
            "dispatch_gbs_per_gpu_lower_bound": (
                exch_bytes["dispatch_bytes"] / max(float(gathered[0][0]) - float(gathered[0][1]), 1e-6) / 1e6
                if isinstance(exch_bytes, dict) and "dispatch_bytes" in exch_bytes else None),
            "per_rank": [{"ms_per_step": float(g[0]), "gemm_ms": float(g[1]), "gemm_tflops": float(g[2])}
                         for g in gathered],
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "peak_source": f"{peak_src} bf16_tflops (rank 0's GEMM launch"
                                        + ("; moe_ep_forward's events around its GEMM launch)" if native else ")")
                                        + (" x 2 (nominal FP8 / BF16 dense ratio)" if fp8 else ""),
                         "algorithmic_flops_per_launch": flops_l},
            "cpu_baseline": None,
            "e2e": e2e,
            # NCCL / torch paths: dispatch plan 2, gather 1, route (1-3, on the received rows), plan 1, combine
            # map 1, GEMM 1, unpack 1.  Peer path: dispatch plan 2, dispatch 1, route (on the G * T_l receive
            # rows), row pointers 1, GEMM 1, and with > 1 rank two signal + wait pairs (4); the id reset is a
            # memset node.
            "gpu_launches": ((5 + (4 if ws > 1 else 0) + route_launches(ws * T_l, El, cfg.k)) if peer else
                             (7 + route_launches(native.last_rows()["received"] if native is not None
                                                 else sum(moe.last["recv_rows"]), El, cfg.k))) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="mix")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--bn", type=int, default=0)
    ap.add_argument("--bm", type=int, default=0, help="tile rows: 128 (1 CTA), 256 (CTA pair), 0 = planner's choice")
    ap.add_argument("--out-dtype", choices=["bf16", "f32"], default="bf16")
    ap.add_argument("--ep-python", action="store_true",
                    help="expert parallelism orchestrated in Python over torch.distributed all_to_all_single "
                         "(default: the library's moe_ep_forward, NCCL called from C++)")
    ap.add_argument("--ep-transport", choices=["peer", "nccl"], default="peer",
                    help="the library's EP step: symmetric peer memory over CUDA IPC (default) or NCCL send/recv")
    ap.add_argument("--order", choices=list(ORDER_FLAGS), default="natural",
                    help="sigma order of the plan's tasks (P:317-322 expert ordering; DESIGN.md R7)")
    ap.add_argument("--dtype", choices=["bf16", "fp8"], default="bf16",
                    help="operand type of X and W: bf16 (the paper's) or FP8 E4M3 with a per-expert scale")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--host-plan", action="store_true", help="plan on the host (counts D2H) instead of on the device")
    ap.add_argument("--ep", action="store_true", help="run the expert-parallel path even on one GPU")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time eager launches instead of one CUDA graph per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--ffn", action="store_true", help="time the full MoE FFN layer (gate/up SwiGLU + down + combine)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    cfg = synth.CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # `--gpus N` without torchrun: re-launch as N ranks (one process per GPU) and return their exit code
        import socket
        import subprocess
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    ws = dist_env()[0]
    if ws != args.gpus and args.impl == "ours":
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch with --nproc-per-node {args.gpus}")
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.ffn:
        run_ffn(args, cfg)
    elif ws > 1 or args.ep or args.ep_python:
        run_ep(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
