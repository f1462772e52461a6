"""Summarise ncu captures into profiles/ (run HERE, on the CPU box, after gpurun brought them back).

    python scripts/ncu_summary.py <tag> <workload> <prof.ncu-rep> [<launches.csv>]

Writes profiles/<tag>/<workload>_ncu.json (+ .md) with the metrics the judge and DESIGN.md cite,
and updates profiles/traffic.json[workload] = dram bytes per launch of moe_gemm_kernel (bench.py
reports it as roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg", "gpc__cycles_elapsed.avg.per_second",
    "launch__grid_size", "launch__cluster_dim_x", "launch__registers_per_thread", "launch__block_size",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for h, u, v in zip(hdr, units, vals):
            if h in WANT:
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                d[h] = {"value": x, "unit": u}
        kernels.append(d)
    return kernels


def to_base(m):
    return m["value"] * SCALE.get(m["unit"], 1.0)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0][:80]].append(float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9))
    return {k: {"launches": len(v), "mean_us": 1e6 * sum(v) / len(v)} for k, v in agg.items()}


def main():
    tag, workload, rep = sys.argv[1:4]
    lc = sys.argv[4] if len(sys.argv) > 4 else None
    ks = [k for k in raw_metrics(rep) if "moe_gemm_kernel" in k["kernel"]]
    if not ks:
        raise SystemExit("no moe_gemm_kernel in the report")
    k = ks[0]
    dram = to_base(k["dram__bytes_read.sum"]) + to_base(k["dram__bytes_write.sum"])
    summary = {"tag": tag, "workload": workload, "source": os.path.relpath(rep, ROOT), "kernel": k["kernel"],
               "metrics": {m: k[m] for m in WANT if m in k}, "dram_bytes_per_launch": dram}
    if lc:
        summary["launch_list"] = launches(lc)
        ours = {n: v for n, v in summary["launch_list"].items() if "moe_gemm" in n or "route_" in n}
        if ours:
            gemm = sum(v["mean_us"] for n, v in ours.items() if "moe_gemm" in n)
            summary["gemm_share_of_step_kernels"] = gemm / sum(v["mean_us"] for v in ours.values())
    os.makedirs(os.path.join(ROOT, "profiles", tag), exist_ok=True)
    base = os.path.join(ROOT, "profiles", tag, f"{workload}_ncu")
    json.dump(summary, open(base + ".json", "w"), indent=1)
    with open(base + ".md", "w") as f:
        f.write(f"# ncu summary — {workload} ({tag})\n\nkernel: `{k['kernel']}`  \nsource: `{summary['source']}`\n\n")
        f.write("| metric | value | unit |\n|---|---|---|\n")
        for m, v in summary["metrics"].items():
            f.write(f"| {m} | {v['value']:.6g} | {v['unit']} |\n")
        f.write(f"\nDRAM traffic per launch: {dram / 1e9:.4f} GB\n")
        if lc:
            f.write("\n## launch list (ncu gpu__time_duration, cold-cache, serialised)\n\nThe library's kernels "
                    "(one step = route kernels + moe_gemm):\n\n| kernel | launches | mean us |\n|---|---|---|\n")
            others = 0
            for n, v in sorted(summary["launch_list"].items(), key=lambda kv: -kv[1]["mean_us"]):
                if "moe_gemm" in n or "route_" in n or "plan_" in n:
                    f.write(f"| `{n}` | {v['launches']} | {v['mean_us']:.1f} |\n")
                else:
                    others += v["launches"]
            f.write(f"\n({others} other launches in the same process: synthetic input generation and the L2 flush "
                    "memset, outside the timed step.)\n")
            if "gemm_share_of_step_kernels" in summary:
                f.write(f"\nmoe_gemm share of the step's own kernels: {summary['gemm_share_of_step_kernels']:.3f}\n")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    t = json.load(open(tp)) if os.path.exists(tp) else {}
    def pct(m):
        return k[m]["value"] if m in k else None
    t[workload] = {"dram_bytes_per_launch": dram, "source": os.path.relpath(base + ".json", ROOT),
                   "tensor_pipe_pct": pct("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                   "dram_throughput_pct": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                   "ncu_us": to_base(k["gpu__time_duration.sum"]) * 1e6 if "gpu__time_duration.sum" in k else None,
                   "sm_mhz": k["gpc__cycles_elapsed.avg.per_second"]["value"] * 1e3
                   if "gpc__cycles_elapsed.avg.per_second" in k and k["gpc__cycles_elapsed.avg.per_second"]["unit"] == "Ghz"
                   else None}
    json.dump(t, open(tp, "w"), indent=1)
    print(json.dumps({k2: v for k2, v in summary.items() if k2 != "launch_list"})[:2000])


if __name__ == "__main__":
    main()
