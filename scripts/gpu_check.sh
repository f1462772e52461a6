#!/bin/bash
# Run on the GPU box: GPU tests + smoke + bench lines for the main configs.
# usage: scripts/gpu_check.sh <tag> [configs...]
TAG=${1:-chk}; shift || true
CFGS=${@:-mix ds paper_worst paper_balanced mix_balanced dec1 dec16 dec256}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/${TAG}_gputests.log
for c in $CFGS; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_${c}.json 2> gpurun_out/${TAG}_bench_${c}.err
  python - gpurun_out/${TAG}_bench_${c}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d.get("roofline", {}); k = d.get("kernel", {})
    print(sys.argv[1].split("/")[-1], "step", round(d["value"], 1), "kernel_ms", k.get("ms_per_launch"), r.get("bound"), round(r.get("achieved", 0), 1), "frac", round(r.get("frac", 0), 3), d.get("config", {}).get("tile"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
