#!/bin/bash
# Run on the GPU box: bench.py lines for every config into gpurun_out/bench_<tag>_<cfg>.json
TAG=${1:-s}
mkdir -p gpurun_out
for c in mix ds dec1 dec16 dec64 dec256 mix_balanced paper_balanced; do
  extra=""; [ "$c" != mix ] && [ "$c" != ds ] && extra="--no-cpu-baseline"
  python bench.py --config $c $extra > gpurun_out/bench_${TAG}_${c}.json 2> gpurun_out/bench_${TAG}_${c}.err
done
python bench.py --ffn --config mix > gpurun_out/bench_${TAG}_ffn_mix.json 2> gpurun_out/bench_${TAG}_ffn_mix.err
python bench.py --host-plan --config mix --no-cpu-baseline > gpurun_out/bench_${TAG}_mix_hostplan.json 2> gpurun_out/bench_${TAG}_mix_hostplan.err
for f in gpurun_out/bench_${TAG}_*.json; do
  python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d.get("roofline", {})
    print(sys.argv[1].split("/")[-1], round(d["value"], 1), d.get("ms_per_step"), r.get("bound"), round(r.get("achieved", 0), 1), round(r.get("frac", 0), 3))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
