#!/bin/bash
# Run on the GPU box: FP8 bench lines (+ bf16 Mix for a same-box reference) and the FP8 Mix ncu capture.
TAG=${1:-f}
mkdir -p gpurun_out
for c in mix ds mix_balanced dec1 dec16 dec256 paper_balanced; do
  extra="--no-cpu-baseline"; [ "$c" = mix ] && extra=""
  python bench.py --dtype fp8 --config $c $extra > gpurun_out/bench_${TAG}_fp8_${c}.json 2> gpurun_out/bench_${TAG}_fp8_${c}.err
  tail -1 gpurun_out/bench_${TAG}_fp8_${c}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', round(d['value'],1), round(d['kernel']['tflops'],1), r['bound'], round(r['achieved'],1), round(r['frac'],3), d['kernel']['ms_per_launch'])" || tail -5 gpurun_out/bench_${TAG}_fp8_${c}.err
done
python bench.py --config mix --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_bf16_mix.json 2>&1
tail -1 gpurun_out/bench_${TAG}_bf16_mix.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bf16 mix', round(d['value'],1), round(d['kernel']['tflops'],1))"
if [ "${PROFILE:-1}" = 1 ]; then bash scripts/profile.sh fp8_mix --dtype fp8 --config mix; fi
