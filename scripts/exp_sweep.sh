#!/bin/bash
# Run on the GPU box: timing-study build (MOE_EXPERIMENTS, wrong Y) — which data movement bounds the kernel.
OUT=gpurun_out/exp_sweep_${1:-a}.txt; : > $OUT
for d in ${DTYPES:-fp8 bf16}; do for c in ${CONFIGS:-mix}; do for x in 0 8 1 2 3 11; do
  MOE_LIB=build_ab/exp/libmoe_sm100.so MOE_GEMM_EXPERIMENT=$x python bench.py --dtype $d --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d $c exp=$x', round(d['kernel']['tflops'],1), d['clocks']['sm_mhz'])" >> $OUT
done; done; done
cat $OUT
