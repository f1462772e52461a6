#!/bin/bash
# Timing study: the wide kernel with the MMA never waiting for the epilogue (experiment 64, wrong Y).
OUT=gpurun_out/exp_tmem.txt; : > $OUT
for d in bf16 fp8; do for c in mix ds mix_balanced; do for x in 0 64; do
  MOE_LIB=build_ab/exp/libmoe_sm100.so MOE_GEMM_EXPERIMENT=$x python bench.py --dtype $d --config $c --steps 15 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d $c exp=$x', round(d['kernel']['tflops'],1))" >> $OUT
done; done; done
cat $OUT
