#!/bin/bash
# Run on the GPU box: same-box A/B of library builds through bench.py (kernel TFLOP/s, step TFLOP/s).
#   scripts/ab_bench.sh "<lib names in build_ab, or new>" "<configs>" "<dtypes>" [rounds]
OUT=gpurun_out/ab_bench_${TAG:-a}.txt; : > $OUT
for r in $(seq 1 ${4:-1}); do for d in $3; do for c in $2; do for L in $1; do
  if [ "$L" = new ]; then unset MOE_LIB; else export MOE_LIB=build_ab/$L/libmoe_sm100.so; fi
  timeout 120 python bench.py --dtype $d --config $c --steps 15 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L $d $c', round(d['kernel']['tflops'],1), round(d['value'],1), round(d['roofline']['frac'],3))" >> $OUT
done; done; done; done
cat $OUT
