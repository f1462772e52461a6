#!/bin/bash
# Run on the GPU box: kernel TFLOP/s per task order per config and dtype, same box.
OUT=gpurun_out/order_sweep_${TAG:-a}.txt; : > $OUT
for r in 1 2; do for d in ${DTYPES:-bf16 fp8}; do for c in ${CONFIGS:-ds mix paper_worst}; do for o in natural alternating half_interval; do
  python bench.py --config $c --dtype $d --order $o --steps 15 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d $c $o', round(d['kernel']['tflops'],1), round(d['value'],1))" >> $OUT
done; done; done; done
cat $OUT
