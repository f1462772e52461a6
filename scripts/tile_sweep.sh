#!/bin/bash
# Run on the GPU box: kernel TFLOP/s per tile shape, config and operand type (same box).
OUT=gpurun_out/tile_sweep_${TAG:-a}.txt; : > $OUT
for d in ${DTYPES:-fp8 bf16}; do for c in ${CONFIGS:-ds paper_balanced mix}; do for t in ${TILES:-"256 512" "256 256" "128 256"}; do
  set -- $t
  python bench.py --config $c --dtype $d --bm $1 --bn $2 --steps 15 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d $c $1x$2', round(d['kernel']['tflops'],1), round(d['value'],1))" >> $OUT
done; done; done
cat $OUT
