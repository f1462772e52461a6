#!/bin/bash
# Run on the GPU box: kernel TFLOP/s of the wide pair tile over tile widths (same box, same process order).
mkdir -p gpurun_out
OUT=gpurun_out/bn_sweep_${1:-a}.txt
: > $OUT
for c in ${CONFIGS:-mix mix_balanced ds paper_balanced ep}; do
  for bn in ${BNS:-512 480 448 416 384 352 320}; do
    python bench.py --config $c --bm 256 --bn $bn --steps 15 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', $bn, round(d['kernel']['tflops'],1), round(d['value'],1), d['clocks']['sm_mhz'])" >> $OUT
  done
done
cat $OUT
