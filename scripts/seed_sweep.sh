#!/bin/bash
# Run on the GPU box: kernel / step TFLOP/s over routing seeds {0, 1, 2} (report the median).
OUT=gpurun_out/seed_sweep_${TAG:-a}.txt; : > $OUT
for d in bf16 fp8; do for c in mix ds mix_balanced dec16 paper_balanced; do for seed in 0 1 2; do
  python bench.py --config $c --dtype $d --seed $seed --steps 15 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$d $c seed=$seed', round(d['kernel']['tflops'],1), round(d['value'],1), r['bound'], round(r['frac'],3))" >> $OUT
done; done; done
cat $OUT
