#!/bin/bash
# Run on the GPU box: balanced grid A/B (MOE_BALANCE = 0 / 1) per config, dtype and seed.
OUT=gpurun_out/balance_ab.txt; : > $OUT
for d in bf16 fp8; do for c in dec1 dec16 dec64 dec256 mix ds mix_balanced paper_balanced; do for seed in 0 1; do for b in 0 1; do
  MOE_BALANCE=$b python bench.py --config $c --dtype $d --seed $seed --steps 15 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$d $c seed=$seed balance=$b', round(d['kernel']['ms_per_launch']*1e3,1), round(r['achieved'],1), round(r['frac'],3))" >> $OUT
done; done; done; done
cat $OUT
