#!/bin/bash
# Same-box A/B of moe_gemm builds: scripts/ab_run.sh "<cfg list>" "<lib names in build_ab or 'new'>" "<flags list>"
for c in $1; do for L in $2; do for f in $3; do
  if [ "$L" = new ]; then unset MOE_LIB; else export MOE_LIB=build_ab/$L/libmoe_sm100.so; fi
  timeout 60 python scripts/gemm_breakdown.py $c 256 256 $f | python -c "import json,sys;d=json.load(sys.stdin);print('$L', d['config'], 'flags', d['flags'], 'TF', round(d['tflops_plain']), 'wait_full', round(d['mma_wait_full_frac'],3), 'wait_tmem', round(d['mma_wait_tmem_frac'],3), 'cyc/tile', round(d['mma_cycles_per_tile']), 'epi', round(d['epi_work_per_tile_cycles']))"
done; done; done
