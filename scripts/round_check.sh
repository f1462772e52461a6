#!/bin/bash
# GPU box, one call: smoke, every GPU test (parity margins logged), bench lines for every config, the
# reference arm, and ncu launch lists + --set full captures of moe_gemm_kernel.  Results in gpurun_out/<tag>_*.
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
MOE_PARITY_LOG=$O/parity_margins.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -3 $O/gpu_tests.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
for c in ds dec1 dec16 dec64 dec256 paper_worst paper_balanced paper_best mix_balanced ep; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
for c in mix ds dec1 dec16; do
  timeout 400 python bench.py --config $c --dtype fp8 --no-cpu-baseline > $O/bench_fp8_$c.json 2> $O/bench_fp8_$c.err; echo "fp8 $c rc=$?"
done
timeout 400 python bench.py --ffn --config mix --no-cpu-baseline > $O/bench_ffn_mix.json 2> $O/bench_ffn_mix.err
timeout 400 python bench.py --ffn --config ds --no-cpu-baseline > $O/bench_ffn_ds.json 2> $O/bench_ffn_ds.err
timeout 400 python bench.py --ep --config mix --no-cpu-baseline > $O/bench_ep1_mix.json 2> $O/bench_ep1_mix.err; echo "ep1 rc=$?"
timeout 400 python bench.py --ep --config ep --no-cpu-baseline --no-e2e > $O/bench_ep1_8x22b.json 2> $O/bench_ep1_8x22b.err; echo "ep1 8x22b rc=$?"
timeout 400 python bench.py --ep --ep-transport nccl --config mix --no-cpu-baseline --no-e2e > $O/bench_ep1_mix_nccl.json 2> $O/bench_ep1_mix_nccl.err
timeout 600 python bench.py --gpus 2 --config mix --no-cpu-baseline --no-e2e --steps 5 > $O/bench_ep2_shared.json 2> $O/bench_ep2_shared.err; echo "ep2 shared rc=$?"
for c in mix ds dec1 paper_worst; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${c}_launches.csv \
      python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_gemm_kernel -s 4 -c 1 -f -o $O/${c}_gemm_full \
      python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "ncu $c rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_gemm_kernel -s 4 -c 1 -f -o $O/fp8_mix_gemm_full \
    python bench.py --config mix --dtype fp8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "all done"
