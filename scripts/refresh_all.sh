#!/bin/bash
# Run on the GPU box: the round's full measurement refresh (tests, smoke, bench lines bf16 + FP8, FFN,
# paper Table 1, comparators, ncu of the Mix / DS / dec1 kernels).
TAG=${1:-fin}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; tail -2 gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
bash scripts/bench_all.sh ${TAG}
PROFILE=0 bash scripts/bench_fp8.sh ${TAG}
python bench.py --ffn --config ds > gpurun_out/bench_${TAG}_ffn_ds.json 2>&1
python scripts/paper_table1.py --out gpurun_out/${TAG}_paper_table1.json > gpurun_out/${TAG}_paper_table1.log 2>&1
python scripts/comparators.py > gpurun_out/${TAG}_comparators.jsonl 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_reference.json 2>&1
echo refresh done
python bench.py --ep --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_ep_native_mix.json 2>&1
python bench.py --ep --dtype fp8 --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_ep_native_mix_fp8.json 2>&1
python bench.py --ep --config ep --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_${TAG}_ep_native_8x22b.json 2>&1
echo refresh ep done
