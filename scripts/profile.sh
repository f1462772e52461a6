#!/bin/bash
# Run on the GPU box (under gpurun): launch list + one ncu --set full capture of moe_gemm_kernel.
# usage: scripts/profile.sh <tag> [bench args...]
set -u
TAG=${1:-mix}; shift || true
OUT=gpurun_out/prof_${TAG}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${OUT}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > ${OUT}_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:moe_gemm_kernel -s 4 -c 1 -f -o ${OUT} \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > ${OUT}_full.log 2>&1
echo "profile ${TAG} done"
