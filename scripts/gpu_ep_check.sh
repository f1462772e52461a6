#!/bin/bash
# GPU box: peer-memory EP tests + bench lines of the EP step (world 1 and shared-GPU multi-rank).
TAG=${1:-ep}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ep_peer.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_peer_tests.log 2>&1; echo "peer tests rc=$?"; tail -15 gpurun_out/${TAG}_peer_tests.log
timeout 300 python bench.py --ep --config mix --no-cpu-baseline --steps 10 > gpurun_out/${TAG}_bench_ep1.json 2> gpurun_out/${TAG}_bench_ep1.err; echo "ep1 rc=$?"; tail -c 1500 gpurun_out/${TAG}_bench_ep1.json; tail -5 gpurun_out/${TAG}_bench_ep1.err
timeout 600 python bench.py --gpus 2 --config mix --no-cpu-baseline --steps 5 --no-e2e > gpurun_out/${TAG}_bench_ep2shared.json 2> gpurun_out/${TAG}_bench_ep2shared.err; echo "ep2 shared rc=$?"; tail -c 1500 gpurun_out/${TAG}_bench_ep2shared.json; tail -5 gpurun_out/${TAG}_bench_ep2shared.err
