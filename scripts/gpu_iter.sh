#!/bin/bash
# One GPU iteration: parity tests, bench line (no CPU baseline), K1 ncu capture.
# usage: scripts/gpu_iter.sh TAG [notests] [noncu]
TAG=${1:-dev}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ "$2" != "notests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
fi
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
if [ "$3" != "noncu" ]; then
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-small"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tile_local' --launch-skip 3 --launch-count 1 -o gpurun_out/prof_k1_$TAG -f $BENCH > gpurun_out/ncu_k1_$TAG.log 2>&1
fi
echo done
