#!/bin/bash
# ncu --set full (with source) of one launch of the named kernel(s) in the bench command
# usage: scripts/gpu_prof_k.sh TAG REGEX [SKIP]
TAG=$1; KRE=$2; SKIP=${3:-3}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-small"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$KRE" --launch-skip $SKIP --launch-count 1 -o gpurun_out/prof_${TAG} -f $BENCH > gpurun_out/ncu_${TAG}.log 2>&1
echo done
