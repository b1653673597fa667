#!/bin/bash
# ncu --set full of selected kernels on the bench command (after a clean run)
TAG=$1; KRE=${2:-"k_tile_local|k_write|k_border|k_number|k_fixup"}; SKIP=${3:-15}; CNT=${4:-5}
cd "$(dirname "$0")/.."
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-small"
timeout 300 $BENCH > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" --launch-skip $SKIP --launch-count $CNT -o gpurun_out/prof_$TAG -f $BENCH > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
