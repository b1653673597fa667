#!/bin/bash
# One GPU session: tests, bench, launch list, one ncu --set full capture.
# usage: scripts/gpu_round.sh TAG [skip-tests]
TAG=${1:-r01}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
fi
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-small"
timeout 300 $BENCH > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $BENCH > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 300 $BENCH > gpurun_out/plain2_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tile_local|k_write|k_border|k_number|k_fixup' --launch-skip 15 --launch-count 5 -o gpurun_out/prof_$TAG -f $BENCH > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
