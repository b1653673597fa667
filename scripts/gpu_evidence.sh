#!/bin/bash
# Round-end evidence on one GPU: full GPU tests, race hunts of every dense
# path, launch list, ncu --set full of the five C4 kernels, per-config kernel
# times, the band-path scale projection.  usage: scripts/gpu_evidence.sh TAG
TAG=${1:-r02}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_$TAG.log
for c in c3_full bernoulli06_2048x8192 handed_over_dense c1_batch64; do
  timeout 900 python scripts/race_hunt.py $c 2000 >> gpurun_out/ev_race_$TAG.log 2>&1
done
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-small"
timeout 300 $BENCH > gpurun_out/ev_plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_$TAG.csv $BENCH > gpurun_out/ev_ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tile_local|k_write|k_border|k_number|k_fixup' --launch-skip 15 --launch-count 5 -o gpurun_out/ev_prof_$TAG -f $BENCH > gpurun_out/ev_ncu_full_$TAG.log 2>&1
timeout 900 python scripts/kernel_times.py > gpurun_out/ev_kt_$TAG.log 2>&1
timeout 900 python scripts/kernel_times.py c1_bernoulli_512:64 c2_blobs_1024:64 >> gpurun_out/ev_kt_$TAG.log 2>&1
timeout 900 python scripts/scale_projection.py > gpurun_out/ev_scale_$TAG.log 2>&1
echo done
