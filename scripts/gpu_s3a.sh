cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_check.sh s3a
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-small"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tile_local' --launch-skip 3 --launch-count 1 -o gpurun_out/prof_k1_s3a -f $BENCH > gpurun_out/ncu_k1_s3a.log 2>&1
echo done
