# DRAM traffic of each kernel with the caches as the pipeline leaves them
# (ncu --cache-control none; few metrics, one pass).  usage: live_traffic.sh TAG [bench args]
TAG=$1; shift
cd "$(dirname "$0")/.."
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-small $*"
timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  -k regex:'k_' --launch-skip 18 --launch-count 12 --csv --log-file gpurun_out/live_$TAG.csv $BENCH > gpurun_out/live_$TAG.log 2>&1
echo rc=$?
