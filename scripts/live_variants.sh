# live-cache DRAM traffic of K1/K5 for experiment builds (see live_traffic.sh)
for v in "$@"; do
  CCL_B200_LIB=libccl_$v.so bash scripts/live_traffic.sh v_$v > /dev/null 2>&1
  echo "== $v"; python scripts/live_summary.py gpurun_out/live_v_$v.csv | grep -E "k_tile|k_write"
done
