# Times experiment builds of the product library side by side (one GPU):
#   CCL_VARIANT=name CCL_DEFS="-D..." python build_native.py product   (here)
#   bash scripts/variants.sh b200 name ...                             (on the box)
mkdir -p gpurun_out
for v in "$@"; do
  CCL_B200_LIB=libccl_$v.so python bench.py --no-small --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']
print('$v', round(d['ms_per_step']*1e3,1), {k: round(e['ms']*1e3,1) for k,e in r['kernels'].items()})"
done
