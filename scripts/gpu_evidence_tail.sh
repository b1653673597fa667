cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c3_full bernoulli06_2048x8192 handed_over_dense c1_batch64; do
  timeout 900 python scripts/race_hunt.py $c 2000 >> gpurun_out/ev_race_r02z.log 2>&1
done
timeout 900 python scripts/kernel_times.py > gpurun_out/ev_kt_r02z.log 2>&1
timeout 900 python scripts/kernel_times.py c1_bernoulli_512:64 c2_blobs_1024:64 > gpurun_out/ev_kt_small_r02z.log 2>&1
timeout 900 python scripts/scale_projection.py > gpurun_out/ev_scale_r02z.log 2>&1
timeout 400 python scripts/fuzz.py 300 777 > gpurun_out/ev_fuzz_r02z.log 2>&1
FUZZ_POISON=9191 timeout 400 python scripts/fuzz.py 300 778 > gpurun_out/ev_fuzz_poison_r02z.log 2>&1
echo done
