for v in "$@"; do
CCL_B200_LIB=libccl_$v.so python - <<'PY'
import os, torch, synth, paper_1606_05973_b200 as ccl
v = os.environ["CCL_B200_LIB"]
for name in ["c1_bernoulli_512", "c2_blobs_1024"]:
    img = torch.from_numpy(synth.generate(name)).cuda()
    H, W = img.shape
    p = ccl.Plan(H, W); o = torch.empty((H, W), dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
    for _ in range(20): p.label(img, o, n)
    torch.cuda.synchronize()
    # single call latency: one call, synchronize, repeat
    import time
    ts = []
    for _ in range(200):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); p.label(img, o, n); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1000)
    ts.sort()
    print(v, name, "single median %.1f us  p10 %.1f" % (ts[len(ts)//2], ts[len(ts)//10]), flush=True)
PY
done
