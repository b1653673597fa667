"""Development timing of K1's phases: K1 truncated after phase `stop` (the
rest of the pipeline is skipped), CUDA events per kernel.  Needs the knob
build:  CCL_VARIANT=knob CCL_DEFS=-DCCL_PHASE_KNOB=1 python build_native.py product
and  CCL_B200_LIB=libccl_knob.so python scripts/k1_phases.py"""
import sys, os, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch, synth
import paper_1606_05973_b200 as ccl
ccl._L.ccl_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]
names = sys.argv[1:] or ["c4_voronoi_21600"]
for name in names:
    if name not in synth.CONFIGS: print("configs:", list(synth.CONFIGS)); continue
    img = torch.from_numpy(synth.generate(name)).cuda()
    plan = ccl.Plan(*img.shape)
    out = torch.empty(img.shape, dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
    prev = 0.0
    for stop in [-1, 0, 1, 2, 3, 4, 5, 6, 99]:
        ccl._L.ccl_debug_set(1, stop)
        plan.set_profiling(20)
        for _ in range(23): plan.label(img, out, n)
        t = plan.kernel_times()
        k1 = t['k_tile_local'] * 1000
        print(f"{name} stop={stop:2d} k_tile_local {k1:8.1f} us  (+{k1 - prev:6.1f})  total {sum(t.values())*1000:8.1f} us", flush=True)
        prev = k1
    ccl._L.ccl_debug_set(1, 99)
    for ex in [1, 0]:
        ccl._L.ccl_debug_set(2, ex)
        plan.set_profiling(20)
        for _ in range(23): plan.label(img, out, n)
        t = plan.kernel_times()
        print(f"{name} exper={ex} " + "  ".join(f"{k} {v*1000:.1f}" for k, v in t.items()) + f"  total {sum(t.values())*1000:.1f} us", flush=True)
    ccl._L.ccl_debug_set(2, 0)
