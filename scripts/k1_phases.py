import sys, os, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch, synth
import paper_1606_05973_b200 as ccl
ccl._L.ccl_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]
name = sys.argv[1] if len(sys.argv) > 1 else "c4_voronoi_21600"
img = torch.from_numpy(synth.generate(name)).cuda()
plan = ccl.Plan(*img.shape)
out = torch.empty(img.shape, dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
for stop, ex in [(1, 0), (2, 0), (99, 0)]:
    ccl._L.ccl_debug_set(1, stop); ccl._L.ccl_debug_set(2, ex)
    plan.set_profiling(20)
    for _ in range(23): plan.label(img, out, n)
    t = plan.kernel_times()
    print(f"{name} stop={stop:2d} k_tile_local {t['k_tile_local']*1000:8.1f} us  total {sum(t.values())*1000:8.1f} us")
ccl._L.ccl_debug_set(1, 99); ccl._L.ccl_debug_set(2, 0)
