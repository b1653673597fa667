import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import numpy as np, torch, oracle, synth
import paper_1606_05973_b200 as ccl, ctypes
ccl._L.ccl_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]

name = sys.argv[1] if len(sys.argv) > 1 else "c3_percolation_8192"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
img = synth.generate(name)
lo, no = oracle.label(img)
t = torch.from_numpy(img).cuda()
plan = ccl.Plan(*img.shape)
bad = 0
for i in range(reps):
    lab, n = plan.label(t); torch.cuda.synchronize()
    lg = lab.cpu().numpy(); ng = int(n.item())
    d = np.argwhere(lg != lo)
    if ng != no or len(d):
        bad += 1
        print(f"rep {i}: N {ng} vs {no}, {len(d)} px differ, first {d[0] if len(d) else None}", flush=True)
        if len(d):
            r, c = d[0]; print("  gpu", lg[r, max(0,c-4):c+5], "\n  ora", lo[r, max(0,c-4):c+5])
print(f"{name} exper={sys.argv[3] if len(sys.argv) > 3 else 0}: {bad}/{reps} bad")
