"""Repeat the small-path limit images many times under four configurations
(small middle on/off x 32-warp K1 on/off) and count mismatches."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
import paper_1606_05973_b200 as ccl
ccl._L.ccl_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]
cases = []
for (H, W) in [(1024, 1024), (1024, 1000), (1024, 1), (33, 1), (992, 640)]:
    cases += [synth.comb(H, W), synth.serpentine(H, W), synth.bernoulli(H, W, 0.6, seed=H + W)]
want = [oracle.label(c) for c in cases]
dev = [torch.from_numpy(c).cuda() for c in cases]
for no_small, no_wide in [(0, 0), (1, 0), (0, 1), (1, 1)]:
    ccl._L.ccl_debug_set(3, no_small)
    ccl._L.ccl_debug_set(4, no_wide)
    bad = {}
    for rep in range(30):
        for i, (t, (lo, no)) in enumerate(zip(dev, want)):
            lab, n = ccl.label(t)
            torch.cuda.synchronize()
            if int(n.item()) != no or not np.array_equal(lab.cpu().numpy(), lo):
                bad[i] = bad.get(i, 0) + 1
    print(f"no_small={no_small} no_wide={no_wide}: mismatches per case {bad}", flush=True)
