import sys, os, ctypes, numpy as np
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_1606_05973_b200 as ccl
img = torch.from_numpy(synth.generate("c4_voronoi_21600")).cuda()
plan = ccl.Plan(*img.shape)
out = torch.empty(img.shape, dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
for _ in range(5): plan.label(img, out, n)
torch.cuda.synchronize()
nTy = (img.shape[0] + 31) // 32
buf = (ctypes.c_ulonglong * (4096 * 6))()
for rep in range(3):
    plan.label(img, out, n); torch.cuda.synchronize()
    assert ccl._L.ccl_debug_k3trace(buf, 4096) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 6)[:nTy].astype(np.int64)
    t0 = a[:, 0].min()
    rel = (a - t0) / 1000.0
    print(f"rep {rep}: kernel span {rel[:,5].max():.1f} us; entry {rel[:,0].min():.1f}-{rel[:,0].max():.1f}; after wait {rel[:,1].min():.1f}-{rel[:,1].max():.1f}")
    d = np.diff(rel[:, 1:], axis=1)
    for i, nm in enumerate(["phase1", "phase2", "lookback", "phase3"]):
        print(f"   {nm:9s} mean {d[:,i].mean():6.2f} max {d[:,i].max():6.2f} us")
    last = np.argsort(rel[:, 5])[-5:]
    for ty in last:
        print("   slowest ty", ty, np.round(rel[ty], 1))
