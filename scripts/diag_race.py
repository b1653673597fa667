import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle, paper_1606_05973_b200 as ccl
H, W, reps, sync = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
img = synth.scaled("c3_percolation_8192", H, W)
lo, no = oracle.label(img)
plan = ccl.Plan(H, W)
d = torch.from_numpy(img).cuda()
out = torch.empty((H, W), dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
bad = 0
for it in range(reps):
    plan.label(d, out, n)
    if sync or it == reps - 1:
        ok = int(n.cpu()) == no and np.array_equal(out.cpu().numpy(), lo)
        bad += not ok
dbg = (ctypes.c_int * 16)()
ccl._L.ccl_debug_wait(dbg)
print(H, W, reps, "sync", sync, "bad", bad, "waitdbg", list(dbg), flush=True)
