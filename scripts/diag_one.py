import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle, paper_1606_05973_b200 as ccl
H, W, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
img = synth.scaled("c3_percolation_8192", H, W)
plan = ccl.Plan(H, W)
d = torch.from_numpy(img).cuda()
out = torch.empty((H, W), dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
for it in range(reps):
    plan.label(d, out, n)
    torch.cuda.synchronize()
lo, no = oracle.label(img)
print(H, W, reps, "ok" if (int(n.cpu()) == no and np.array_equal(out.cpu().numpy(), lo)) else "MISMATCH", flush=True)
