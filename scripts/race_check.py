import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle, paper_1606_05973_b200 as ccl
for (H, W) in [(1500, 4100), (1500, 4096), (2048, 2048)]:
    img = synth.scaled("c3_percolation_8192", H, W)
    lo, no = oracle.label(img)
    plan = ccl.Plan(H, W)
    d = torch.from_numpy(img).cuda()
    out = torch.empty((H, W), dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
    bad = 0; badn = 0
    for it in range(200):
        plan.label(d, out, n)
        if it % 10 == 0 or it < 5:
            o = out.cpu().numpy(); nn = int(n.cpu())
            if nn != no: badn += 1
            if not np.array_equal(o, lo):
                bad += 1
                diff = np.argwhere(o != lo)
                if bad <= 2: print(H, W, "it", it, "n", nn, no, "ndiff", len(diff), diff[:3], o[tuple(diff[0])], lo[tuple(diff[0])])
    print(H, W, "bad", bad, "badn", badn, flush=True)
