"""Repeat the full C3 labeling many times; on a mismatch, describe it: count,
differing pixels, their tiles, and whether ground-truth components were split
(a lost union) or merged (a spurious one)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
import paper_1606_05973_b200 as ccl

name = sys.argv[1] if len(sys.argv) > 1 else "c3_percolation_8192"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 400
img = synth.generate(name)
lo, no = oracle.label(img)
ref = torch.from_numpy(lo).cuda()
t = torch.from_numpy(img).cuda()
plan = ccl.Plan(*img.shape)
out = torch.empty_like(ref)
n = torch.empty(1, dtype=torch.int32, device="cuda")
bad = 0
for i in range(reps):
    plan.label(t, out, n)
    torch.cuda.synchronize()
    nn = int(n.item())
    if nn == no and torch.equal(out, ref):
        continue
    bad += 1
    if bad > 4:
        continue
    o = out.cpu().numpy()
    d = np.argwhere(o != lo)
    tiles = sorted({(int(r) // 32, int(c) // 1024) for r, c in d})
    gt = np.unique(lo[o != lo])
    got = np.unique(o[o != lo])
    print(f"run {i}: n {nn} vs {no}, {len(d)} px differ, tiles {tiles[:8]}{'...' if len(tiles) > 8 else ''}, "
          f"gt comps {len(gt)}, gpu labels {len(got)}, first px {tuple(d[0])} gpu {o[tuple(d[0])]} gt {lo[tuple(d[0])]}",
          flush=True)
print(f"{name}: {bad} of {reps} runs differ", flush=True)
