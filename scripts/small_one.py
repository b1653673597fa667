"""One image per call, a few calls (for ncu): python scripts/small_one.py [name] [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1606_05973_b200 as ccl
name = sys.argv[1] if len(sys.argv) > 1 else "c1_bernoulli_512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
img = torch.from_numpy(synth.generate(name)).cuda()
plan = ccl.Plan(*img.shape)
out = torch.empty(img.shape, dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
for _ in range(reps):
    plan.label(img, out, n)
torch.cuda.synchronize()
print("ok", int(n.item()))
