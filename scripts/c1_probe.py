"""C1 (512x512 Bernoulli 0.5) single calls through one plan, for an ncu
capture of the small-image path (k_tile_local_wide, k_small_middle, k_write)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_05973_b200 as ccl  # noqa: E402
import synth  # noqa: E402
img = torch.from_numpy(synth.generate("c1_bernoulli_512")).cuda()
plan = ccl.Plan(*img.shape)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    plan.label(img)
torch.cuda.synchronize()
print("ok")
