"""Per-kernel times on C3 (dense near-percolation noise): how much the K1
hand-over pass takes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1606_05973_b200 as ccl
for name in sys.argv[1:] or ["c3_percolation_8192"]:
    img = torch.from_numpy(synth.generate(name)).cuda()
    plan = ccl.Plan(*img.shape)
    out = torch.empty(img.shape, dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
    for _ in range(3): plan.label(img, out, n)
    plan.set_profiling(10)
    for _ in range(10): plan.label(img, out, n)
    torch.cuda.synchronize()
    print(name, {k: round(v * 1e3, 1) for k, v in plan.kernel_times().items()}, flush=True)
