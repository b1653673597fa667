"""Development probe: C4 through ccl_label_banded (all bands on one GPU, one
after another) vs one plan call -- the cost of the band protocol itself."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1606_05973_b200 as ccl
img = torch.from_numpy(synth.generate("c4_voronoi_21600")).cuda()
H, W = img.shape
out = torch.empty((H, W), dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
plan = ccl.Plan(H, W)
print(f"plan: {t(lambda: plan.label(img, out, n)):.3f} ms")
for nb in [1, 2, 4, 8]:
    print(f"banded nb={nb}: {t(lambda: ccl.label_banded(img, nb, out, n)):.3f} ms (incl. workspace alloc per call)", flush=True)
