"""Quick GPU check used during development: parity on a few cases with details."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, synth
import paper_1606_05973_b200 as ccl

def run(img, tag):
    t = torch.from_numpy(img).cuda()
    lab, n = ccl.label(t); torch.cuda.synchronize()
    lg, ng = lab.cpu().numpy(), int(n.item())
    lo, no = oracle.label(img)
    bad = np.argwhere(lg != lo)
    ok = ng == no and len(bad) == 0
    print(f"{tag:40s} {str(img.shape):16s} N gpu={ng} oracle={no} diff={len(bad)} {'OK' if ok else 'FAIL'}", flush=True)
    if not ok and len(bad):
        r, c = bad[0]
        print("  first diff at", (r, c), "gpu", lg[r, max(0,c-3):c+4], "oracle", lo[r, max(0,c-3):c+4])
    return ok

allok = True
for (H, W, p) in [(1,1,1.0),(3,7,0.5),(2,40,0.5),(8,64,0.5),(32,1024,0.5),(33,1025,0.5),(64,2048,0.41),(100,3000,0.7),(1000,1000,0.5),(300,2052,0.95)]:
    allok &= run(synth.bernoulli(H, W, p, 7), f"bern{p}")
for name in synth.CONFIGS:
    img = synth.scaled(name, 600, 2600)
    allok &= run(img, name + "@600x2600")
for name in synth.CONFIGS:
    img = synth.generate(name)
    allok &= run(img, name)
# timing
img = torch.from_numpy(synth.generate("c4_voronoi_21600")).cuda()
plan = ccl.Plan(*img.shape)
out = torch.empty(img.shape, dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
for _ in range(3): plan.label(img, out, n)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): plan.label(img, out, n)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"C4 ms/step {ms:.3f}  Gpx/s {img.numel()/ms/1e6:.1f}  frac(5B/px vs 6549 GB/s) {5*img.numel()/ms/1e9/6549.4*1000:.3f}")
plan.set_profiling(True); plan.label(img, out, n); print(plan.kernel_times())
print("ALL OK" if allok else "SOME FAILED")
