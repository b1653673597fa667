"""A handful of small labelings through every code path (small-image path,
32-warp K1 + normal middle, 8-warp K1 with hand-over, batch, threshold, row
bands), each checked against the oracle (a quick all-paths check; compute-sanitizer is closed on this pool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
import paper_1606_05973_b200 as ccl

def check(img, lab, n, tag):
    lo, no = oracle.label(img)
    ok = int(n) == no and np.array_equal(lab, lo)
    print(tag, img.shape, "ok" if ok else "MISMATCH", flush=True)
    return ok

allok = True
for (H, W, p) in [(300, 500, 0.5), (700, 1024, 0.41), (130, 3000, 0.6), (2048, 8192, 0.45)]:
    img = synth.bernoulli(H, W, p, seed=H + W)
    if H == 130:
        img[5::7] = 0
        img[5::7, ::2] = 1
    lab, n = ccl.label(torch.from_numpy(img).cuda())
    torch.cuda.synchronize()
    allok &= check(img, lab.cpu().numpy(), n.item(), "single")
imgs = np.stack([synth.bernoulli(200, 300, 0.5, seed=s) for s in range(5)])
lab, n = ccl.label_batch(torch.from_numpy(imgs).cuda())
torch.cuda.synchronize()
for b in range(5):
    allok &= check(imgs[b], lab[b].cpu().numpy(), n[b].item(), "batch")
gray = np.random.default_rng(1).integers(0, 256, (400, 1100), dtype=np.uint8)
lab, n = ccl.label(torch.from_numpy(gray).cuda(), threshold=127)
torch.cuda.synchronize()
allok &= check((gray > 127).astype(np.uint8), lab.cpu().numpy(), n.item(), "threshold")
img = synth.scaled("c4_voronoi_21600", 400, 2100)
lab, n = ccl.label_banded(torch.from_numpy(img).cuda(), 3)
torch.cuda.synchronize()
allok &= check(img, lab.cpu().numpy(), n.item(), "banded")
print("ALL OK" if allok else "FAILED")
