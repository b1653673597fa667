import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
import paper_1606_05973_b200 as ccl
img = synth.serpentine(1024, 1024)
lo, no = oracle.label(img)
t = torch.from_numpy(img).cuda()
shown = 0
for rep in range(200):
    lab, n = ccl.label(t)
    torch.cuda.synchronize()
    lg = lab.cpu().numpy()
    if int(n.item()) != no or not np.array_equal(lg, lo):
        d = lg != lo
        rows = np.unique(np.nonzero(d)[0])
        print(f"rep {rep}: n {int(n.item())} vs {no}; bad rows {rows[:5]}..{rows[-3:]} ({len(rows)}); tiles {np.unique(rows // 32)}; gpu labels {np.unique(lg[d])[:8]} oracle {np.unique(lo[d])[:8]}", flush=True)
        shown += 1
        if shown > 6: break
print("done")
