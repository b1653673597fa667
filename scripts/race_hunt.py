"""Repeat one labeling case many times (the race stress cases of
tests/test_gpu_races.py, or a synth recipe name) and report every run that is
not bit-exact with the oracle, plus the plan's path counters (which K1 code
paths ran).  usage: python scripts/race_hunt.py CASE [REPS]
CASE: c3_full | bernoulli06_2048x8192 | handed_over_dense | c1_batch64 | <synth name>"""
import sys, os, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, synth, oracle
import paper_1606_05973_b200 as ccl
from test_gpu_races import _handed_over_dense

case = sys.argv[1] if len(sys.argv) > 1 else "c3_full"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 400
batch = None
if case == "c3_full":
    img = synth.generate("c3_percolation_8192")
elif case == "bernoulli06_2048x8192":
    img = synth.bernoulli(2048, 8192, 0.6, seed=5)
elif case == "handed_over_dense":
    img = _handed_over_dense()
elif case == "c1_batch64":
    batch = [synth.bernoulli(512, 512, 0.5, seed=100 + b) for b in range(64)]
else:
    img = synth.generate(case)
if batch:
    want = [oracle.label(im) for im in batch]
    ref = torch.from_numpy(np.stack([w[0] for w in want])).cuda()
    nref = torch.tensor([w[1] for w in want], dtype=torch.int32, device="cuda")
    t = torch.from_numpy(np.stack(batch)).cuda()
    plan = ccl.Plan(512, 512, batch=64)
else:
    lo, no = oracle.label(img)
    ref = torch.from_numpy(lo).cuda()
    nref = torch.tensor([no], dtype=torch.int32, device="cuda")
    t = torch.from_numpy(img).cuda()
    plan = ccl.Plan(*img.shape)
out = torch.empty_like(ref)
n = torch.empty_like(nref)
bad = 0
for i in range(reps):
    out.fill_(-7)
    plan.label(t, out, n)
    torch.cuda.synchronize()
    if torch.equal(n, nref) and torch.equal(out, ref):
        continue
    bad += 1
    if bad <= 4:
        d = (out != ref).nonzero()
        print(f"run {i}: n {n.tolist()[:4]} vs {nref.tolist()[:4]}, {len(d)} px differ, first {d[0].tolist()}",
              flush=True)
print(json.dumps({"case": case, "reps": reps, "bad": bad, "counters": plan.counters()}), flush=True)
