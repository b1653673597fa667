"""K1 truncated after each phase (ccl_debug_set(1, stop)), one launch per
stop -- run under ncu --metrics smsp__inst_executed.sum to get the
instruction count of every phase (cumulative).  Needs the knob build (see
scripts/k1_phases.py)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1606_05973_b200 as ccl
img = torch.from_numpy(synth.generate(sys.argv[1] if len(sys.argv) > 1 else "c4_voronoi_21600")).cuda()
plan = ccl.Plan(*img.shape)
out = torch.empty(img.shape, dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
for stop in [-1, 0, 1, 2, 3, 4, 5, 99]:
    ccl._L.ccl_debug_set(1, stop)
    plan.label(img, out, n)
    torch.cuda.synchronize()
    print("stop", stop, flush=True)
