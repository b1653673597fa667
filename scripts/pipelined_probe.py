"""Frame-stream throughput: consecutive C4 labelings on one stream (the bench
step) vs two plans on two streams, so one frame's label write (K5, HBM-bound)
can overlap the next frame's tile pass (K1, issue-bound).  Device-timed with
events; every output is checked equal to the serial result."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1606_05973_b200 as ccl

name = sys.argv[1] if len(sys.argv) > 1 else "c4_voronoi_21600"
K = 24
img = torch.from_numpy(synth.generate(name)).cuda()
H, W = img.shape
plans = [ccl.Plan(H, W), ccl.Plan(H, W)]
outs = [torch.empty((H, W), dtype=torch.int32, device="cuda") for _ in range(2)]
ns = [torch.empty(1, dtype=torch.int32, device="cuda") for _ in range(2)]
ref = torch.empty((H, W), dtype=torch.int32, device="cuda"); nref = torch.empty(1, dtype=torch.int32, device="cuda")
plans[0].label(img, ref, nref)
torch.cuda.synchronize()


def run(streams, nplans):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    for rep in range(2):  # warm-up pass, then the timed pass
        torch.cuda.synchronize()
        a.record(cur)
        for s in streams:
            s.wait_stream(cur)
        for k in range(K):
            i = k % len(streams)
            p = k % nplans
            plans[p].label(img, outs[p], ns[p], stream=streams[i])
        for s in streams:
            cur.wait_stream(s)
        b.record(cur)
        torch.cuda.synchronize()
    for p in range(nplans):
        assert torch.equal(outs[p], ref) and int(ns[p]) == int(nref)
    us = a.elapsed_time(b) * 1e3 / K
    return us, H * W / us / 1e3


s0 = torch.cuda.Stream()
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
sh = torch.cuda.Stream(priority=-1)
s1 = torch.cuda.Stream()
for label, streams, nplans in [("serial, 1 stream", [s0], 1),
                               ("2 plans, 2 streams", [s0, s1], 2),
                               ("2 plans, 2 streams (2nd high priority)", [s0, sh], 2),
                               ("serial again", [s0], 1)]:
    us, g = run(streams, nplans)
    print(f"{name} {label}: {us:.1f} us/frame, {g:.0f} Gpx/s")
