"""Probe: do two C4 frames labelled on two streams (two plans) overlap one
frame's issue-bound K1 with the other's HBM-bound K5?  Prints us per frame for
one stream (PDL-chained, as bench.py) and for two streams, equal and mixed
priorities.  usage: python scripts/two_stream_probe.py [frames]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_05973_b200 as ccl  # noqa: E402
import synth  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 40
img = torch.from_numpy(synth.generate("c4_voronoi_21600")).cuda()
H, W = img.shape
plans = [ccl.Plan(H, W), ccl.Plan(H, W)]
outs = [torch.empty((H, W), dtype=torch.int32, device="cuda") for _ in range(2)]
ns = [torch.empty(1, dtype=torch.int32, device="cuda") for _ in range(2)]
ref, nref = plans[0].label(img)
torch.cuda.synchronize()
ref = ref.clone()


def run(streams, K):
    for i in range(K):
        j = i % len(streams)
        plans[j].label(img, outs[j], ns[j], stream=streams[j])


def timeit(streams, K):
    run(streams, 6)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for s in streams:
        s.wait_event(e0)
    run(streams, K)
    for s in streams:
        ev = torch.cuda.Event()
        ev.record(s)
        cur.wait_event(ev)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / K


s0 = torch.cuda.Stream()
print("one stream      us/frame", round(timeit([s0], K), 1))
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
print("two streams     us/frame", round(timeit([sa, sb], K), 1))
hi, lo = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
print("two, hi/lo prio us/frame", round(timeit([hi, lo], K), 1))
for j in range(2):
    assert torch.equal(outs[j], ref) and int(ns[j].item()) == int(nref.item()), "labels differ"
print("labels bit-identical to the one-stream run")
