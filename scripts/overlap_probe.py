"""Two frames in flight: plans P0, P1 on streams s0, s1, frames alternating,
so one frame's labeling kernels (K5, HBM-bound) can share the GPU with the
next frame's K1 (issue-bound).  Prints us/frame for 1 and 2 streams.
usage: python scripts/overlap_probe.py [config] [frames]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1606_05973_b200 as ccl
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c4_voronoi_21600"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 40
img = torch.from_numpy(synth.generate(name)).cuda()
H, W = img.shape
for nst in (1, 2, 3, 1, 2):
    plans = [ccl.Plan(H, W) for _ in range(nst)]
    outs = [torch.empty((H, W), dtype=torch.int32, device="cuda") for _ in range(nst)]
    ns = [torch.empty(1, dtype=torch.int32, device="cuda") for _ in range(nst)]
    streams = [torch.cuda.Stream() for _ in range(nst)]
    for i in range(3 * nst):
        plans[i % nst].label(img, outs[i % nst], ns[i % nst], stream=streams[i % nst])
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    main = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(main)
    for i in range(K):
        j = i % nst
        plans[j].label(img, outs[j], ns[j], stream=streams[j])
    for s in streams:
        main.wait_stream(s)
    t1.record()
    torch.cuda.synchronize()
    us = t0.elapsed_time(t1) * 1000 / K
    print(f"{name} streams={nst} {us:.1f} us/frame  {H * W / us / 1e3:.1f} Gpx/s  N={[int(n.item()) for n in ns]}",
          flush=True)
    del plans, outs
    torch.cuda.empty_cache()
