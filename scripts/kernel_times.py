"""Per-kernel CUDA-event times (Plan.set_profiling) of one plan per config:
where a config's step time goes.  usage: python scripts/kernel_times.py [names...]"""
import sys, os, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_1606_05973_b200 as ccl

import numpy as np
names = sys.argv[1:] or list(synth.CONFIGS)
for name in names:
    batch = None
    if ":" in name:  # name:B = a batch of B copies through ccl_plan_create_batch
        name, batch = name.split(":")[0], int(name.split(":")[1])
    img = synth.generate(name)
    H, W = img.shape
    if batch:
        t = torch.from_numpy(np.stack([img] * batch)).cuda()
        plan = ccl.Plan(H, W, batch=batch)
        o = torch.empty((batch, H, W), dtype=torch.int32, device="cuda")
        n = torch.empty(batch, dtype=torch.int32, device="cuda")
        name = f"{name}:{batch}"
    else:
        t = torch.from_numpy(img).cuda()
        plan = ccl.Plan(H, W)
        o = torch.empty((H, W), dtype=torch.int32, device="cuda")
        n = torch.empty(1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        plan.label(t, o, n)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        plan.label(t, o, n)
    b.record()
    torch.cuda.synchronize()
    plan.set_profiling(20)
    for _ in range(20):
        plan.label(t, o, n)
    kt = plan.kernel_times()
    us = a.elapsed_time(b) / 20 * 1e3
    print(json.dumps({"config": name, "us_per_call": us, "gpx_s": t.numel() / us / 1e3,
                      "kernels_us": {k: round(v * 1e3, 1) for k, v in kt.items()},
                      "counters": plan.counters()}), flush=True)
    del t, o, plan
