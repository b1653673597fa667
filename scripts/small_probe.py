"""Small-image latency: host-side enqueue cost vs device time (per-kernel
events) vs CUDA-graph replay of the same plan call."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1606_05973_b200 as ccl
for name in ["c1_bernoulli_512", "c2_blobs_1024"]:
    img = torch.from_numpy(synth.generate(name)).cuda()
    H, W = img.shape
    plan = ccl.Plan(H, W)
    out = torch.empty((H, W), dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
    for _ in range(20): plan.label(img, out, n)
    torch.cuda.synchronize()
    reps = 2000
    t0 = time.perf_counter()
    for _ in range(reps): plan.label(img, out, n)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host enqueue {1e6*(t1-t0)/reps:.1f} us/call, wall {1e6*(t2-t0)/reps:.1f} us/call")
    plan.set_profiling(50)
    for _ in range(50): plan.label(img, out, n)
    torch.cuda.synchronize()
    kt = plan.kernel_times(); plan.set_profiling(0)
    print("  per-kernel (events, serialised):", {k: round(v * 1e3, 1) for k, v in kt.items()}, "sum", round(sum(kt.values()) * 1e3, 1))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): plan.label(img, out, n)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            for _ in range(10): plan.label(img, out, n)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.replay(); torch.cuda.synchronize()
        a.record()
        for _ in range(100): g.replay()
        b.record(); torch.cuda.synchronize()
        print(f"  graph replay: {a.elapsed_time(b) * 1e3 / 1000:.1f} us/call (device)")
    except Exception as e:
        print("  graph capture failed:", repr(e)[:200])
