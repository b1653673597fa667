"""Is the single small-image call host-bound?  C1/C2 one image per call:
eager plan.label x N vs the same call captured once in a CUDA graph and
replayed (torch.cuda.CUDAGraph around the library's launches)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
import paper_1606_05973_b200 as ccl
for name in ["c1_bernoulli_512", "c2_blobs_1024"]:
    img = synth.generate(name)
    H, W = img.shape
    t = torch.from_numpy(img).cuda()
    plan = ccl.Plan(H, W)
    o = torch.empty((H, W), dtype=torch.int32, device="cuda")
    n = torch.empty(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(5):
            plan.label(t, o, n, stream=s)
    torch.cuda.synchronize()
    reps = 200
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        h0 = time.perf_counter()
        for _ in range(reps):
            plan.label(t, o, n, stream=s)
        h1 = time.perf_counter()
        b.record(s)
    torch.cuda.synchronize()
    eager = a.elapsed_time(b) / reps * 1e3
    host = (h1 - h0) / reps * 1e6
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.label(t, o, n, stream=s)
    torch.cuda.synchronize()
    o.zero_()
    g.replay(); torch.cuda.synchronize()
    lo, no = oracle.label(img)
    ok = int(n.item()) == no and np.array_equal(o.cpu().numpy(), lo)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    graph = a.elapsed_time(b) / reps * 1e3
    print(f"{name}: eager {eager:.1f} us/call (host enqueue {host:.1f} us/call), graph replay {graph:.1f} us/call, graph output bit-exact {ok}", flush=True)
