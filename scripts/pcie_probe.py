"""D2H / H2D copy bandwidth with pinned buffers: one cudaMemcpyAsync vs the
same bytes split over 2 / 4 streams, and H2D + D2H at once (the e2e path's
bound)."""
import sys, time, torch
n = 1866240000
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
hi = torch.empty(466560000, dtype=torch.uint8).pin_memory()
di = torch.empty(466560000, dtype=torch.uint8, device="cuda")
def run(k, both=False):
    ss = [torch.cuda.Stream() for _ in range(k + 1)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in range(3):
        for i, s in enumerate(ss[:k]):
            with torch.cuda.stream(s):
                a, b = n * i // k, n * (i + 1) // k
                h[a:b].copy_(d[a:b], non_blocking=True)
        if both:
            with torch.cuda.stream(ss[k]):
                di.copy_(hi, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"D2H split {k}{' + H2D 466 MB concurrently' if both else ''}: {dt*1e3:.1f} ms, {n/dt/1e9:.1f} GB/s", flush=True)
for k in (1, 2, 4):
    run(k)
run(1, True)
run(2, True)
