"""Strong-scaling projection on ONE GPU: the per-rank work of an N-band run
(the band of rank 0, H/N rows of C4) timed through a whole-image plan and
through the row-band path with one rank (the protocol's kernels without the
NCCL exchange).  The N-GPU step is then about the band time plus three small
all-gathers (2W int64 + 2W int32, N int32, 2W int32 per band)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1606_05973_b200 as ccl
img = synth.generate("c4_voronoi_21600")
H, W = img.shape
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
uid = ccl.nccl_unique_id()
comm = ccl.NcclComm(uid, 1, 0)
for N in [1, 2, 4, 8]:
    bh = H // N
    band = torch.from_numpy(img[:bh].copy()).cuda()
    out = torch.empty((bh, W), dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
    plan = ccl.Plan(bh, W)
    tp = t(lambda: plan.label(band, out, n))
    sp = ccl.ShardPlan(bh, W, 0, bh, comm)
    ts = t(lambda: sp.label(band, out, n))
    plan.set_profiling(20)
    for _ in range(20): plan.label(band, out, n)
    torch.cuda.synchronize()
    kt = plan.kernel_times(); plan.set_profiling(0)
    sp.set_profiling(20)
    for _ in range(20): sp.label(band, out, n)
    torch.cuda.synchronize()
    st = sp.kernel_times(); sp.set_profiling(0)
    print(f"N={N}: band {bh}x{W}: plan {tp*1e3:.1f} us, band path (1 rank) {ts*1e3:.1f} us, "
          f"projected whole-image {H*W/(ts*1e-3)/1e9:.0f} Gpx/s before the exchange; kernels "
          + " ".join(f"{k} {v*1e3:.1f}" for k, v in kt.items())
          + "; band-path stages " + " ".join(f"{k} {v*1e3:.1f}" for k, v in st.items()), flush=True)
