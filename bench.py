#!/usr/bin/env python
"""bench.py -- throughput of the B200 CCL hot path (BASELINE.json metric:
"8-conn CCL Gpixel/s on 21600^2 image at 1/2/4/8 B200; % of HBM roofline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the whole hot path (all SURVEY.md section 8(a) rows:
load+predicate, tile-local scan+union, border merge, flatten/root ranking,
decoupled-lookback numbering, label write) over the 21600x21600 C4 workload
(configs[3]: 20,000-cell Voronoi class map + 5% flips), input resident in HBM.
At N>1 (torchrun) the image is split into row bands, one per rank
(ccl_label_sharded, NCCL over NVLink); value = H*W / max-over-ranks step time.

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement".
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


METRIC = "8-conn CCL Gpixel/s on 21600² image at 1/2/4/8 B200; % of HBM roofline"
WORKLOAD = "c4_voronoi_21600"
# algorithmic bytes per pixel: 1 B image read + 4 B label write
# (k_tile_local reads the image, k_write writes the labels; the rest move intermediates)
ALG_BYTES_PER_PX = {"path": 5, "k_tile_local": 1, "k_write": 4,
                    "k_border": 0, "k_number": 0, "k_label": 0, "k_fixup": 0}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default=WORKLOAD)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-runs", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-small", action="store_true", help="skip the C1/C2 single vs batched lines")
    ap.add_argument("--shard", action="store_true",
                    help="use the row-band (NCCL) path even on one GPU (tests the multi-GPU code path)")
    return ap.parse_args()


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: STREAM-style copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s earlier measurement on this pool)"


def ncu_issue(kernel, workload, sm_mhz=1965.0, sms=148):
    """Instruction-issue utilisation of a kernel from the committed ncu --set
    full summary: executed warp instructions / (duration x issue peak = 148 SMs
    x 4 schedulers x 1 warp-instruction per clock at the SM clock)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            e = json.load(f)[workload][kernel]
        rate = float(e["warp_inst"]) / (float(e["duration_ms"]) * 1e-3)
        peak = sms * 4 * sm_mhz * 1e6
        return {"unit": "warp-instructions/s", "achieved": rate, "peak": peak, "frac": rate / peak,
                "issue_active_pct": e.get("issue_active_pct"), "source": "profiles/ncu_summary.json (ncu --set full)"}
    except Exception:
        return None


def ncu_traffic(kernel, workload):
    """dram read+write bytes per launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d[workload][kernel]
        return float(e["dram_bytes_read"]) + float(e["dram_bytes_write"])
    except Exception:
        return None


class ClockSampler:
    """Samples SM clocks and clock-event reasons through NVML in a thread while
    the timed region runs (the recipe's nvidia-smi clocks line, via the same
    library)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x100: "display_clock_setting",
               0x10: "sync_boost", 0x1: "gpu_idle"}

    def __init__(self, device_index, period_s=0.002):
        self.samples, self.reasons = [], 0
        self.period = period_s
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device_index]) if vis else device_index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        n = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append(n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM))
                self.reasons |= n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def report(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        reasons = [v for k, v in sorted(self.REASONS.items()) if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def make_roofline(ktimes, H, W, bh, ms, ws, peak, peak_src, workload):
    """The path is HBM-bound by its algorithmic bytes (SURVEY.md section 8(d):
    1 B read + 4 B written per pixel).  Top level = the dominant kernel (its
    algorithmic bytes per launch / its average launch time, CUDA events on the
    launch stream); `path` = the whole step against the peak.  At N > 1 every
    figure is per GPU: this rank's band (bh rows) over the max-over-ranks step
    time -- the per-GPU roofline % = 5*H*W / (n * B_peak * t) of SURVEY.md 8(d)."""
    alg = ALG_BYTES_PER_PX["path"] * H * W
    ach_gpu = alg / ws / (ms * 1e-3) / 1e9
    kern = {}
    for k, t in ktimes.items():
        e = {"ms": t, "share": t / sum(ktimes.values())}
        if ALG_BYTES_PER_PX.get(k):
            e["algorithmic_bytes"] = ALG_BYTES_PER_PX[k] * bh * W
            e["achieved_gbs"] = e["algorithmic_bytes"] / (t * 1e-3) / 1e9
            e["frac"] = e["achieved_gbs"] / peak
        if ws == 1:
            tr = ncu_traffic(k, workload)
            if tr is not None:
                e["ncu_dram_bytes"] = tr
            iss = ncu_issue(k, workload)
            if iss is not None:
                e["issue"] = iss
        kern[k] = e
    tr_all = [kern[k].get("ncu_dram_bytes") for k in kern if k in ALG_BYTES_PER_PX]
    dom = max((k for k in ktimes if ALG_BYTES_PER_PX.get(k)), key=ktimes.get)
    d = kern[dom]
    r = {"bound": "hbm", "kernel": dom,
         "achieved": d.get("achieved_gbs", 0.0), "peak": peak, "unit": "GB/s",
         "frac": d.get("frac", 0.0), "traffic": d.get("ncu_dram_bytes"),
         "algorithmic_bytes_per_launch": d.get("algorithmic_bytes", 0),
         "peak_source": peak_src,
         "path": {"achieved": ach_gpu, "frac": ach_gpu / peak, "frac_of_8tbps": ach_gpu / 8000.0,
                  "algorithmic_bytes_per_step": alg // ws if ws > 1 else alg,
                  "per_gpu": ws > 1,
                  "traffic": sum(tr_all) if tr_all and all(t is not None for t in tr_all) else None},
         "kernels": kern}
    if ws > 1:
        r["note"] = ("per GPU: rank 0's band; stage times from rank 0's ShardPlan events; "
                     "xband_* stages = the cross-band protocol incl. its NCCL all-gathers")
    # K1 moves 1 B/px of algorithmic bytes but is bound by instruction issue
    # (shared-memory union-find, bit-parallel scans): its issue utilisation
    # (ncu, committed summary) is reported beside the HBM roofline
    iss = ncu_issue("k_tile_local", workload) if ws == 1 else None
    if iss is not None:
        r["issue"] = dict(iss, kernel="k_tile_local")
    return r


def cpu_model():
    """Host CPU model name and logical core count (report the
    box's host as measured)."""
    name = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    name = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return name, os.cpu_count()


def time_paremsp(img, runs):
    """the multi-core host PARemSP (paremsp/, OpenMP, all
    host cores), output checked against the oracle's by the caller."""
    import paremsp
    ts, out = [], None
    for _ in range(runs):
        t0 = time.perf_counter()
        out = paremsp.label(img)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), out


def other_configs(dev, stream, reps=10):
    """Single-image throughput on the other BASELINE.json configs (C1, C2,
    C3, C5a-d): parity cases, reported beside the C4 bench line; each call
    labels one device-resident image (CUDA events on the launch stream)."""
    import torch
    import synth
    import paper_1606_05973_b200 as ccl
    res = {}
    for name in synth.CONFIGS:
        if name == WORKLOAD:
            continue
        img = synth.generate(name)
        H, W = img.shape
        t = torch.from_numpy(img).to(dev)
        plan = ccl.Plan(H, W, device=dev)
        o = torch.empty((H, W), dtype=torch.int32, device=dev)
        n = torch.empty(1, dtype=torch.int32, device=dev)
        for _ in range(3):
            plan.label(t, o, n)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            plan.label(t, o, n)
        b.record(stream)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b) / reps
        res[name] = {"H": H, "W": W, "us_per_call": ms * 1e3, "gpx_s": H * W / (ms * 1e-3) / 1e9,
                     "path_frac": 5 * H * W / (ms * 1e-3) / 1e9 / peak_hbm()[0],
                     "n_components": int(n.item())}
        del t, o, plan
    return res


def time_oracle(img, runs):
    import oracle
    ts, out = [], None
    for _ in range(runs):
        t0 = time.perf_counter()
        out = oracle.label(img)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), out


def small_images(dev, stream, batch=64, reps=20):
    import numpy as np
    import torch
    import synth
    import paper_1606_05973_b200 as ccl
    res = {}
    for name in ["c1_bernoulli_512", "c2_blobs_1024"]:
        img = synth.generate(name)
        H, W = img.shape
        single = torch.from_numpy(img).to(dev)
        stack = torch.from_numpy(np.stack([img] * batch)).to(dev)
        p1, pb = ccl.Plan(H, W, device=dev), ccl.Plan(H, W, device=dev, batch=batch)
        o1, ob = torch.empty((H, W), dtype=torch.int32, device=dev), torch.empty((batch, H, W), dtype=torch.int32, device=dev)
        n1, nb = torch.empty(1, dtype=torch.int32, device=dev), torch.empty(batch, dtype=torch.int32, device=dev)
        out = {}
        for tag, fn, px in (("single", lambda: p1.label(single, o1, n1), H * W),
                            (f"batch{batch}", lambda: pb.label(stack, ob, nb), batch * H * W)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                fn()
            b.record(stream)
            torch.cuda.synchronize(dev)
            ms = a.elapsed_time(b) / reps
            # us_per_call: back-to-back calls (each call's launch overlaps
            # the previous call's tail); isolated_us: one call between two
            # synchronisations (median of reps), the latency a lone call sees
            iso = []
            for _ in range(reps):
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize(dev)
                iso.append(a.elapsed_time(b) * 1e3)
            out[tag] = {"us_per_call": ms * 1e3, "gpx_s": px / (ms * 1e-3) / 1e9,
                        "isolated_us": statistics.median(iso)}
        res[name] = out
    return res


class stdout_to_stderr:
    """NCCL prints its version banner on stdout at communicator creation (this
    image sets NCCL_DEBUG=VERSION), which would break the one-JSON-line
    contract: point file descriptor 1 at stderr while communicators are made."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def two_streams(plan, d_img, H, W, dev, K):
    """K frames of the workload alternating over two plans on two streams."""
    import torch
    import paper_1606_05973_b200 as ccl
    plans = [plan, ccl.Plan(H, W, device=dev)]
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    outs = [torch.empty((H, W), dtype=torch.int32, device=dev) for _ in range(2)]
    ns = [torch.empty(1, dtype=torch.int32, device=dev) for _ in range(2)]
    cur = torch.cuda.current_stream(dev)

    def run(k):
        for i in range(k):
            j = i & 1
            plans[j].label(d_img, outs[j], ns[j], stream=streams[j])

    for s in streams:
        s.wait_stream(cur)
    run(6)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for s in streams:
        s.wait_event(e0)
    run(K)
    for s in streams:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize(dev)
    us = e0.elapsed_time(e1) * 1e3 / K
    same = bool(torch.equal(outs[0], outs[1]) and int(ns[0].item()) == int(ns[1].item()))
    del plans[1]
    return {"us_per_frame": us, "gpx_s": H * W / (us * 1e-6) / 1e9, "frames": K,
            "labels_identical_across_plans": same,
            "note": "two plans on two streams, frames alternating (serving context, not value)"}


def run_reference(args):
    """The reference arm for this tier: the CPU oracle as it stands (plain C
    ARemSP + canonical renumbering, single-threaded) on the same workload."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    import synth
    img = synth.generate(args.workload)
    H, W = img.shape
    import oracle
    # each step labels a bounded sample: the whole image while the run fits in
    # about two minutes, else the first rows of it (a row band, as PARemSP's
    # chunks) sized to that budget -- the rate is per pixel either way
    t0 = time.perf_counter()
    oracle.label(img)
    t_full = time.perf_counter() - t0
    budget_s = 120.0
    rows = H
    if (args.steps + max(0, args.warmup - 1)) * t_full > budget_s:
        rows = max(1, int(H * budget_s / ((args.steps + max(0, args.warmup - 1)) * t_full)))
    sample = np.ascontiguousarray(img[:rows]) if rows < H else img
    for _ in range(max(0, args.warmup - 1)):
        oracle.label(sample)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.label(sample)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    v = rows * W / t / 1e9
    t = H * W / (v * 1e9)  # per full image at the measured rate
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "Gpx/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": {"workload": args.workload, "H": H, "W": W},
        "cpu_baseline": {"value": v, "unit": "Gpx/s", "cores": 1, "kind": "oracle",
                         "sample": (f"full {H}x{W} {args.workload} image per step" if rows == H else
                                    f"first {rows} of {H} rows of the {H}x{W} {args.workload} image per step "
                                    f"(the run bounded to ~{budget_s:.0f} s)") + " (single-threaded C oracle)"},
        "e2e": {"value": v, "unit": "Gpx/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import synth
    import paper_1606_05973_b200 as ccl

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        with stdout_to_stderr():
            dist.init_process_group("nccl", device_id=dev)

    img = synth.generate(args.workload)
    H, W = img.shape
    # contiguous row bands, remainder to the last ranks (PARemSP chunking)
    bands = [H // ws + (1 if k >= ws - H % ws else 0) for k in range(ws)]
    row0 = sum(bands[:rank])
    bh = bands[rank]
    band = np.ascontiguousarray(img[row0:row0 + bh])
    d_img = torch.from_numpy(band).to(dev)
    out = torch.empty((bh, W), dtype=torch.int32, device=dev)
    n_out = torch.empty(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    if ws == 1 and not args.shard:
        plan = ccl.Plan(H, W, device=dev)
        step = lambda: plan.label(d_img, out, n_out)  # noqa: E731
        nTx, nTy = (W + 1023) // 1024, (H + 31) // 32
        # mirrors cclb::pipeline_launches: k_border only runs when tiles have neighbours
        launches_per_step = 5 + (1 if (nTy - 1) * nTx + (nTx - 1) * H > 0 else 0)
    else:
        with stdout_to_stderr():
            uid = ccl.nccl_unique_id() if rank == 0 else None
            obj = [uid]
            if dist:
                dist.broadcast_object_list(obj, src=0)
            comm = ccl.NcclComm(obj[0], ws, rank)
        splan = ccl.ShardPlan(bh, W, row0, H, comm)
        step = lambda: splan.label(d_img, out, n_out)  # noqa: E731
        plan = None
        # our kernels per band step (ccl_bands.cu): K1 (+ its hand-over pass), K2, boundary rows
        # (+ representative minima), slot representatives (+ the slot union-find's start),
        # slot unions, link, K3, export, K4 (+ band offset), K5 (the 2 NCCL
        # all-gathers are not counted)
        launches_per_step = 11

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = H * W / (ms * 1e-3) / 1e9
    result_labels = out.cpu().numpy() if not args.no_parity else None

    # single-call latency: one step with the device idle before it (a
    # synchronize, then CUDA events around the one call) -- the timed loop
    # above chains steps back to back (the next step's first kernel is
    # scheduled while the previous step's last kernel drains)
    lat = []
    for _ in range(5):
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        torch.cuda.synchronize(dev)
        lat.append(a.elapsed_time(b))
    latency_ms = statistics.median(lat)
    n_gpu = int(n_out.item())

    peak, peak_src = peak_hbm()
    # Per-kernel (per-stage) times: the same K steps again with CUDA events
    # recorded on the launch stream between the kernels.  Kept out of the
    # timed region above because events between kernels serialise the
    # programmatic dependent launches the pipeline uses.  At N > 1 every rank
    # profiles its own band (ShardPlan); rank 0's times are reported.
    prof = plan if plan is not None else splan
    prof.set_profiling(args.steps)
    if dist:
        dist.barrier()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize(dev)
    ktimes = prof.kernel_times()
    prof.set_profiling(0)
    roofline = make_roofline(ktimes, H, W, bh, ms, ws, peak, peak_src, args.workload)

    line = {
        "metric": METRIC, "value": value, "unit": "Gpx/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": args.workload, "H": H, "W": W, "bands": bands,
                   "l2": "inputs larger than L2 (466.6 MB image in, 1.87 GB labels out vs 126 MB L2); no flush"},
        "clocks": clk.report(),
        "gpu_launches": (launches_per_step * args.steps) if launches_per_step else None,
        "single_call_latency_ms": latency_ms,
        "roofline": roofline,
    }

    # ---- serving context (not `value`): two frames in flight, two plans on
    # two streams, frames alternating; device-resident, CUDA events.  Only the
    # kernels' tails overlap (K5 takes every warp slot while it runs), see
    # DESIGN.md section 11.
    if ws == 1 and plan is not None and not args.no_small:
        line["frames_two_streams"] = two_streams(plan, d_img, H, W, dev, args.steps)

    # ---- the paper's <= 1 MB regime (C1, C2): one image per call vs a batch
    # of 64 per call (ccl_label_batch), device-resident, CUDA events
    if ws == 1 and plan is not None and not args.no_small:
        line["small_images"] = small_images(dev, stream)
        line["other_configs"] = other_configs(dev, stream)

    # ---- end to end through the public API with host buffers (N=1): frames
    # back to back through ccl_plan_label_host_async (each call's H2D and
    # kernels overlap the previous call's D2H; the copies of every step are
    # inside the timed region), wall clock from the first call to the final
    # synchronize; plus one synchronous call's latency
    if ws == 1 and plan is not None and not args.no_e2e:
        h_img = torch.from_numpy(img).pin_memory()
        h_labs = [torch.empty((H, W), dtype=torch.int32).pin_memory() for _ in range(2)]
        h_ns = [torch.empty(1, dtype=torch.int32).pin_memory() for _ in range(2)]
        plan.label_host(h_img, h_labs[0], h_ns[0])  # warm the staging buffers
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        plan.label_host(h_img, h_labs[0], h_ns[0])
        single_ms = (time.perf_counter() - t0) * 1e3
        for i in range(2):
            plan.label_host_async(h_img, h_labs[i % 2], h_ns[i % 2])
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            plan.label_host_async(h_img, h_labs[i % 2], h_ns[i % 2])
        stream.synchronize()
        ems = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        e2e_ok = int(h_ns[0][0]) == n_gpu and (result_labels is None or
                                                 bool(np.array_equal(h_labs[0].numpy(), result_labels)))
        line["e2e"] = {"value": H * W / (ems * 1e-3) / 1e9, "unit": "Gpx/s",
                       "h2d_bytes_per_step": H * W, "d2h_bytes_per_step": H * W * 4 + 4,
                       "ms_per_step": ems, "mode": "pipelined frames (ccl_plan_label_host_async), wall clock",
                       "single_call_ms": single_ms, "labels_match_device_run": e2e_ok}
        del h_labs

    # ---- end to end at N > 1 (or --shard): every rank copies its band in from
    # pinned host memory, labels it through the sharded API, and reads its
    # labels and N back; max over ranks of the per-step time
    if plan is None and not args.no_e2e:
        h_band = torch.from_numpy(band).pin_memory()
        h_lab = torch.empty((bh, W), dtype=torch.int32).pin_memory()
        h_n = torch.empty(1, dtype=torch.int32).pin_memory()

        def e2e_step():
            d_img.copy_(h_band, non_blocking=True)
            splan.label(d_img, out, n_out)
            h_lab.copy_(out, non_blocking=True)
            h_n.copy_(n_out, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize(dev)
        ems = a.elapsed_time(b) / args.e2e_steps
        if dist:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        line["e2e"] = {"value": H * W / (ems * 1e-3) / 1e9, "unit": "Gpx/s",
                       "h2d_bytes_per_step": H * W, "d2h_bytes_per_step": H * W * 4 + 4 * ws,
                       "ms_per_step": ems}

    # ---- parity at N > 1: every rank checks its band of the timed output
    # against the oracle's labels of the whole image (one flag, max over ranks)
    if plan is None and result_labels is not None and not args.no_cpu_baseline:
        import oracle
        lab_o, n_o = oracle.label(img)
        bad = int(n_o != n_gpu or not np.array_equal(lab_o[row0:row0 + bh], result_labels))
        if dist:
            t = torch.tensor([bad], dtype=torch.int32, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            bad = int(t.item())
        line["parity"] = {"vs": "oracle", "bit_exact": bad == 0, "n_components": n_gpu,
                          "checked": "every rank's band"}

    # ---- CPU baseline (the oracle as it stands) + parity of the timed output
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu, ncpu = cpu_model()
        t, (lab_o, n_o) = time_oracle(img, args.cpu_runs)
        line["cpu_baseline"] = {"value": H * W / t / 1e9, "unit": "Gpx/s", "cores": 1, "kind": "oracle",
                                "host_cpu": cpu, "host_logical_cores": ncpu,
                                "sample": f"full {H}x{W} {args.workload} image, median of {args.cpu_runs} runs, "
                                          "single-threaded C oracle (ARemSP + canonical renumbering)"}
        if result_labels is not None:
            same = (n_o == n_gpu) and bool(np.array_equal(lab_o, result_labels))
            line["parity"] = {"vs": "oracle", "bit_exact": same, "n_components": n_gpu}
        # the paper's own parallel design on all host cores
        tp, (lab_p, n_p, used) = time_paremsp(img, args.cpu_runs)
        line["cpu_baseline_paremsp"] = {
            "value": H * W / tp / 1e9, "unit": "Gpx/s", "cores": used, "kind": "paremsp_openmp",
            "host_cpu": cpu, "host_logical_cores": ncpu,
            "bit_exact_vs_oracle": bool(n_p == n_o and np.array_equal(lab_p, lab_o)),
            "sample": f"full {H}x{W} {args.workload} image, median of {args.cpu_runs} runs, PARemSP "
                      "(paremsp/: OpenMP row chunks, locked boundary merger, parallel flatten + "
                      "canonical renumbering)"}
        del lab_p
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
