"""Per-kernel roofline table of C4 from the committed bench line and ncu summary.
usage: python scripts/roofline_table.py profiles/r02_bench.json profiles/ncu_summary.json > profiles/r02_roofline.txt"""
import json, sys
b = json.load(open(sys.argv[1]))
n = json.load(open(sys.argv[2]))["c4_voronoi_21600"]
r = b["roofline"]
peak = r["peak"]
issue_peak = 148 * 4 * 1965e6
print("Per-kernel roofline, C4 21600x21600 (466.56 Mpx) on one B200 -- r02")
print(f"  event us: bench.py second pass with CUDA events between kernels ({sys.argv[1]})")
print(f"  ncu: --set full, cold cache, serialised ({sys.argv[2]}; profiles/r02_ncu_summary.txt)")
print(f"  peak: MEASURED_PEAKS.json hbm_gbs = {peak} GB/s (copy, read+write); issue peak 148 SMs x 4 x 1965 MHz"
      f" = {issue_peak:.4g} warp-inst/s")
print()
print(f"{'kernel':13s} {'event_us':>8s} {'ncu_us':>7s} {'alg_MB':>8s} {'dram_MB':>8s} {'alg_GB/s':>8s} "
      f"{'alg_frac':>8s} {'dram_GB/s':>9s} {'issue_frac':>10s}")
for k, e in r["kernels"].items():
    s = n.get(k, {})
    us = e["ms"] * 1e3
    alg = e.get("algorithmic_bytes", 0) / 1e6
    dram = (s.get("dram_bytes_read", 0) + s.get("dram_bytes_write", 0)) / 1e6
    ncu_us = s.get("duration_ms", 0) * 1e3
    ag = alg / us * 1e3 if us else 0  # MB/us = TB/s -> GB/s
    dg = dram / ncu_us * 1e3 if ncu_us else 0
    iss = s.get("warp_inst", 0) / (ncu_us * 1e-6) / issue_peak if ncu_us else 0
    print(f"{k:13s} {us:8.1f} {ncu_us:7.1f} {alg:8.1f} {dram:8.1f} {ag:8.0f} "
          f"{ag/peak:8.3f} {dg:9.0f} {iss:10.2f}")
p = r["path"]
print()
print(f"path: {b['ms_per_step']*1e3:.1f} us per step, 5 B/px = 2.33 GB -> {p['achieved']:.0f} GB/s = "
      f"{p['frac']:.3f} of the measured peak, {p['achieved']/8000:.3f} of 8 TB/s")
