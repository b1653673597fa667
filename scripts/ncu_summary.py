"""Summarise an ncu --set full report: per kernel duration, DRAM bytes,
throughput, occupancy, top stall reasons and the hottest source lines.

  python scripts/ncu_summary.py gpurun_out/prof_TAG.ncu-rep [--json profiles/ncu_summary.json]
      [--workload c4_voronoi_21600] [--lines N]
"""
import argparse
import csv
import re
import io
import json
import os
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_shared_mem", "occ_limit_smem"),
    ("launch__grid_size", "grid"),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def ncu_csv(args):
    out = subprocess.run([NCU] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--json")
    ap.add_argument("--workload", default="c4_voronoi_21600")
    ap.add_argument("--lines", type=int, default=12)
    a = ap.parse_args()
    rows = ncu_csv(["-i", a.report, "--page", "raw", "--csv"])
    hdr, units = rows[0], rows[1]
    summary = {}
    for r in rows[2:]:
        name = re.sub(r"<.*", "", r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]).replace("void ", "").strip()
        e = {}
        for m, key in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                e[key] = v * UNIT.get(units[i], 1.0) if key in ("duration", "dram_read", "dram_write") else v
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__average_warps_issue_stalled_", "")
                                   .replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        e["top_stalls"] = [[n, round(v, 3)] for v, n in sorted(stalls, reverse=True)[:6]]
        summary.setdefault(name, []).append(e)
    out = {}
    for name, es in summary.items():
        e = es[-1]
        out[name] = {"duration_ms": e.get("duration", 0) * 1e3,
                     "dram_bytes_read": e.get("dram_read"), "dram_bytes_write": e.get("dram_write"),
                     "dram_pct": e.get("dram_pct"), "sm_pct": e.get("sm_pct"),
                     "warps_active_pct": e.get("warps_active_pct"), "warp_inst": e.get("warp_inst"),
                     "issue_active_pct": e.get("issue_active_pct"),
                     "threads_per_inst": e.get("threads_per_inst"), "regs": e.get("regs"),
                     "occ_limit_smem": e.get("occ_limit_smem"), "top_stalls": e["top_stalls"]}
        gbs = ((e.get("dram_read") or 0) + (e.get("dram_write") or 0)) / max(e.get("duration", 1e-9), 1e-12) / 1e9
        out[name]["dram_gbs"] = gbs
        print(f"== {name}: {out[name]['duration_ms']:.3f} ms  DRAM {gbs:.0f} GB/s "
              f"(r {(e.get('dram_read') or 0)/1e6:.1f} MB, w {(e.get('dram_write') or 0)/1e6:.1f} MB)  "
              f"sm {e.get('sm_pct', 0):.0f}%  warps {e.get('warps_active_pct', 0):.0f}%  "
              f"issue {e.get('issue_active_pct', 0):.0f}%  inst {e.get('warp_inst', 0)/1e6:.1f}M  "
              f"thr/inst {e.get('threads_per_inst', 0):.1f}")
        print("   stalls:", ", ".join(f"{n} {v}" for n, v in e["top_stalls"]))
        if a.lines:
            src = ncu_csv(["-i", a.report, "--page", "source", "--csv", "-k", f"regex:{name}",
                           "--print-source", "cuda,sass"])
            if len(src) > 3:
                h = src[2]
                try:
                    i_s, i_ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
                except ValueError:
                    continue
                lines = []
                for rr in src[3:]:
                    if len(rr) > max(i_s, i_ie) and rr[0]:
                        try:
                            lines.append((int(rr[i_s] or 0), int(rr[i_ie] or 0), rr[0], rr[1].strip()[:90]))
                        except ValueError:
                            pass
                ts = sum(l[0] for l in lines) or 1
                ti = sum(l[1] for l in lines) or 1
                for s_, ie, ln, txt in sorted(lines, reverse=True)[:a.lines]:
                    print(f"   L{ln:>4} stall {100*s_/ts:5.1f}% inst {100*ie/ti:5.1f}%  {txt}")
    if a.json:
        allj = {}
        if os.path.exists(a.json):
            with open(a.json) as f:
                allj = json.load(f)
        allj[a.workload] = out
        allj[a.workload]["_report"] = os.path.basename(a.report)
        with open(a.json, "w") as f:
            json.dump(allj, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
