"""Instruction / stall shares of a kernel between its barriers (BAR.SYNC):
usage: python scripts/ncu_segments.py REPORT KERNEL_REGEX NUNITS [dump_segment]"""
import csv, io, subprocess, sys
rep, k, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
dump = int(sys.argv[4]) if len(sys.argv) > 4 else -1
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; ie = h.index("Instructions Executed"); st = h.index("Warp Stall Sampling (All Samples)")
seg = 0; acc = {}; accs = {}; tot = 0; tots = 0
for r in rows[2:]:
    if len(r) <= ie or not r[0].startswith("0x"):
        continue
    n = int(r[ie] or 0); s = int(r[st] or 0); tot += n; tots += s
    acc[seg] = acc.get(seg, 0) + n; accs[seg] = accs.get(seg, 0) + s
    if seg == dump and n > 0:
        print(f"{n / units:8.1f} {s:6d} {r[1].strip()}")
    if "BAR.SYNC" in r[1] or "BAR.RED" in r[1]:
        seg += 1
for g in sorted(acc):
    print(f"seg {g}: inst {100 * acc[g] / tot:5.1f}% ({acc[g] / units:7.0f}/unit)  stall {100 * accs[g] / max(tots, 1):5.1f}%")
print(f"total {tot / 1e6:.1f}M warp-inst, {tot / units:.0f}/unit")
