"""Per-source-line instruction and stall shares of one kernel in an ncu report.
usage: python scripts/ncu_lines.py REPORT KERNEL_REGEX [min_pct]"""
import csv, io, subprocess, sys
rep, k = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if "Instructions Executed" in r)
start = rows.index(h) + 1
i_s, i_ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
L = []
for r in rows[start:]:
    if not r or not r[0].isdigit():
        if r and r[0] == "File Path": break
        continue
    try:
        L.append((int(r[0]), int(r[i_ie] or 0), int(r[i_s] or 0), r[1].strip()[:100]))
    except (ValueError, IndexError):
        pass
ti = sum(l[1] for l in L) or 1
ts = sum(l[2] for l in L) or 1
print(f"total warp inst {ti/1e6:.1f}M, stall samples {ts}")
for ln, ie, s, t in sorted(L):
    if 100 * ie / ti >= thr or 100 * s / ts >= thr:
        print(f"L{ln:>4} inst {100*ie/ti:5.1f}% stall {100*s/ts:5.1f}%  {t}")
