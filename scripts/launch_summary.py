"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel launches, total / average time and share of the step.
usage: python scripts/launch_summary.py LAUNCHES.csv > profiles/rNN_launches_summary.txt"""
import csv, io, re, sys
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
agg = {}
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"<.*", "", r["Kernel Name"].split("(")[0].split("::")[-1]).replace("void ", "").strip()
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1000 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000)
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + us)
tot = sum(t for _, t in agg.values()) or 1.0
print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches) of")
print("  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity  (C4 21600x21600)")
print(f"{'kernel':14s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:14s} {n:8d} {t:10.1f} {t / n:9.1f} {100 * t / tot:5.1f}%")
