"""Summarise scripts/live_traffic.sh output (ncu --cache-control none: DRAM
bytes of each kernel with the caches as the pipeline leaves them).
usage: python scripts/live_summary.py gpurun_out/live_TAG.csv > profiles/rNN_live_traffic.txt"""
import csv, io, re, sys
from collections import defaultdict
L = open(sys.argv[1]).read().splitlines()
i = next(i for i, l in enumerate(L) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(L[i:]))))
per = defaultdict(lambda: defaultdict(list))
order = []
for r in rows:
    name = re.sub(r"<.*", "", r["Kernel Name"].split("(")[0]).replace("void ", "").strip()
    if name not in order:
        order.append(name)
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1}.get(u, 1)
    per[name][r["Metric Name"]].append(v)
print("kernel          us      DRAM read MB  DRAM write MB  L2 hit %   (ncu --cache-control none, averaged over launches)")
for n in order:
    m = per[n]
    avg = lambda k: sum(m[k]) / len(m[k]) if m[k] else float("nan")
    print(f"{n:14s} {avg('gpu__time_duration.sum'):7.1f} {avg('dram__bytes_read.sum')/1e6:12.1f} {avg('dram__bytes_write.sum')/1e6:14.1f} {avg('lts__t_sector_hit_rate.pct'):9.1f}")
