"""Per-phase instruction / stall attribution of K1 from an ncu --set full
capture (--import-source on) and the library's line table.
usage: python scripts/k1_phase_profile.py REP.ncu-rep [LIB.so]
Helper lines (inlined device functions) are charged to the phase of the
nearest preceding k1_tile line in address order."""
import csv, io, os, re, subprocess, sys, tempfile
rep = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1606_05973_b200/libccl_b200.so"
src = open("paper_1606_05973_b200/csrc/ccl_kernels.cu").read().splitlines()
def line_of(pat):
    for i, l in enumerate(src, 1):
        if pat in l:
            return i
    raise SystemExit("marker not found: " + pat)
marks = [("P0 load+pack", line_of("// ---- P0: the pixels")), ("P0b holes+heads", line_of("// ---- P0b:")),
         ("P2a copies", line_of("// ---- P2a:")), ("P2b merges", line_of("// ---- P2b:")),
         ("P3 flatten", line_of("// ---- P3:")), ("P4 numbering", line_of("// ---- P4:")),
         ("P4c border", line_of("// ---- P4c:"))]
k1_lo = line_of("__device__ __forceinline__ void k1_tile(")
k1_hi = line_of("k_tile_local(const uint8_t *__restrict__ img, Geometry g")
def phase(ln):
    name = "prologue"
    for n, m in marks:
        if ln >= m:
            name = n
    return name
kern = sys.argv[3] if len(sys.argv) > 3 else "_ZN4cclb12k_tile_localILb0ELb0ELb0EEEvPKhNS_8GeometryENS_9WorkspaceEiiii"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "ccl_kernels", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
off2ph, cur, inside, ln = {}, "prologue", False, 0
for l in dis.splitlines():
    if l.startswith("//--------------------- .text."):
        inside = l.split(".text.")[1].split()[0] == kern
        continue
    if not inside:
        continue
    m = re.search(r'line (\d+)', l)
    if m and "//##" in l:
        ln = int(m.group(1))
        if k1_lo <= ln <= k1_hi:
            cur = phase(ln)
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m:
        off2ph[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:k_tile_local", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
iA, iI, iS = 0, hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = None
agg = {}
seen = set()
for r in rows[hi + 1:]:
    if len(r) <= iI or not r[0].startswith("0x"):
        continue
    a = int(r[0], 16)
    if a in seen:  # newer ncu lists the SASS page twice
        continue
    seen.add(a)
    base = a if base is None else base
    ph = off2ph.get(a - base, "?")
    n = int(r[iI] or 0); s = int(r[iS] or 0)
    e = agg.setdefault(ph, [0, 0]); e[0] += n; e[1] += s
tn = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
order = ["prologue"] + [n for n, _ in marks] + ["?"]
print(f"{'phase':18s} {'warp-inst':>10s} {'share':>6s} {'stall-samples':>13s}")
for k in order:
    if k in agg:
        print(f"{k:18s} {agg[k][0]/1e6:9.2f}M {100*agg[k][0]/tn:5.1f}% {100*agg[k][1]/ts:12.1f}%")
print(f"{'total':18s} {tn/1e6:9.2f}M")
