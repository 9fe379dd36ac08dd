"""Per-instruction stall-sample share of the FIRST kernel in an ncu source-page csv."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
# the file may hold several kernels: take the block after the first header only
h = rows[1]
ai, si, ni, ei = (h.index(x) for x in ("Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"))
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) <= ei:
        continue
    try:
        n, e = float(r[ni] or 0), float(r[ei] or 0)
    except ValueError:
        continue
    data.append((int(r[ai], 16), n, e, r[si]))
data.sort()
tot = sum(d[1] for d in data)
tote = sum(d[2] for d in data)
print("samples", tot, "warp-instr", tote)
base = data[0][0] if data else 0
for a, n, e, s in data:
    if tot and n / tot > thr:
        print(f"{a - base:06x} {n / tot * 100:5.1f}% exec={e:9.0f} {s[:100]}")
