"""Top SASS lines of an `ncu --page source --csv --print-source sass` dump by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ai, si, ni, ei = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
def num(x):
    try:
        return float(x)
    except ValueError:
        return None
data = [r for r in rows[2:] if len(r) > ei and num(r[ni] or 0) is not None]
tot = sum(float(r[ni] or 0) for r in data)
tot_e = sum(float(r[ei] or 0) for r in data)
print(f"total samples {tot:.0f}, warp-instructions executed {tot_e:.3g}")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 40
if len(sys.argv) > 3 and sys.argv[3] == "exec":
    data.sort(key=lambda r: -float(r[ei] or 0))
else:
    data.sort(key=lambda r: -float(r[ni] or 0))
for r in data[:k]:
    print(f"{r[ai]:>6s} {float(r[ni] or 0)/tot*100:5.1f}% exec={float(r[ei] or 0):10.0f}  {r[si][:90]}")
