"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    name = r[ki].split("(")[0]
    agg.setdefault(name, []).append(float(r[mi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{k:55s} n={len(v):4d} mean_us={sum(v)/len(v)/1e3:9.2f} total_share={sum(v)/tot:6.3f}")
