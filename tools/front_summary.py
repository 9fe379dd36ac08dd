"""Per-kernel summary of an ncu --metrics launch list (csv): launches, mean
duration, share of the summed duration, warp instructions per launch, active
warps and DRAM bytes per launch.  python tools/front_summary.py FILE.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ii = h.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[1:]:
    try:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "")[:40]
agg = defaultdict(lambda: defaultdict(float))
for i, m in per.items():
    a = agg[names[i]]
    a["n"] += 1
    for k, v in m.items():
        a[k] += v
tot = sum(a.get("gpu__time_duration.sum", 0) for a in agg.values())
print(f"{'kernel':42s} {'n':>4s} {'us':>8s} {'share':>6s} {'Minst':>8s} {'warps%':>7s} {'MB dram':>8s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0)):
    n = a["n"]
    d = a.get("gpu__time_duration.sum", 0)
    print(f"{k:42s} {int(n):4d} {d / n / 1e3:8.2f} {d / tot:6.3f} {a.get('smsp__inst_executed.sum', 0) / n / 1e6:8.3f} "
          f"{a.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0) / n:7.1f} "
          f"{(a.get('dram__bytes_read.sum', 0) + a.get('dram__bytes_write.sum', 0)) / n / 1e6:8.2f}")
