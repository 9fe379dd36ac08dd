"""Per-kernel DRAM bytes, duration and achieved GB/s from an ncu --csv metrics log."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, ui, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    key = (r[ii], r[ki].split("(")[0])
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
             "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
    per.setdefault(key, {})[r[mi]] = v * scale.get(u, 1)
agg = collections.OrderedDict()
for (i, k), m in per.items():
    a = agg.setdefault(k, [0, 0.0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[3] += m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0)
    a[4] += m.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", 0)
print(f"{'kernel':28s} {'n':>3s} {'us':>8s} {'DRAM MB':>9s} {'GB/s':>8s} {'dram%':>6s} {'sm%':>6s}")
for k, (n, t, b, dp, sp) in agg.items():
    print(f"{k:28s} {n:3d} {t / n * 1e6:8.2f} {b / n / 1e6:9.2f} {b / t / 1e9:8.1f} {dp / n:6.1f} {sp / n:6.1f}")
