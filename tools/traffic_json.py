"""profiles/traffic.json from the round's ncu captures: the timed blend's DRAM
bytes per launch, issue-slot and pipe utilisation (ncu --set full), and the
DRAM bytes of one whole frame (every kernel of the frame, from the launch
list; cold-cache and serialised, so an upper bound on the pipelined traffic).

    python tools/traffic_json.py LAUNCHES.csv BLEND.ncu-rep > profiles/traffic.json
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

PER_FRAME = {"k_count_scan": 3, "k_onesweep": 5}   # launches per frame (tile grid <= 256 rows)
FRAME_KERNELS = ("k_zero", "k_cull", "k_count_scan", "k_cull_emit", "k_slice", "k_vis_emit", "k_sort_hist", "k_onesweep",
                 "k_bin_count", "k_bin_offsets", "k_row_items", "k_row_scan", "k_row_count", "k_tile_scan",
                 "k_row_scatter", "k_blend_wi")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, name = defaultdict(dict), {}
    for r in rows[1:]:
        try:
            per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("fdgs::", "").split("<")[0]
    agg = defaultdict(list)
    for i, m in per.items():
        agg[name[i]].append(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
    return {k: sum(v) / len(v) for k, v in agg.items()}


def blend_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    m = dict(zip(h, v))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    u = dict(zip(h, units))

    def nbytes(key):
        return float(m[key].replace(",", "")) * scale.get(u.get(key, "byte"), 1)

    def f(key):
        return round(float(m[key].replace(",", "")) / 100.0, 4) if key in m else None
    return {"issue_slots_busy": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "pipes": {p: f(f"sm__inst_executed_pipe_{p}.avg.pct_of_peak_sustained_active")
                      for p in ("fma", "alu", "xu", "lsu", "fmaheavy")},
            "dram": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")}


def main():
    dram = launches(sys.argv[1])
    bm = blend_metrics(sys.argv[2])
    frame = sum(dram.get(k, 0.0) * PER_FRAME.get(k, 1) for k in FRAME_KERNELS)
    out = {"k_blend_wi": int(bm["dram"]),
           "_src": "ncu --set full of k_blend_wi (one C3 frame of tools/blend_ab.py): dram__bytes_read.sum + "
                   "dram__bytes_write.sum per launch",
           "k_blend_wi_issue_slots_busy": bm["issue_slots_busy"],
           "k_blend_wi_pipes": bm["pipes"],
           "_src_issue": "same capture: sm__inst_issued / sm__inst_executed_pipe_* pct_of_peak_sustained_active",
           "frame_dram_bytes": int(frame),
           "_src_frame": "ncu launch list of bench.py (C3, working sets): mean DRAM bytes per launch of each of the "
                         "frame's kernels x its launches per frame, summed (cold cache, serialised)",
           "per_kernel_dram_bytes": {k: int(v) for k, v in sorted(dram.items()) if k in FRAME_KERNELS}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
