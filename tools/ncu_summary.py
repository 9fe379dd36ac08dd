"""Key metrics per profiled kernel from an ncu report (details page)."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
cur = None
for row in r[1:]:
    if row[mi] in WANT:
        k = row[ii] + " " + row[ki].split("(")[0][:40]
        if k != cur:
            print("==", k)
            cur = k
        print(f"    {row[mi]:38s} {row[vi]:>12s} {row[ui]}")
