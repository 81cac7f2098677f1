"""Print the headline counters of every kernel in an ncu report (ncu -i ... --page details --csv)."""
import csv
import subprocess
import sys

WANT = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp",
        "Branch Efficiency", "DRAM Throughput", "L2 Hit Rate", "Memory Throughput", "Local Memory Spilling Requests"]

for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, ni, ui, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    seen = {}
    for r in rows[1:]:
        if len(r) > vi and r[ni] in WANT:
            seen.setdefault((r[ii], r[ki]), {})[r[ni]] = f"{r[vi]} {r[ui]}".strip()
    for (i, k), m in seen.items():
        print(f"[{path}] #{i} {k[:70]}")
        for name in WANT:
            if name in m:
                print(f"    {name:42s} {m[name]}")
