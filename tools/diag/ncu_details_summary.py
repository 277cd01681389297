"""Headline metrics of an ncu --page details CSV (exported on the GPU box by
tools/diag/ncu_captures.sh) plus the SASS stall aggregation of its source
page: ncu_details_summary.py NAME "note" > profiles/r02_ncu_NAME.txt"""
import csv
import os
import subprocess
import sys

name, note = sys.argv[1], sys.argv[2]
d = os.path.join("gpurun_out", "ncu")
rows = list(csv.reader(open(os.path.join(d, f"{name}_details.csv"))))
hdr = rows[0]
kern = rows[1][hdr.index("Kernel Name")] if len(rows) > 1 else "?"
want = ["Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Block Size", "Grid Size", "Achieved Occupancy",
        "Theoretical Occupancy", "Executed Instructions", "Eligible Warps Per Scheduler"]
print(f"# ncu --set full --clock-control none: {note}")
print(f"kernel: {kern.split('(')[0]}")
seen = set()
for r in rows[1:]:
    if len(r) > 14 and r[12] in want and r[12] not in seen:
        seen.add(r[12])
        print(f"  {r[12]:34s} {r[14]} {r[13]}")
for r in rows[1:]:
    if len(r) > 17 and r[11] in ("Compute Workload Analysis", "GPU Speed Of Light Throughput") and r[15] == "" and "pipeline" in r[17][:200].lower():
        print("  note:", r[17][:300])
        break
src = os.path.join(d, f"{name}_source.csv.gz")
if os.path.exists(src):
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "sass_hot.py"), src, "60"],
                         capture_output=True, text=True).stdout
    print("\n## SASS warp-stall samples (tools/diag/sass_hot.py)")
    print(out)
