"""Print the headline ncu 'details' metrics of every kernel in a report."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Block Limit Shared Mem",
        "Block Limit Registers", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "Eligible Warps Per Scheduler",
        "No Eligible", "Dynamic Shared Memory Per Block"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
cur = None
for r in rows[1:]:
    if r[ix["ID"]] != cur:
        cur = r[ix["ID"]]
        print(f"== [{cur}] {r[ix['Kernel Name']][:110]}")
        seen = set()
    m = r[ix["Metric Name"]]
    if m in WANT and m not in seen:
        seen.add(m)
        print(f"   {m:40s} {r[ix['Metric Value']]:>14s} {r[ix['Metric Unit']]}")
