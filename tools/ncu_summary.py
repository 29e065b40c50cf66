"""Print key metrics of every kernel in an .ncu-rep (details page)."""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Avg. Active Threads Per Warp",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Dynamic Shared Memory Per Block", "Block Size", "Grid Size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, ni, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
idi = hdr.index("ID")
cur = None
for r in rows[1:]:
    if r[idi] != cur:
        cur = r[idi]
        print(f"== [{cur}] {r[ki][:100]}")
    if r[ni] in KEYS:
        print(f"   {r[ni]:40s} {r[vi]:>16s} {r[ui]}")
