"""Summarise an ncu report: key metrics + stall-sample profile by SASS region."""
import csv, subprocess, sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active",
        "Achieved Occupancy", "Registers Per Thread", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Eligible Warps Per Scheduler", "Dynamic Shared Memory Per Block", "Grid Size"]
rows_ = list(csv.reader(raw.splitlines()))
h_ = rows_[0]
iN, iU, iV = h_.index("Metric Name"), h_.index("Metric Unit"), h_.index("Metric Value")
seen = set()
for row in rows_[1:]:
    if len(row) > iV and row[iN] in keys and row[iN] not in seen:
        seen.add(row[iN])
        print(f"{row[iN]:45s} {row[iV]:>20s} {row[iU]}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                      text=True).stdout
rows = list(csv.reader(sass.splitlines()))
hdr = rows[1]
data = rows[2:]
i_src = hdr.index("Source")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_ex = hdr.index("Instructions Executed")
tot = sum(int(r[i_s] or 0) for r in data)
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot)
for b in range(0, len(data), blk):
    s = sum(int(r[i_s] or 0) for r in data[b:b + blk])
    ex = sum(int(r[i_ex] or 0) for r in data[b:b + blk])
    if s / tot > 0.01:
        ops = [r[i_src].split()[1] if r[i_src].strip().startswith('@') else r[i_src].split()[0] for r in data[b:b + blk]]
        print(f"{b:5d} {100 * s / tot:5.1f}% exec {ex / 1e6:8.1f}M", Counter(ops).most_common(5))
