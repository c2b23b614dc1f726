"""Key ncu details per profiled launch (duration, occupancy, throughput, stall breakdown)."""
import csv, subprocess, sys
rep = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
want = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Compute (SM) Throughput",
        "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Block Limit Registers", "Block Limit Shared Mem",
        "Waves Per SM", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
cur = None
for r in rows[1:]:
    if len(r) != len(h):
        continue
    if flt and flt not in r[ki]:
        continue
    k = (r[ii], r[ki][:50])
    if k != cur:
        cur = k
        print("==", k)
    if r[mi] in want or "Stall" in r[mi] or "stall" in r[mi]:
        print("   ", r[mi], r[vi], r[ui])
