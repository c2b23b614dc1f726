"""Key metrics per captured kernel of an ncu --set full report:
python tools/ncu_summary.py report.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
M = [("time", "gpu__time_duration.sum"), ("dram_rd", "dram__bytes_read.sum"), ("dram_wr", "dram__bytes_write.sum"),
     ("occ%", "sm__warps_active.avg.pct_of_peak_sustained_active"), ("regs", "launch__registers_per_thread"),
     ("sm%", "sm__throughput.avg.pct_of_peak_sustained_elapsed"), ("l1%", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
     ("l2%", "lts__throughput.avg.pct_of_peak_sustained_elapsed"), ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
     ("fma%", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
     ("ldsect", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"), ("shwf", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
     ("bankc", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
     ("st_mio", "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"),
     ("st_lsb", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
     ("st_bar", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"),
     ("st_ssb", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio")]
idx = [(n, h.index(k)) for n, k in M if k in h]
print("kernel".ljust(34) + "".join(n.rjust(10) for n, _ in idx))
print("".ljust(34) + "".join(units[i][:9].rjust(10) for _, i in idx))
for r in rows[2:]:
    name = r[h.index("Kernel Name")].replace("mgb::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    print(name[:33].ljust(34) + "".join(r[i][:9].rjust(10) for _, i in idx))
