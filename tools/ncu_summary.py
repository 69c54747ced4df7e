"""Text summary of an ncu --set full report: duration, DRAM bytes, L1TEX
throughput, shared-memory wavefronts and conflict excess, warps active,
occupancy limits, issue activity, then the top source lines by conflicts
and by stall samples (tools/ncu_src_conflicts.py)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "l1tex__throughput.avg.pct_of_peak_sustained_active",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__block_size",
     "launch__grid_size"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
for r in rows[2:]:
    print("Kernel", r[h.index("Kernel Name")])
    for k in M:
        if k in h:
            i = h.index(k)
            print(f"   {k} = {r[i]} {units[i]}")
print(subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_src_conflicts.py"), rep, "8"],
                     capture_output=True, text=True).stdout)
