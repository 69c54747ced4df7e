"""One line per ncu summary (tools/ncu_summary.py output): time, DRAM bytes
and fraction of the measured HBM peak, L1TEX busy, shared wavefronts and
conflict excess, warps active, issue activity, registers, block size."""
import re
import sys

SC = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}
for f in sys.argv[1:]:
    t = open(f).read()

    def g(k):
        m = re.search(re.escape(k) + r" = ([0-9.]+) ?(\S*)", t)
        return (float(m.group(1)) * SC.get(m.group(2), 1)) if m else float("nan")
    m = re.search(r"Kernel (.*)", t)
    if not m:
        print(f, "no kernel")
        continue
    d = g("gpu__time_duration.sum")
    dram = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
    wf, cf = g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"), g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    print(f"{f.split('/')[-1][:-4]:9s} {d * 1e3:7.3f} ms  DRAM {dram / 1e9:6.3f} GB ({dram / d / 1e9 / 6557.1:.2f} of peak)"
          f"  L1TEX {g('l1tex__throughput.avg.pct_of_peak_sustained_active'):.0f}%  smem wavefronts {wf / 1e6:.0f} M"
          f" (excess {cf / wf * 100:.0f}%)  warps {g('sm__warps_active.avg.pct_of_peak_sustained_active'):.0f}%"
          f"  issue {g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f}%"
          f"  fp64 {g('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.0f}%"
          f"  regs {g('launch__registers_per_thread'):.0f}  block {g('launch__block_size'):.0f}")
