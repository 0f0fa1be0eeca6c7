"""One line per kernel of an ncu report: time, issue, warps, pipes, instructions, DRAM bytes, registers.
usage: python tools/ncu_brief.py REPORT"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
K = [("time_ms", "gpu__time_duration.sum"), ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
     ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
     ("fp64%", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
     ("alu%", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
     ("lsu%", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
     ("Minst", "smsp__inst_executed.sum"), ("rdMB", "dram__bytes_read.sum"), ("wrMB", "dram__bytes_write.sum"),
     ("regs", "launch__registers_per_thread")]
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0]
    vals = []
    for lab, k in K:
        if k in h:
            v = float(r[h.index(k)].replace(",", "") or 0)
            if lab == "Minst":
                v /= 1e6
            vals.append(f"{lab}={v:.4g}")
    print(f"{name[:40]:40s} " + " ".join(vals))
