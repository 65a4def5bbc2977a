"""Key raw metrics per kernel from an ncu report: python scripts/ncu_raw.py <rep> [kernel-regex]."""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
kre = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
pat = re.compile(r"(Kernel Name|gpu__time_duration.sum|dram__bytes_(read|write).sum$|"
                 r"l1tex__data_pipe_lsu_wavefronts_mem_shared.sum$|l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$|"
                 r"l1tex__throughput.avg.pct_of_peak_sustained_active|sm__warps_active.avg.pct_of_peak_sustained_active|"
                 r"launch__registers_per_thread$|launch__grid_size|launch__block_size|smsp__inst_executed.sum$|"
                 r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio|smsp__issue_active.avg.pct|"
                 r"l1tex__t_sectors_pipe_lsu_mem_global_op_(ld|st).sum$|lts__t_sectors_srcunit_tex_op_read.sum$|"
                 r"dram__throughput.avg.pct_of_peak_sustained_elapsed|launch__occupancy_limit_(registers|shared_mem))")
idx = [i for i, x in enumerate(h) if pat.search(x)]
for r in rows[2:]:
    if kre and not kre.search(r[h.index("Kernel Name")]):
        continue
    print("---")
    for i in idx:
        try:
            if "stalled" in h[i] and float(r[i]) < 0.3:
                continue
        except ValueError:
            pass
        print(" ", h[i].replace("smsp__average_warps_issue_stalled_", "stall_").replace("_per_issue_active.ratio", ""), r[i])
