"""Print selected raw metrics of an ncu report: python scripts/ncu_raw.py REP [metric-substr ...]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2:] or ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "lts__t_sectors.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
                        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                        "smsp__issue_active.avg.pct_of_peak_sustained_active",
                        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                        "launch__registers_per_thread", "launch__occupancy_limit"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
for v in rows[2:]:
    for i, n in enumerate(h):
        if any(w in n for w in want):
            print(f"{n:70s} {u[i]:>12s} {v[i]}")
    print()
