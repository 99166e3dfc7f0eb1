"""Summarise an ncu report: python scripts/ncu_summary.py REPORT.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr = r[0]
ki, mi, vi, ui, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                               "Metric Unit", "ID"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Eligible Warps Per Scheduler", "Grid Size", "Block Size"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
rh = rr[0]
dr = rh.index("dram__bytes_read.sum")
dw = rh.index("dram__bytes_write.sum")
rk = rh.index("Kernel Name")
traffic = {}
for i, row in enumerate(rr[2:]):
    traffic[str(i)] = (row[rk], row[dr], rr[1][dr], row[dw], rr[1][dw])
cur = None
for row in r[1:]:
    if pat and not pat.search(row[ki]):
        continue
    if row[idi] != cur:
        cur = row[idi]
        t = traffic.get(cur)
        print(f"--- {cur} {row[ki][:70]}  dram read {t[1]} {t[2]} write {t[3]} {t[4]}")
    if row[mi] in want:
        print(f"    {row[mi]:32s} {row[vi]} {row[ui]}")
