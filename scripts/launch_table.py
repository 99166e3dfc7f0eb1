"""Per-kernel totals of an ncu launch list with time and DRAM bytes (markdown table):
    python scripts/launch_table.py LAUNCHES.csv [title]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
data = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        h = {n: i for i, n in enumerate(r)}
        continue
    if not h or len(r) < len(h):
        continue
    name = r[h["Kernel Name"]].split("(")[0].replace("void ", "").replace("fastilu::", "")
    m, v = r[h["Metric Name"]], float(r[h["Metric Value"]].replace(",", ""))
    d = data[name]
    if m == "gpu__time_duration.sum":
        d[0] += 1
        d[1] += v
    elif m == "dram__bytes_read.sum":
        d[2] += v
    elif m == "dram__bytes_write.sum":
        d[3] += v
tot = sum(d[1] for d in data.values())
if len(sys.argv) > 2:
    print(f"# {sys.argv[2]}\n")
print("| kernel | launches | time (ms) | share | DRAM GB | GB/s |")
print("|---|---|---|---|---|---|")
for k, (c, t, rd, wr) in sorted(data.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {c} | {t / 1e6:.2f} | {t / tot * 100:.1f}% | {(rd + wr) / 1e9:.2f} | "
          f"{(rd + wr) / t if t else 0:.0f} |")
print(f"| total | | {tot / 1e6:.2f} | 100% | | |")
