"""Warp-stall breakdown (share of samples, top SASS opcodes per reason) of one kernel in an ncu
report:  python scripts/ncu_stalls.py REP KERNEL_REGEX"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h, data = rows[hi], rows[hi + 1:]
ix = {n: i for i, n in enumerate(h)}
cols = [c for c in h if c.startswith("stall_") and "(" not in c]
tot = {c: 0.0 for c in cols}
byop = {}
ninst = 0
for r in data:
    if len(r) < len(h):
        continue
    src = r[ix["Source"]].split()
    if not src or src[0] == "Source":  # repeated header rows (one per function)
        continue
    ninst += 1
    op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
    for c in cols:
        v = float(r[ix[c]] or 0)
        tot[c] += v
        byop.setdefault(op, {}).setdefault(c, 0.0)
        byop[op][c] += v
T = sum(tot.values()) or 1.0
print(f"{kern}: {ninst} SASS instructions, {int(T)} stall samples")
for c in sorted(cols, key=lambda c: -tot[c])[:12]:
    top = sorted(((v.get(c, 0.0), k) for k, v in byop.items()), reverse=True)[:5]
    print(f"  {c:26s} {100 * tot[c] / T:5.1f}%  " + ", ".join(f"{k} {100 * x / T:.1f}" for x, k in top))
