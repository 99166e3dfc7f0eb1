"""Summarise one round's ncu evidence into profiles/ (committed).

    python scripts/make_profile_summary.py --tag r1 --workload c4_27pt_256_ilu1 \
        --launches gpurun_out/X_launches.csv --report gpurun_out/X.ncu-rep

Writes profiles/<tag>_<workload>_launches.md (per-kernel launch counts, device time and share of
the step from the `--metrics gpu__time_duration.sum --clock-control none` launch list) and
profiles/<tag>_<workload>_ncu.md (per-kernel Speed-of-Light metrics and DRAM bytes from the
`--set full` capture), and merges the sweep kernel's per-launch DRAM traffic into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("fastilu::", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
             "ms": 1.0, "second": 1e3, "s": 1e3}
    agg = {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        k = short(r[ki])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    return agg


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = r[0]
    ki, mi, vi, ui, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                   "Metric Unit", "ID"))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh = rr[0]
    units = rr[1]
    cols = {m: rh.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                      "gpu__time_duration.sum")}
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
            "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    kern = {}
    for i, row in enumerate(rr[2:]):
        d = {m: float(row[c].replace(",", "")) * mult.get(units[c], 1) for m, c in cols.items()}
        kern[str(i)] = (short(row[rh.index("Kernel Name")]), d)
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Achieved Occupancy", "Registers Per Thread", "Executed Ipc Active",
            "Issue Slots Busy", "Eligible Warps Per Scheduler", "Grid Size", "Block Size"]
    met = {}
    for row in r[1:]:
        if row[mi] in want:
            met.setdefault(row[idi], {})[row[mi]] = f"{row[vi]} {row[ui]}".strip()
    return kern, met


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    base = os.path.join(ROOT, "profiles", f"{a.tag}_{a.workload}")
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v[1] for v in agg.values())
        with open(base + "_launches.md", "w") as f:
            f.write(f"# {a.tag} launch list, {a.workload} (one step: compute + apply)\n\n")
            f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over "
                    "`scripts/profile_step.py` (cold-cache, serialised: compare shares, not "
                    "absolutes).\n\n")
            if a.note:
                f.write(a.note + "\n\n")
            f.write("| kernel | launches | device time (ms) | share |\n|---|---|---|---|\n")
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"| `{k}` | {v[0]} | {v[1]:.3f} | {100 * v[1] / tot:.1f}% |\n")
            f.write(f"| total | {sum(v[0] for v in agg.values())} | {tot:.3f} | 100% |\n")
    if a.report:
        kern, met = details(a.report)
        with open(base + "_ncu.md", "w") as f:
            f.write(f"# {a.tag} ncu --set full, {a.workload}\n\n")
            if a.note:
                f.write(a.note + "\n\n")
            for i, (name, d) in kern.items():
                f.write(f"## launch {i}: `{name}`\n\n")
                f.write(f"- DRAM read {d['dram__bytes_read.sum'] / 1e9:.3f} GB, write "
                        f"{d['dram__bytes_write.sum'] / 1e9:.3f} GB, duration "
                        f"{d['gpu__time_duration.sum']:.3f} ms\n")
                for k, v in met.get(i, {}).items():
                    f.write(f"- {k}: {v}\n")
                f.write("\n")
        # the dominant (full) sweep kernel, not sweep 1's variants (_init / _first)
        sweeps = [d for name, d in kern.values()
                  if "sweep" in name and not name.endswith(("_init", "_first"))]
        if sweeps:
            tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
            cur = json.load(open(tp)) if os.path.exists(tp) else {}
            d = sweeps[0]
            cur[a.workload] = {"sweep_dram_bytes": d["dram__bytes_read.sum"] +
                               d["dram__bytes_write.sum"],
                               "sweep_dram_read": d["dram__bytes_read.sum"],
                               "sweep_dram_write": d["dram__bytes_write.sum"],
                               "source": os.path.basename(base) + "_ncu.md"}
            json.dump(cur, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main()
