"""Summarize bench JSON lines: python scripts/summarize.py FILE..."""
import json
import sys

for fn in sys.argv[1:]:
    for l in open(fn):
        l = l.strip()
        if not l.startswith("{"):
            if l:
                print("  ", l[:200])
            continue
        d = json.loads(l)
        c = d.get("config", {})
        if "sweep_ms" not in d:
            print(json.dumps(d)[:400])
            continue
        ns = c.get("nsweeps", 1)
        print(f"{c.get('workload')}: ms/step {d['ms_per_step']:.2f} | sweep {d['sweep_ms']/ns:.3f} ms/sweep "
              f"{d['sweep_nnz_updates_per_s']:.3g} upd/s roof {d['roofline']['achieved']:.0f} GB/s "
              f"({d['roofline']['frac']:.3f}) | init {d['init_ms']:.3f} apply {d['apply_ms']:.3f} "
              f"tri {d['trisolve_gbs'] or 0:.0f} GB/s | composite {d['composite_gbs']:.0f} GB/s | "
              f"clk {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')} | e2e "
              f"{(d.get('e2e') or {}).get('value', 0):.3g}")
