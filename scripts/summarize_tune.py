"""python scripts/summarize_tune.py LOG"""
import json
import sys

cur = None
for l in open(sys.argv[1]):
    if l.startswith("=="):
        cur = l.strip()
    elif l.startswith("{"):
        d = json.loads(l)
        ns = d["config"]["nsweeps"]
        print(f"{cur:55s} sweep {d['sweep_ms']/ns:7.3f} ms  frac {d['roofline']['frac']:.3f}  "
              f"{d.get('kernel_config','')[:80]}")
