"""Time compute(ns) on one problem under several layout choices (env switches), one process.

    python scripts/time_paths.py --kind 3dof --g 48 --k 1 --ns 3 --paths default NO_TSELL NO_BSR

Each path: create, then 2 warm-up computes and the median of 5 of the library's own sweep timing
(CUDA events around the sweep loop, fastilu_get_timings)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2506_05793_b200 as F
import problems as P

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="3dof")
ap.add_argument("--g", type=int, default=32)
ap.add_argument("--k", type=int, default=1)
ap.add_argument("--ns", type=int, default=3)
ap.add_argument("--paths", nargs="+", default=["default", "NO_TSELL", "NO_BSR"])
a = ap.parse_args()
A = P.make(a.kind, a.g)
for path in a.paths:
    env = {} if path == "default" else {f"FASTILU_{v}": "1" for v in path.split("+")}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    t0 = time.time()
    f = F.FastILU(A.row_ptr, A.col_idx, A.values, a.k)
    tc = time.time() - t0
    ms = []
    for it in range(7):
        f.compute(a.ns)
        if it >= 2:
            ms.append(f.timings()["sweeps_ms"] / max(a.ns, 1))
    print(json.dumps({"kind": a.kind, "g": a.g, "k": a.k, "path": path, "info": f.info(),
                      "create_s": round(tc, 2), "ms_per_sweep": float(np.median(ms))}))
    f.close()
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
