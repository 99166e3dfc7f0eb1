"""Time compute(ns) on one problem under several layout choices (env switches), one process.

    python scripts/time_paths.py --kind 3dof --g 48 --k 1 --ns 3 \
        --paths default NO_TSELL BSR_SMEM_KB=0+BSR_MINB=4

A path is "default" or '+'-joined FASTILU_* settings (NAME or NAME=value).  All handles are
created first; then --rounds rounds visit the paths in turn (interleaved, so clock or thermal
drift hits every path alike), each timing 5 computes with the library's own sweep timing (CUDA
events around the sweep loop, fastilu_get_timings).  Reports the best round's median per path."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2506_05793_b200 as F  # noqa: E402
import problems as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="3dof")
ap.add_argument("--g", type=int, default=32)
ap.add_argument("--k", type=int, default=1)
ap.add_argument("--ns", type=int, default=3)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--paths", nargs="+", default=["default", "NO_TSELL", "NO_BSR"])
a = ap.parse_args()
A = P.make(a.kind, a.g)
handles = []
for path in a.paths:
    env = {} if path == "default" else dict(
        (f"FASTILU_{v.split('=')[0]}", v.split("=")[1] if "=" in v else "1")
        for v in path.split("+"))
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    t0 = time.time()
    f = F.FastILU(A.row_ptr, A.col_idx, A.values, a.k)
    handles.append((path, f, time.time() - t0, []))
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
for r in range(a.rounds):
    for path, f, tc, meds in handles:
        ms = []
        for it in range(6):
            f.compute(a.ns)
            if it >= 1:
                ms.append(f.timings()["sweeps_ms"] / max(a.ns, 1))
        meds.append(float(np.median(ms)))
for path, f, tc, meds in handles:
    print(json.dumps({"kind": a.kind, "g": a.g, "k": a.k, "path": path, "info": f.info(),
                      "create_s": round(tc, 2), "ms_per_sweep": min(meds),
                      "rounds": [round(m, 4) for m in meds]}))
    f.close()
