"""BASELINE config 5: FastILU-preconditioned GMRES(60) on the anisotropic 7-point Laplacian.

    python scripts/gmres_bench.py [--g 256] [--nsweeps 2] [--ntri 1 2 3 4 5] [--oracle]

Arm A (GPU): FastILU(0) with `nsweeps` sweeps, `ntri` Jacobi sweeps per apply, GMRES(60) to
1e-6 relative residual, x0 = 0, b = A x_true with x_true ~ U[0,1).  Reports
inner iterations and device time-to-solution (compute + GMRES).  --oracle adds arm C: the CPU
oracle's exact ILU(0) with exact substitution (iterations and CPU time), one JSON line each.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_05793_b200 as F  # noqa: E402
import problems as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--g", type=int, default=256)
ap.add_argument("--nsweeps", type=int, default=2)
ap.add_argument("--ntri", type=int, nargs="+", default=[1, 2, 3, 4, 5])
ap.add_argument("--oracle", action="store_true")
args = ap.parse_args()
a = P.aniso3d_7pt(args.g)
xt = P.x_true(a.n)
rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
b = np.bincount(rows, weights=a.values * xt[a.col_idx], minlength=a.n)  # b = A x_true
f = F.FastILU(a.row_ptr, a.col_idx, a.values, 0)
tb = torch.tensor(b, device="cuda")
tx = torch.zeros_like(tb)
for nt in args.ntri:
    f.compute(args.nsweeps)  # warm-up (JIT, caches)
    f.gmres(tb, tx, 60, 1e-6, 5000, nt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f.compute(args.nsweeps)
    it, rr = f.gmres(tb, tx, 60, 1e-6, 5000, nt)
    e1.record()
    torch.cuda.synchronize()
    err = float(np.abs(tx.cpu().numpy() - xt).max())
    print(json.dumps({"config": "c5", "arm": "A (GPU FastILU)", "g": args.g, "n": a.n,
                      "nsweeps": args.nsweeps, "ntri": nt, "iterations": it, "relres": rr,
                      "time_to_solution_ms": e0.elapsed_time(e1), "max_err_vs_x_true": err,
                      "kernel_config": f.info()}), flush=True)
if args.oracle:
    import oracle
    t0 = time.perf_counter()
    fe = oracle.compute(a, 0, 0)
    fe.vals = oracle.exact_ilu(fe.pattern, fe.ahat)
    t1 = time.perf_counter()
    x, it, rr = oracle.gmres(a, b, oracle.exact_preconditioner(fe), 60, 1e-6, 5000)
    t2 = time.perf_counter()
    print(json.dumps({"config": "c5", "arm": "C (CPU oracle exact ILU(0) + substitution)",
                      "g": args.g, "n": a.n, "iterations": it, "relres": rr,
                      "factor_s": t1 - t0, "gmres_s": t2 - t1, "cores": 1}), flush=True)
