"""A short GMRES(60) run on the config-5 matrix, for ncu launch lists of the Krylov kernels:
    ncu --metrics gpu__time_duration.sum ... python scripts/profile_gmres.py [--g 256] [--iters 60]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_05793_b200 as F  # noqa: E402
import problems as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--g", type=int, default=256)
ap.add_argument("--iters", type=int, default=60)
ap.add_argument("--ntri", type=int, default=1)
args = ap.parse_args()
a = P.make("aniso7pt", args.g)
f = F.FastILU(a.row_ptr, a.col_idx, a.values, 0)
f.compute(2)
b = torch.tensor(P.rhs_positive(a.n), device="cuda")
x = torch.zeros_like(b)
it, rr = f.gmres(b, x, restart=60, rtol=1e-12, max_iters=args.iters, ntrisweeps=args.ntri)
torch.cuda.synchronize()
print("iterations", it, "relres", rr)
