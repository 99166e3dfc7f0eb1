"""One FastILU step (compute + apply) on a workload, for ncu captures:
    ncu ... python scripts/profile_step.py --workload c3a_27pt_128_ilu1 [--steps 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_05793_b200 as F  # noqa: E402
import problems as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3a_27pt_128_ilu1")
ap.add_argument("--steps", type=int, default=1)
args = ap.parse_args()
kind, g, k, ns, nt = P.WORKLOADS[args.workload]
a = P.make(kind, g)
f = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
b = torch.tensor(P.rhs_positive(a.n), device="cuda")
x = torch.empty_like(b)
for _ in range(args.steps):
    f.compute(ns)
    f.apply(b, x, nt)
torch.cuda.synchronize()
print("done", f.timings())
