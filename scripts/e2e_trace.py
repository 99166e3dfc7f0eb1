"""Timeline of the e2e step (fastilu_solve_host: host values + b in, x out) with FASTILU_TRACE=1:
when each value chunk and b land on the device, when the compute ends, the apply starts/ends and
the D2H of x ends (ms from the compute's start; CUDA events).
    FASTILU_TRACE=1 python scripts/e2e_trace.py [--workload c4_27pt_256_ilu1] [--reps 3]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_05793_b200 as F  # noqa: E402
import problems as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4_27pt_256_ilu1")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
kind, g, k, ns, nt = P.WORKLOADS[args.workload]
a = P.make(kind, g)
f = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
av = torch.from_numpy(a.values).pin_memory().numpy()
bh = torch.from_numpy(P.rhs_positive(a.n)).pin_memory().numpy()
xh = torch.empty(a.n, dtype=torch.float64).pin_memory().numpy()
for r in range(args.reps + 1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f.solve_host(av, ns, bh, nt, out=xh)
    print(f"rep {r}: wall {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
