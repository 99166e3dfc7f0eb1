"""Small ragged cases of every default-path kernel, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): the staged TMA sweep (27-pt ILU(1) and ILU(2)), its init-fused first sweep,
the register-pivot sweep (7-pt ILU(0), W <= 16), the template scale / Ahat / Jacobi kernels, the
CSR path, the block path, a tolerance-mode compute, and (round 2) the asynchronous block sweeps on
the template and block layouts, the warm-up, the host-pipelined compute_host / solve_host, GMRES
and set_factors.  Checks parity with the oracle where the result is deterministic, so a run under
a tool still proves the kernels computed the right thing.

    compute-sanitizer --tool racecheck python tests/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2506_05793_b200 as F  # noqa: E402
import problems as P  # noqa: E402

CASES = [("27pt", 12, 11, 1, 3, 4), ("27pt", 9, 10, 2, 2, 3), ("7pt", 20, 17, 0, 3, 4)]


def check(a, k, ns, nt, **kw):
    b = P.rhs_positive(a.n)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k, **kw)
    f.compute(ns)
    x = f.apply_host(b, nt)
    fo = oracle.compute(a, k, ns)
    assert np.array_equal(f.factors()[0], fo.vals), "factors"
    assert np.array_equal(x, oracle.apply(fo, b, nt)), "x"
    info = f.info()
    f.close()
    return info


for kind, g, gz, k, ns, nt in CASES:
    a = P.make(kind, g, gz)
    print(kind, g, gz, k, check(a, k, ns, nt)[:60], flush=True)
os.environ["FASTILU_NO_TSELL"] = "1"
a = P.make("27pt", 8, 7)
print("csr", check(a, 1, 2, 2)[:40], flush=True)
print("bsr", check(P.elasticity_pattern_3dof(4), 1, 2, 2)[:40], flush=True)
del os.environ["FASTILU_NO_TSELL"]
a = P.make("27pt", 10, 9)
f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
s = f.compute_tol(1e-6, 50)
print("tol sweeps", s, flush=True)
# asynchronous in-place sweeps with the Block Size option (non-deterministic by design: only the
# fixed point is checked), template and block layouts
for nnz in (8, 64):
    f.compute_async(40, nnz)
print("async template ok", flush=True)
f.close()
e = P.elasticity_pattern_3dof(4)
fb = F.FastILU(e.row_ptr, e.col_idx, e.values, 1)
fb.compute_async(3, 18)
print("async block ok", fb.info()[:30], flush=True)
fb.close()
# warm-up (stored iterate 0, nested level masks), bitwise vs the oracle's warm-up
a = P.make("27pt", 8, 9)
f = F.FastILU(a.row_ptr, a.col_idx, a.values, 2)
f.compute_warmup(1)
fo = oracle.compute_warmup(a, 2, 1)
assert np.array_equal(f.factors()[0], fo.vals), "warm-up factors"
print("warmup ok", flush=True)
f.close()
# host-pipelined compute_host / solve_host (two or more row chunks) and set_factors
a = P.make("27pt", 20, 21)
b = P.rhs_positive(a.n)
f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
x = f.solve_host(np.ascontiguousarray(a.values), 3, b, 4)
fo = oracle.compute(a, 1, 3)
assert np.array_equal(f.factors()[0], fo.vals), "solve_host factors"
assert np.array_equal(x, oracle.apply(fo, b, 4)), "solve_host x"
vals, s_ = f.factors()[0], None
print("solve_host ok", flush=True)
f.close()
import torch  # noqa: E402
a = P.make("aniso7pt", 12, 13)
f = F.FastILU(a.row_ptr, a.col_idx, a.values, 0)
f.compute(2)
bt = torch.tensor(P.rhs_positive(a.n), device="cuda")
xt = torch.zeros_like(bt)
it, rr = f.gmres(bt, xt, restart=20, rtol=1e-6, max_iters=200, ntrisweeps=3)
assert rr <= 1e-6, rr
print("gmres ok", it, flush=True)
ex = oracle.compute(a, 0, 60)
f.set_factors(ex.vals, ex.s)
x = f.apply_host(P.rhs_positive(a.n), 3)
assert np.array_equal(x, oracle.apply(ex, P.rhs_positive(a.n), 3)), "set_factors x"
print("set_factors ok", flush=True)
f.close()
print("sanitize case done")
