"""Small ragged cases of every default-path kernel, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): the staged TMA sweep (27-pt ILU(1) and ILU(2)), its init-fused first sweep,
the register-pivot sweep (7-pt ILU(0), W <= 16), the template scale / Ahat / Jacobi kernels, the
CSR path, the block path, and a tolerance-mode compute.  Checks parity with the oracle so a run
under a tool still proves the kernels computed the right thing.

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
print("sanitize case done")
