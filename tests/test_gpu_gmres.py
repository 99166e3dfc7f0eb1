"""FastILU-preconditioned GMRES(60) on the GPU (BASELINE config 5; NEXT row f1) against the
oracle's GMRES with the oracle's FastILU preconditioner (same factors and Jacobi apply, which
are bitwise equal): the iteration counts agree (within one, since the Krylov dot products are
summed in a different order) and both reach the 1e-6 relative residual."""
import numpy as np
import pytest
import torch

import oracle
import paper_2506_05793_b200 as F
import problems as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("g,ns,nt", [(16, 2, 5), (32, 2, 5), (32, 2, 2), (24, 10, 10)])
def test_gmres_matches_oracle(g, ns, nt):
    a = P.aniso3d_7pt(g)
    xt = P.x_true(a.n)
    b = oracle.spmv(a, xt)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 0)
    f.compute(ns)
    tb = torch.tensor(b, device="cuda")
    tx = torch.zeros_like(tb)
    it, rr = f.gmres(tb, tx, restart=60, rtol=1e-6, max_iters=2000, ntrisweeps=nt)
    fo = oracle.compute(a, 0, ns)
    _, it_o, rr_o = oracle.gmres(a, b, oracle.fastilu_preconditioner(fo, nt), 60, 1e-6, 2000)
    assert rr <= 1e-6 and rr_o <= 1e-6
    assert abs(it - it_o) <= 1, (it, it_o)
    x = tx.cpu().numpy()
    assert np.linalg.norm(b - oracle.spmv(a, x)) <= 1e-6 * np.linalg.norm(b) * (1 + 1e-9)


def test_gmres_27pt_ilu1_restarts():
    a = P.laplace3d_27pt(20)
    b = oracle.spmv(a, P.x_true(a.n))
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
    f.compute(3)
    tb = torch.tensor(b, device="cuda")
    tx = torch.zeros_like(tb)
    it, rr = f.gmres(tb, tx, restart=5, rtol=1e-9, max_iters=500, ntrisweeps=3)
    fo = oracle.compute(a, 1, 3)
    _, it_o, rr_o = oracle.gmres(a, b, oracle.fastilu_preconditioner(fo, 3), 5, 1e-9, 500)
    assert rr <= 1e-9 and abs(it - it_o) <= 1, (it, it_o)
