"""The paper's asynchronous in-place sweeps and its "Block Size (number of nonzeroes per thread)"
option on both layouts that support them: the
template-SELL layout (27-pt / 7-pt stencils) and the block layout (3-dof patterns).  Asynchronous
results are non-deterministic, so they are checked by what the paper states and the mathematics
fixes: the same fixed point (the exact ILU(k), computed by the oracle), a preconditioner "of
similar quality" (defect after s sweeps, GMRES iterations), and the trend of GMRES iterations
with the number of sweeps (tab:fastilu_sweep)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2506_05793_b200 as F
import problems as P

pytestmark = pytest.mark.gpu


def _exact(a, k):
    pat = oracle.symbolic(a.row_ptr, a.col_idx, k)
    _, ahat, _ = oracle.scale_init(a, pat)
    return pat, ahat, oracle.exact_ilu(pat, ahat)


@pytest.mark.parametrize("kind,g,k,ept", [("27pt", 8, 1, 8), ("27pt", 8, 1, 16),
                                          ("27pt", 8, 1, 63), ("27pt", 7, 2, 32),
                                          ("7pt", 12, 0, 2), ("7pt", 12, 1, 0)])
def test_template_async_block_sizes_reach_fixed_point(kind, g, k, ept):
    a = P.make(kind, g)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    assert f.info().startswith("path=tsell")
    f.compute_async(120, ept)
    _, _, ex = _exact(a, k)
    np.testing.assert_allclose(f.factors()[0], ex, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("ept", [9, 27, 81])
def test_block_async_reaches_fixed_point(ept, monkeypatch):
    monkeypatch.setenv("FASTILU_NO_TSELL", "1")
    a = P.elasticity_pattern_3dof(5)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 2)
    assert f.info().startswith("path=bsr3"), f.info()
    f.compute_async(150, ept)
    _, _, ex = _exact(a, 2)
    np.testing.assert_allclose(f.factors()[0], ex, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("ept", [0, 8, 63])
def test_async_block_quality(ept):
    """Defect ||(Ahat - LU)|_S||_F after two asynchronous sweeps (evaluated by the oracle) is not
    worse than after two synchronous ones (the in-row Gauss-Seidel order can only help on these
    M-matrices)."""
    a = P.laplace3d_27pt(16)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
    f.compute_async(2, ept)
    va = f.factors()[0]
    f.compute(2)
    vs = f.factors()[0]
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 1)
    _, ahat, _ = oracle.scale_init(a, pat)
    assert oracle.sweep(pat, ahat, va)[1] <= oracle.sweep(pat, ahat, vs)[1] * 1.05


@pytest.mark.parametrize("g", [16, 32, 64])
def test_async_gmres_iterations_vs_sync(g):
    """PAPER.md:717 "it usually leads to a preconditioner of similar quality": GMRES(60)
    iterations to 1e-6 with 2 asynchronous sweeps <= with 2 synchronous sweeps + 1 (config 5's
    anisotropic 7-pt ILU(0), 5 Jacobi sweeps per apply)."""
    a = P.aniso3d_7pt(g)
    b = oracle.spmv(a, P.x_true(a.n))
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 0)
    tb = torch.tensor(b, device="cuda")
    tx = torch.zeros_like(tb)
    f.compute(2)
    it_s, rr_s = f.gmres(tb, tx, 60, 1e-6, 3000, 5)
    f.compute_async(2)
    it_a, rr_a = f.gmres(tb, tx, 60, 1e-6, 3000, 5)
    assert rr_s <= 1e-6 and rr_a <= 1e-6
    assert it_a <= it_s + 1, (it_a, it_s)


def test_3dof_sweep_trend_async_vs_sync(monkeypatch, capsys):
    """The paper's Table-6 experiment (tab:fastilu_sweep): 3-dof 27-pt 32^3,
    ILU(3), GMRES(60) to 1e-6 with exact triangular solves, iterations vs the number of FastILU
    sweeps s_max (paper, H100: 25, 17, 14, 12, 11, 10 for s_max = 1..6 with its elasticity
    coefficients, which are not given; ours are the 80/-1 placeholder values, so only the trend is
    comparable).  Factors from the GPU (synchronous block sweep and asynchronous with 9 and 81
    nonzeros per thread), preconditioner applied by the oracle's exact substitution."""
    a = P.elasticity_pattern_3dof(32)
    b = oracle.spmv(a, P.x_true(a.n))
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 3)
    assert f.info().startswith("path=bsr3"), f.info()
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 3)
    rows = {}
    for name, run in (("sync", lambda s: f.compute(s)),
                      ("async9", lambda s: f.compute_async(s, 9)),
                      ("async81", lambda s: f.compute_async(s, 81))):
        its = []
        for s in range(1, 7):
            run(s)
            v, sc = f.factors()
            fo = oracle.Factors(pat, sc, None, v, None)
            its.append(oracle.gmres(a, b, oracle.exact_preconditioner(fo), 60, 1e-6, 400)[1])
        rows[name] = its
    with capsys.disabled():
        print("\n3-dof 32^3 ILU(3) GMRES(60) iterations, s_max = 1..6 (paper: 25 17 14 12 11 10)")
        for k, v in rows.items():
            print(f"  {k:8s} {v}")
    for k, v in rows.items():
        assert all(v[i + 1] <= v[i] + 1 for i in range(5)), (k, v)  # more sweeps never hurt
        assert v[-1] < v[0], (k, v)
    for s in range(6):
        assert rows["async9"][s] <= rows["sync"][s] + 2 and rows["async81"][s] <= rows["sync"][s] + 2
