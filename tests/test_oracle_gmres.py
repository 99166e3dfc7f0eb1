"""Pins for the oracle's GMRES(m) (the paper's protocol PAPER.md:728-733)."""
import numpy as np
import scipy.linalg as sla

import oracle
import problems as P


def test_identity_one_iteration():
    n = 50
    a = P.Csr(np.arange(n + 1), np.arange(n), np.ones(n))
    b = P.rhs_signed(n)
    x, it, rr = oracle.gmres(a, b, lambda v: v)
    assert it == 1 and rr <= 1e-12 and np.allclose(x, b)


def test_exact_lu_preconditioner_two_iterations():
    a = P.random_sparse(120, 0.05, seed=3)
    A = a.to_dense()
    lu = sla.lu_factor(A)
    b = P.rhs_signed(a.n)
    x, it, rr = oracle.gmres(a, b, lambda v: sla.lu_solve(lu, v))
    assert it <= 2 and rr <= 1e-6
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-6, atol=1e-9)


def test_unpreconditioned_spd_converges_within_n():
    a = P.laplace3d_7pt(4)  # n = 64, SPD
    b = P.rhs_signed(a.n)
    x, it, rr = oracle.gmres(a, b, lambda v: v, restart=64, rtol=1e-10)
    assert it <= a.n and rr <= 1e-10
    np.testing.assert_allclose(x, np.linalg.solve(a.to_dense(), b), rtol=1e-8, atol=1e-10)


def test_restart_cycles_reach_tolerance():
    a = P.laplace3d_27pt(6)
    b = P.rhs_signed(a.n)
    x, it, rr = oracle.gmres(a, b, lambda v: v, restart=5, rtol=1e-8)
    assert it > 5 and rr <= 1e-8
    assert np.linalg.norm(b - oracle.spmv(a, x)) <= 1e-8 * np.linalg.norm(b) * (1 + 1e-6)


def test_survey_g18_iteration_counts_g16():
    """SURVEY.md reading G18 (an independent survey-time computation, not the oracle): on the
    anisotropic 7-pt 16^3 problem with x_true ~ U[0,1), b = A x_true, GMRES(60) to 1e-6 takes
    8 iterations with exact ILU(0) + exact substitution and 16 with 2 FastILU sweeps + 5 Jacobi
    sweeps.  Counts may move by one with rounding."""
    a = P.aniso3d_7pt(16)
    b = oracle.spmv(a, P.x_true(a.n))
    fe = oracle.compute(a, 0, 0)
    pat = fe.pattern
    fe.vals = oracle.exact_ilu(pat, fe.ahat)
    _, it_c, rr = oracle.gmres(a, b, oracle.exact_preconditioner(fe), restart=60, rtol=1e-6)
    assert abs(it_c - 8) <= 1 and rr <= 1e-6
    fa = oracle.compute(a, 0, 2)
    _, it_a, rr = oracle.gmres(a, b, oracle.fastilu_preconditioner(fa, 5), restart=60, rtol=1e-6)
    assert abs(it_a - 16) <= 1 and rr <= 1e-6
