"""Pins for the oracle's numeric steps, each against something other than the oracle:

* scaling/init (R4, R5): dense D^-1/2 A D^-1/2 by numpy; diag(Ahat) = +-1 within ulps.
* exact ILU (the sweep map's fixed point): tridiagonal ILU(0) == Thomas LU bitwise; dense KIJ
  Gaussian elimination dropping outside S == row-wise IKJ bitwise; k >= n => LAPACK getrf.
* sweeps (R1-R3): synchronous sweeps reach the exact ILU bitwise within the
  dependency-DAG depth (computed here independently); residual non-increasing above the roundoff
  floor; diagonal A exact after one sweep; lower-bidiagonal 5x5; damping omega<1
  converges to the same fixed point; zero pivot detection (R8).
* trisolve (R6): substitution == scipy solve_triangular; Jacobi == substitution
  bitwise after nlevels sweeps; T = I; one sweep = D^-1 b; apply == dense solve of
  (D^1/2 L U D^1/2) x = b when ntri >= nlevels.
* windowed oracle: equals the global run on interior planes, bitwise.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import problems as P


def dense_LU(pat, vals):
    n = pat.n
    L = np.eye(n)
    U = np.zeros((n, n))
    for i in range(n):
        for p in range(pat.row_ptr[i], pat.row_ptr[i + 1]):
            j = pat.col_idx[p]
            if j < i:
                L[i, j] = vals[p]
            else:
                U[i, j] = vals[p]
    return L, U


def to_S(pat, dense):
    out = np.empty(pat.nnz)
    for i in range(pat.n):
        for p in range(pat.row_ptr[i], pat.row_ptr[i + 1]):
            out[p] = dense[i, pat.col_idx[p]]
    return out


# ----------------------------------------------------------------------------- scaling
def test_scaling_matches_dense_formula():
    a = P.laplace3d_27pt(4)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 1)
    s, ahat, vals = oracle.scale_init(a, pat)
    A = a.to_dense()
    d = np.abs(np.diag(A))
    Dm = np.diag(1.0 / np.sqrt(d))
    Ah = Dm @ A @ Dm
    np.testing.assert_allclose(to_S(pat, Ah), ahat, rtol=1e-15, atol=0)
    np.testing.assert_allclose(np.abs(np.diag(Ah)), 1.0, rtol=4e-16)
    # initial guess: L0 = strict-lower(Ahat) / diag(Ahat) columnwise, U0 = upper(Ahat), fill 0
    L, U = dense_LU(pat, vals)
    np.testing.assert_allclose(L, np.tril(Ah, -1) / np.diag(Ah)[None, :] + np.eye(a.n), rtol=1e-15)
    np.testing.assert_allclose(U, np.triu(Ah), rtol=1e-15)


def test_zero_diag_is_reported():
    a = P.laplace3d_7pt(3)
    v = a.values.copy()
    s, e = a.row_ptr[5], a.row_ptr[6]
    v[s + int(np.searchsorted(a.col_idx[s:e], 5))] = 0.0
    b = P.Csr(a.row_ptr, a.col_idx, v)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.compute(b, 0, 1)
    assert ei.value.status == "ZERO_DIAG" and ei.value.index == 5


# ----------------------------------------------------------------------------- exact ILU
def test_tridiagonal_ilu0_is_thomas_bitwise():
    a = P.tridiagonal(40)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 0)
    vals = oracle.exact_ilu(pat, a.values)  # exact ILU of the given matrix itself
    A = a.to_dense()
    n = a.n
    u = [A[0, 0]]
    ell = [None]
    for i in range(1, n):
        li = A[i, i - 1] / u[i - 1]
        ell.append(li)
        u.append(A[i, i] - li * A[i - 1, i])
    L, U = dense_LU(pat, vals)
    for i in range(n):
        assert U[i, i] == u[i]
        if i:
            assert L[i, i - 1] == ell[i]
            assert U[i - 1, i] == A[i - 1, i]


def _dense_kij_dropping(pat, ahat):
    n = pat.n
    inS = np.zeros((n, n), dtype=bool)
    W = np.zeros((n, n))
    for i in range(n):
        for p in range(pat.row_ptr[i], pat.row_ptr[i + 1]):
            inS[i, pat.col_idx[p]] = True
            W[i, pat.col_idx[p]] = ahat[p]
    for k in range(n):
        for i in range(k + 1, n):
            if not inS[i, k]:
                continue
            W[i, k] = W[i, k] / W[k, k]
            for j in range(k + 1, n):
                if inS[i, j] and inS[k, j]:
                    W[i, j] = W[i, j] - W[i, k] * W[k, j]
    return to_S(pat, W)


@pytest.mark.parametrize("kind,g,k", [("7pt", 3, 0), ("27pt", 3, 1), ("27pt", 4, 1),
                                       ("27pt", 4, 2), ("7pt", 4, 1)])
def test_exact_ilu_equals_dense_elimination_bitwise(kind, g, k):
    a = P.make(kind, g)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, k)
    s, ahat, _ = oracle.scale_init(a, pat)
    got = oracle.exact_ilu(pat, ahat)
    want = _dense_kij_dropping(pat, ahat)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("kind,g", [("7pt", 4), ("27pt", 3)])
def test_full_level_is_lapack_lu(kind, g):
    a = P.make(kind, g)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, a.n)  # k >= n: nothing dropped
    s, ahat, _ = oracle.scale_init(a, pat)
    vals = oracle.exact_ilu(pat, ahat)
    L, U = dense_LU(pat, vals)
    A = a.to_dense()
    Ah = A / np.sqrt(np.outer(np.diag(A), np.diag(A)))
    lu, piv = sla.lu_factor(Ah)
    assert np.array_equal(piv, np.arange(a.n))  # column-diagonally dominant: no row swaps
    np.testing.assert_allclose(np.triu(lu), U, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(np.tril(lu, -1) + np.eye(a.n), L, rtol=1e-13, atol=1e-15)


# ----------------------------------------------------------------------------- sweeps
def _final_after(pat):
    """Sweeps after which each entry is bitwise final: 1 + max over its dependencies
    (l_ik, u_kj for k < min(i,j) with (k,j) in S, plus u_jj when i > j)."""
    n = pat.n
    rows = [dict((int(pat.col_idx[p]), p) for p in range(pat.row_ptr[i], pat.row_ptr[i + 1]))
            for i in range(n)]
    fa = np.zeros(pat.nnz, dtype=np.int64)
    # entries only depend on entries of lower rows or earlier columns of the same row:
    # process rows ascending, columns ascending
    for i in range(n):
        for j in sorted(rows[i]):
            p = rows[i][j]
            m = min(i, j)
            deps = []
            for k in sorted(rows[i]):
                if k >= m:
                    break
                if j in rows[k]:
                    deps += [rows[i][k], rows[k][j]]
            if i > j:
                deps.append(rows[j][j])
            fa[p] = 1 + (max(fa[d] for d in deps) if deps else 0)
    return fa


@pytest.mark.parametrize("kind,g,k", [("7pt", 5, 0), ("27pt", 4, 1), ("27pt", 4, 2),
                                       ("aniso7pt", 5, 0), ("7pt", 4, 2)])
def test_sweeps_reach_exact_ilu_bitwise(kind, g, k):
    a = P.make(kind, g)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, k)
    s, ahat, vals = oracle.scale_init(a, pat)
    exact = oracle.exact_ilu(pat, ahat)
    bound = int(_final_after(pat).max())
    hist = []
    for sw in range(1, bound + 2):
        new, r = oracle.sweep(pat, ahat, vals)
        hist.append(r)
        if np.array_equal(new, vals):
            break
        vals = new
    assert sw <= bound + 1
    assert np.array_equal(vals, exact)
    # residual r(s-1) is non-increasing above the roundoff floor
    nrm = np.linalg.norm(ahat)
    floor = 1e3 * np.finfo(float).eps * nrm
    for r0, r1 in zip(hist, hist[1:]):
        if r1 > floor:
            assert r1 <= r0 * (1 + 1e-12)
    assert hist[-1] <= floor


def test_residual_is_frobenius_of_restricted_defect():
    a = P.laplace3d_27pt(4)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 1)
    s, ahat, vals = oracle.scale_init(a, pat)
    for _ in range(3):
        L, U = dense_LU(pat, vals)
        Ah = np.zeros((a.n, a.n))
        for i in range(a.n):
            for p in range(pat.row_ptr[i], pat.row_ptr[i + 1]):
                Ah[i, pat.col_idx[p]] = ahat[p]
        want = np.linalg.norm(to_S(pat, Ah - L @ U))
        vals, r = oracle.sweep(pat, ahat, vals)
        assert r == pytest.approx(want, rel=1e-12)


def test_diagonal_matrix_immediate():
    n = 9
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int32)
    v = np.linspace(1.0, 5.0, n) * np.where(np.arange(n) % 2, -1, 1)
    f = oracle.compute(P.Csr(rp, ci, v), 0, 1)
    assert f.resid[0] == 0.0
    assert np.array_equal(f.vals, f.ahat)  # L = I, U = diag(Ahat) after one sweep
    np.testing.assert_allclose(np.abs(f.vals), 1.0, rtol=4e-16)


def test_lower_bidiagonal_exact_lu():
    # 5x5 lower-bidiagonal + diagonal, k=0, omega=1, 5 sweeps -> exact LU
    A = np.diag([2.0, 3.0, 4.0, 5.0, 6.0]) + np.diag([-1.0, -0.5, -2.0, -1.5], -1)
    rp = [0]
    ci = []
    vals = []
    for i in range(5):
        for j in range(5):
            if A[i, j] != 0:
                ci.append(j)
                vals.append(A[i, j])
        rp.append(len(ci))
    a = P.Csr(rp, ci, vals)
    f = oracle.compute(a, 0, 5)
    L, U = dense_LU(f.pattern, f.vals)
    Ah = A / np.sqrt(np.outer(np.diag(A), np.diag(A)))
    np.testing.assert_allclose(L @ U, Ah, rtol=0, atol=1e-14)


def test_damped_sweeps_same_fixed_point():
    a = P.laplace3d_27pt(4)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 1)
    s, ahat, vals = oracle.scale_init(a, pat)
    exact = oracle.exact_ilu(pat, ahat)
    for _ in range(200):
        vals, r = oracle.sweep(pat, ahat, vals, omega=0.7)
    np.testing.assert_allclose(vals, exact, rtol=1e-13, atol=1e-15)


def test_zero_pivot_reported():
    # A = [[1,1],[1,1]]: u22 = 1 - l21 u12 = 0 after one sweep
    a = P.Csr([0, 2, 4], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0])
    oracle.compute(a, 0, 0)  # iterate 0 has a non-zero diagonal
    with pytest.raises(oracle.OracleError) as ei:
        oracle.compute(a, 0, 1)
    assert ei.value.status == "ZERO_PIVOT" and ei.value.index == 1


# ----------------------------------------------------------------------------- trisolve
def _nlevels(pat, lower):
    lev = np.zeros(pat.n, dtype=np.int64)
    order = range(pat.n) if lower else range(pat.n - 1, -1, -1)
    for i in order:
        cols = pat.col_idx[pat.row_ptr[i]:pat.row_ptr[i + 1]]
        deps = cols[cols < i] if lower else cols[cols > i]
        lev[i] = 1 + (lev[deps].max() if deps.size else 0)
    return int(lev.max())


def _factors(kind, g, k, ns):
    a = P.make(kind, g)
    f = oracle.compute(a, k, ns)
    return a, f


@pytest.mark.parametrize("kind,g,k", [("7pt", 6, 0), ("27pt", 4, 1)])
def test_substitution_matches_scipy(kind, g, k):
    a, f = _factors(kind, g, k, 2)
    L, U = dense_LU(f.pattern, f.vals)
    y = P.rhs_signed(a.n)
    z = oracle.subst_lower(f.pattern, f.vals, y)
    np.testing.assert_allclose(z, sla.solve_triangular(L, y, lower=True, unit_diagonal=True),
                               rtol=1e-13, atol=1e-14)
    w = oracle.subst_upper(f.pattern, f.vals, z)
    np.testing.assert_allclose(w, sla.solve_triangular(U, z, lower=False), rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("kind,g,k", [("7pt", 6, 0), ("27pt", 4, 1), ("7pt", 5, 1)])
def test_jacobi_exact_after_nlevels_bitwise(kind, g, k):
    a, f = _factors(kind, g, k, 3)
    pat = f.pattern
    y = P.rhs_signed(a.n)
    zl = oracle.subst_lower(pat, f.vals, y)
    nl = _nlevels(pat, True)
    assert np.array_equal(oracle.jacobi_lower(pat, f.vals, y, nl), zl)
    wu = oracle.subst_upper(pat, f.vals, zl)
    nu = _nlevels(pat, False)
    assert np.array_equal(oracle.jacobi_upper(pat, f.vals, zl, nu), wu)


def test_jacobi_identity_and_first_sweep():
    n = 7
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int32)
    pat = oracle.Pattern(rp, ci, np.zeros(n, dtype=np.int32))
    b = P.rhs_signed(n)
    assert np.array_equal(oracle.jacobi_lower(pat, np.ones(n), b, 1), b)
    assert np.array_equal(oracle.jacobi_upper(pat, np.ones(n), b, 1), b)
    a, f = _factors("27pt", 3, 1, 2)
    z = P.rhs_signed(a.n)
    L, U = dense_LU(f.pattern, f.vals)
    assert np.array_equal(oracle.jacobi_upper(f.pattern, f.vals, z, 1), z / np.diag(U))
    assert np.array_equal(oracle.jacobi_lower(f.pattern, f.vals, z, 1), z)


def test_apply_is_scaled_preconditioner_solve():
    a, f = _factors("27pt", 4, 1, 3)
    pat = f.pattern
    b = P.rhs_positive(a.n)
    nt = max(_nlevels(pat, True), _nlevels(pat, False))
    x = oracle.apply(f, b, nt)
    L, U = dense_LU(pat, f.vals)
    Dh = np.diag(1.0 / f.s)  # D^{1/2}
    M = Dh @ L @ U @ Dh
    np.testing.assert_allclose(x, np.linalg.solve(M, b), rtol=1e-12)


def test_damped_trisolve_converges_to_substitution():
    a, f = _factors("7pt", 5, 0, 2)
    y = P.rhs_positive(a.n)
    z = oracle.jacobi_lower(f.pattern, f.vals, y, 300, omega=0.8)
    np.testing.assert_allclose(z, oracle.subst_lower(f.pattern, f.vals, y), rtol=1e-13)


# ----------------------------------------------------------------------------- windowed oracle
def test_windowed_equals_global_interior():
    g, gz = 4, 30
    a = P.laplace3d_27pt(g, gz=gz)
    b = P.rhs_positive(a.n)
    k, ns, nt = 1, 3, 5
    fg = oracle.compute(a, k, ns)
    xg = oracle.apply(fg, b, nt)
    plane = g * g
    lo_p, hi_p = 1, 23
    lo, hi, fw, xw = oracle.windowed(a, plane, lo_p, hi_p, k, ns, b_full=b, ntri=nt)
    # compare planes 14..15: >= ns+nt+k+4 planes above the cut, >= nt+2 below
    for z in (14, 15):
        for i in range(z * plane, (z + 1) * plane):
            gi = slice(fg.pattern.row_ptr[i], fg.pattern.row_ptr[i + 1])
            wi = slice(fw.pattern.row_ptr[i - lo], fw.pattern.row_ptr[i - lo + 1])
            assert np.array_equal(fg.pattern.col_idx[gi], fw.pattern.col_idx[wi] + lo)
            assert np.array_equal(fg.vals[gi], fw.vals[wi])
        assert np.array_equal(xg[z * plane:(z + 1) * plane], xw[z * plane - lo:(z + 1) * plane - lo])


# ----------------------------------------------------------------------------- Manteuffel shift
def test_shift_is_factoring_the_shifted_matrix():
    """Reading R9: compute with shift alpha == compute on
    A' = A + alpha diag(|a_ii|) built explicitly here (bitwise); alpha = 0 changes nothing."""
    a = P.laplace3d_27pt(5)
    alpha = 0.3
    v = a.values.copy()
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    d = a.col_idx == rows
    v[d] = v[d] + alpha * np.abs(v[d])
    f1 = oracle.compute(a, 1, 3, shift=alpha)
    f2 = oracle.compute(P.Csr(a.row_ptr, a.col_idx, v), 1, 3)
    assert np.array_equal(f1.vals, f2.vals) and np.array_equal(f1.s, f2.s)
    assert np.array_equal(oracle.compute(a, 1, 3, shift=0.0).vals, oracle.compute(a, 1, 3).vals)


# ----------------------------------------------------------------------------- warm-up (R10)
def test_warmup_level0_is_plain_compute():
    a = P.laplace3d_27pt(6)
    f0 = oracle.compute_warmup(a, 0, 3)
    f1 = oracle.compute(a, 0, 3)
    assert np.array_equal(f0.vals, f1.vals) and np.array_equal(f0.resid, f1.resid)


def test_warmup_reaches_exact_ilu():
    """The sweep map's fixed point does not depend on the initial guess: enough warm-up sweeps
    give the exact ILU(k) bitwise (k = 2, 4^3 27-pt; bound from the dependency DAG)."""
    a = P.laplace3d_27pt(4)
    f = oracle.compute_warmup(a, 2, 40)
    assert np.array_equal(f.vals, oracle.exact_ilu(f.pattern, f.ahat))
    assert f.resid[-1] <= 1e-15  # the defect a - l u_jj keeps one rounding at the fixed point


def test_warmup_trend_gmres():
    """PAPER.md:612 vs 617 (tab:fastilu_nx16 b): warm-up never needs more GMRES iterations."""
    a = P.laplace3d_27pt(12)
    b = oracle.spmv(a, P.x_true(a.n))
    for k in (1, 2, 3):
        i0 = oracle.gmres(a, b, oracle.fastilu_preconditioner(oracle.compute(a, k, 2), 30))[1]
        i1 = oracle.gmres(a, b, oracle.fastilu_preconditioner(oracle.compute_warmup(a, k, 2),
                                                                30))[1]
        assert i1 <= i0, (k, i0, i1)


# ----------------------------------------------------------------------------- exact residual sum
def test_fsum_is_exactly_rounded():
    """The residual accumulator (Shewchuk partials) == math.fsum bitwise, on inputs where a
    left-to-right sum loses everything (cancellation, tiny terms under huge ones, ties)."""
    import math
    rng = np.random.default_rng(5)
    cases = [
        np.array([1e16, 1.0, -1e16, 1.0]),
        np.array([1.0, 1e-16, 1e-16, 1e-16, 1e-16]),
        np.array([2.0 ** 53, 1.0, 1.0, -2.0 ** 53]),
        np.array([1.0, 2.0 ** -53, 2.0 ** -106]),             # half-way case decided by the tail
        np.array([1.0, 2.0 ** -53, -2.0 ** -106]),
        rng.standard_normal(10000) * 10.0 ** rng.integers(-20, 20, 10000),
        rng.random(100000) ** 2,
        np.zeros(0),
    ]
    for x in cases:
        got = oracle.fsum(x)
        assert got == math.fsum(x), (got, math.fsum(x))
    y = rng.random(1000)
    assert sum(y.tolist()) != math.fsum(y) or True  # (documentation: naive sums may differ)


def test_residual_sum_is_exact_fsum_of_squares():
    """r(s-1)^2 of the oracle == math.fsum of the per-entry squared defects, which the test
    obtains from dense algebra at iterate s-1 on an input where every defect is exact:
    A with entries in {1, -1/2} and k = 0 on a 1D chain (all products are exact dyadics)."""
    import math
    n = 12
    A = np.eye(n) + np.diag([-0.5] * (n - 1), 1) + np.diag([-0.5] * (n - 1), -1)
    a = P.Csr(*_dense_to_csr(A))
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 0)
    s, ahat, vals = oracle.scale_init(a, pat)
    L, U = dense_LU(pat, vals)
    D = to_S(pat, A - L @ U)          # iterate 0 has only dyadic values: L @ U is exact
    _, r = oracle.sweep(pat, ahat, vals)
    assert r * r == pytest.approx(math.fsum(D * D), rel=2 * np.finfo(float).eps)
    assert r == math.sqrt(math.fsum(D * D))


def _dense_to_csr(A):
    rp, ci, v = [0], [], []
    for i in range(A.shape[0]):
        for j in range(A.shape[1]):
            if A[i, j] != 0.0:
                ci.append(j)
                v.append(A[i, j])
        rp.append(len(ci))
    return rp, ci, v


# ----------------------------------------------------------------------------- damping (R1, R6)
def _golden(name):
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", name)))


def _frac(x):
    from fractions import Fraction
    return float(Fraction(x))


def test_damped_sweeps_hand_derived():
    """omega = 0.7 iterates s = 1..3 and r(0..2) of the 3x3 tridiagonal example derived by hand
    in tests/golden/README.md from Fig. algo:fastILU_comp + readings R1-R4.
    The swapped-weight mutant (w old + (1-w) new) already fails at sweep 1 (u22 = 37/40)."""
    gd = _golden("damped_3x3.json")
    a = P.Csr(*_dense_to_csr(np.array(gd["matrix"]["dense"])))
    w = _frac(gd["omega"])
    for s, want in gd["sweeps"].items():
        f = oracle.compute(a, 0, int(s), omega=w)
        assert f.pattern.nnz == 7 and np.array_equal(f.s, np.ones(3))
        np.testing.assert_allclose(f.vals, [_frac(v) for v in want], rtol=4 * np.finfo(float).eps,
                                   atol=0)
    f = oracle.compute(a, 0, 3, omega=w)
    want_r2 = [_frac(v) for v in gd["resid_squared"].values()]
    np.testing.assert_allclose(f.resid ** 2, want_r2, rtol=1e-14)


def test_damped_jacobi_hand_derived():
    """omega_tri = 0.8 Jacobi iterates t = 1..3 for L and U (reading R6),
    derived by hand in tests/golden/README.md."""
    gd = _golden("damped_3x3.json")["jacobi"]
    wt = _frac(gd["omega_tri"])
    rp = np.array([0, 2, 5, 7], dtype=np.int64)
    ci = np.array([0, 1, 0, 1, 2, 1, 2], dtype=np.int32)
    pat = oracle.Pattern(rp, ci, np.zeros(7, dtype=np.int32))
    lo = gd["lower"]["strict_L"]
    up = gd["upper"]["U"]
    vals_L = np.array([1.0, 0.0, _frac(lo["l21"]), 1.0, 0.0, _frac(lo["l32"]), 1.0])
    vals_U = np.array([_frac(up["u11"]), _frac(up["u12"]), 0.0, _frac(up["u22"]), _frac(up["u23"]),
                       0.0, _frac(up["u33"])])
    y = np.array([_frac(v) for v in gd["lower"]["y"]])
    z = np.array([_frac(v) for v in gd["upper"]["z"]])
    for t, want in gd["lower"]["z"].items():
        np.testing.assert_allclose(oracle.jacobi_lower(pat, vals_L, y, int(t), omega=wt),
                                   [_frac(v) for v in want], rtol=4 * np.finfo(float).eps, atol=0)
    for t, want in gd["upper"]["w"].items():
        np.testing.assert_allclose(oracle.jacobi_upper(pat, vals_U, z, int(t), omega=wt),
                                   [_frac(v) for v in want], rtol=4 * np.finfo(float).eps, atol=0)


@pytest.mark.parametrize("w", [0.3, 0.7, 1.0])
def test_damped_2x2_closed_form(w):
    """2x2, unit diagonal, k = 0: l21 stays c and u22(s) - (1 - cb) = (1 - w)(u22(s-1) - (1 - cb))
    (R1-R3), so u22(s) = 1 - cb (1 - (1 - w)^s): geometric convergence at rate 1 - w."""
    b, c = -0.4, -0.6
    a = P.Csr([0, 2, 4], [0, 1, 0, 1], [1.0, b, c, 1.0])
    for s in range(1, 7):
        f = oracle.compute(a, 0, s, omega=w)
        assert f.vals[2] == pytest.approx(c, rel=1e-15)
        assert f.vals[3] == pytest.approx(1 - c * b * (1 - (1 - w) ** s), rel=1e-15)


def test_omega_zero_is_the_identity_and_update_is_affine():
    """omega = 0 leaves every iterate unchanged (sweep and Jacobi); for any omega the damped
    update satisfies out(w) - old = w (out(1) - old) up to rounding: the weight w multiplies
    the new value, 1 - w the old one (R1), not the other way round."""
    a = P.laplace3d_27pt(4)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 1)
    s, ahat, vals = oracle.scale_init(a, pat)
    vals, _ = oracle.sweep(pat, ahat, vals)          # a generic iterate (fill no longer 0)
    same, _ = oracle.sweep(pat, ahat, vals, omega=0.0)
    assert np.array_equal(same, vals)
    full, _ = oracle.sweep(pat, ahat, vals, omega=1.0)
    for w in (0.25, 0.7):
        got, _ = oracle.sweep(pat, ahat, vals, omega=w)
        np.testing.assert_allclose(got - vals, w * (full - vals), rtol=1e-12, atol=1e-15)
    y = P.rhs_positive(a.n)
    assert np.array_equal(oracle.jacobi_lower(pat, full, y, 3, omega=0.0), np.zeros(a.n))
    z1 = oracle.jacobi_lower(pat, full, y, 1, omega=1.0)
    np.testing.assert_allclose(oracle.jacobi_lower(pat, full, y, 1, omega=0.6), 0.6 * z1,
                               rtol=1e-15)


# ----------------------------------------------------------------------------- warm-up embedding (R10)
def test_warmup_embedding_dense():
    """compute_warmup(k=2, 1 sweep per level) == level 0 sweep, then the level-0 factors placed
    into S_1 through a dense n x n matrix (fill = +0.0), one S_1 sweep, the same into S_2, one
    S_2 sweep (reading R10).  The embedding here is independent of the oracle's
    (a dense matrix, indexed by (row, column))."""
    a = P.laplace3d_27pt(4)
    n = a.n
    vals, r_hist, pat = None, [], None
    for L in range(3):
        pat = oracle.symbolic(a.row_ptr, a.col_idx, L)
        s, ahat, v0 = oracle.scale_init(a, pat)
        if vals is None:
            v = v0
        else:
            D = np.zeros((n, n))
            for i in range(n):
                for p in range(prev.row_ptr[i], prev.row_ptr[i + 1]):
                    D[i, prev.col_idx[p]] = vals[p]
            v = to_S(pat, D)
        vals, r = oracle.sweep(pat, ahat, v)
        r_hist.append(r)
        prev = pat
    f = oracle.compute_warmup(a, 2, 1)
    assert np.array_equal(f.pattern.col_idx, pat.col_idx)
    assert np.array_equal(f.vals, vals)
    assert np.array_equal(f.resid, np.array(r_hist))


def test_warmup_without_fill_is_one_longer_run():
    """A pattern with no fill at any level (tridiagonal, S_0 = S_1 = S_2) makes the warm-up's
    embedding the identity: FastILU(0), FastILU(1), FastILU(2) with ns sweeps each == one
    FastILU(0) run with 3 ns sweeps, bitwise (factors and residual history)."""
    a = P.tridiagonal(30)
    ns = 2
    f = oracle.compute_warmup(a, 2, ns)
    g = oracle.compute(a, 0, 3 * ns)
    assert np.array_equal(f.vals, g.vals)
    assert np.array_equal(f.resid, g.resid)


# ----------------------------------------------------------------------------- OpenMP mode
def test_threads_bitwise():
    """The OpenMP-over-rows mode is bitwise the single-thread oracle (factors, residuals, x)."""
    a = P.laplace3d_27pt(9, gz=7)
    b = P.rhs_positive(a.n)
    try:
        oracle.set_threads(1)
        f1 = oracle.compute(a, 1, 3)
        x1 = oracle.apply(f1, b, 5, omega_tri=0.9)
        assert oracle.set_threads(4) in (1, 4)
        f4 = oracle.compute(a, 1, 3)
        x4 = oracle.apply(f4, b, 5, omega_tri=0.9)
    finally:
        oracle.set_threads(1)
    assert np.array_equal(f1.vals, f4.vals) and np.array_equal(f1.resid, f4.resid)
    assert np.array_equal(x1, x4)
