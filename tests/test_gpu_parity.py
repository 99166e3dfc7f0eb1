"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Tolerance (north_star): factors per entry |g - o| <= 1e-12 |o| (and g == o
where o == 0); x per entry <= 1e-12 |o| with b > 0; pattern bit-exact.  Every kernel uses the
oracle's operation order (ascending pivots / columns, explicitly rounded products and
differences), so factors and x are in fact bitwise equal (asserted separately).  Inputs: seeded
generators in problems/ only.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2506_05793_b200 as F
import problems as P

pytestmark = pytest.mark.gpu

RTOL = 1e-12
# r(s-1) is ONE scalar summed over nnz(S) squares.  The oracle sums them exactly and rounds once
# (oracle.fsum, pinned to math.fsum); the GPU adds the same squared defects (its factors are
# bitwise the oracle's) along chains of at most ~150 additions at these sizes (per-thread fma
# chain over its targets + 5 shuffles + warps per block + partials per reduce thread + a
# 10-level tree), each adding <= eps relative error to a sum of non-negative terms, so
# |dr^2|/r^2 <= 150 eps = 3.3e-14 and |dr|/r <= 1.7e-14 (Higham, Accuracy and Stability, 4.2).
RTOL_RESID = 1e-13


def gpu_run(a, k, ns, nt=0, b=None, omega=1.0, omega_tri=1.0, alias=False, shift=0.0):
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k, omega=omega, omega_tri=omega_tri,
                  shift=shift)
    f.compute(ns)
    vals, s = f.factors()
    x = None
    if b is not None:
        tb = torch.tensor(b, dtype=torch.float64, device="cuda")
        tx = tb if alias else torch.empty_like(tb)
        f.apply(tb, tx, nt)
        torch.cuda.synchronize()
        x = tx.cpu().numpy()
    return f, vals, s, x


def assert_rel(g, o, rtol=RTOL, what=""):
    g, o = np.asarray(g), np.asarray(o)
    assert g.shape == o.shape, what
    zero = o == 0
    assert np.array_equal(g[zero], o[zero]), f"{what}: entries that are exactly 0 in the oracle"
    err = np.abs(g - o) / np.where(zero, 1.0, np.abs(o))
    i = int(np.argmax(err)) if err.size else 0
    assert err.size == 0 or err.max() <= rtol, f"{what}: max rel err {err.max():.3e} at {i}"


def full_check(a, k, ns, nt, omega=1.0, omega_tri=1.0, bitwise=True, shift=0.0):
    b = P.rhs_positive(a.n)
    f, vals, s, x = gpu_run(a, k, ns, nt, b, omega, omega_tri, shift=shift)
    fo = oracle.compute(a, k, ns, omega, shift=shift)
    rp, ci, lev = f.pattern()
    assert np.array_equal(rp, fo.pattern.row_ptr)
    assert np.array_equal(ci, fo.pattern.col_idx)
    assert np.array_equal(lev.astype(np.int32), fo.pattern.level)
    assert np.array_equal(s, fo.s)
    assert_rel(vals, fo.vals, what="factors")
    if bitwise:
        assert np.array_equal(vals, fo.vals), "factors not bitwise equal to the oracle"
    np.testing.assert_allclose(f.residual_history(), fo.resid, rtol=RTOL_RESID)
    xo = oracle.apply(fo, b, nt, omega_tri)
    assert_rel(x, xo, what="x")
    if bitwise:  # every trisolve kernel sums in the oracle's order (G14)
        assert np.array_equal(x, xo), "x not bitwise equal to the oracle"
    return f


# ------------------------------------------------------------------ BASELINE configs[0]
def test_config1_7pt_10_ilu0():
    full_check(P.laplace3d_7pt(10), 0, 3, 5)


@pytest.mark.parametrize("kind,g,gz,k,ns,nt", [
    ("27pt", 12, None, 1, 3, 5),
    ("27pt", 10, None, 2, 3, 5),
    ("27pt", 9, 13, 1, 4, 3),       # ragged grid
    ("aniso7pt", 16, None, 0, 2, 5),
    ("7pt", 17, None, 1, 3, 5),
    ("7pt", 11, None, 2, 2, 4),
    ("27pt", 8, None, 3, 2, 2),
])
def test_stencils(kind, g, gz, k, ns, nt):
    full_check(P.make(kind, g, gz), k, ns, nt)


@pytest.mark.parametrize("kind,g,gz,k,ns,nt", [
    ("27pt", 12, None, 1, 3, 5),
    ("27pt", 9, 11, 2, 3, 3),
    ("7pt", 17, None, 0, 3, 5),
])
@pytest.mark.parametrize("path", ["csr-classes", "csr-hash"])
def test_csr_kernels(kind, g, gz, k, ns, nt, path, monkeypatch):
    """The general CSR kernels (template path disabled): class-program and hash sweeps."""
    monkeypatch.setenv("FASTILU_NO_TSELL", "1")
    if path == "csr-hash":
        monkeypatch.setenv("FASTILU_NO_CLASSES", "1")
    f = full_check(P.make(kind, g, gz), k, ns, nt)
    assert f.info().startswith(f"path={path}"), f.info()


@pytest.mark.parametrize("kind,g,k", [("27pt", 12, 1), ("27pt", 10, 2), ("7pt", 20, 0),
                                       ("aniso7pt", 16, 1)])
def test_template_path_active(kind, g, k):
    """Stencil patterns take the template-SELL path with the JIT-specialised sweep."""
    f = full_check(P.make(kind, g), k, 3, 3)
    assert f.info().startswith("path=tsell"), f.info()


def test_3dof_pattern():
    full_check(P.elasticity_pattern_3dof(5), 1, 3, 3)


@pytest.mark.parametrize("seed,k", [(11, 0), (12, 2)])
def test_random_sparse(seed, k):
    full_check(P.random_sparse(700, 0.006, seed=seed), k, 3, 4)


def test_damping():
    full_check(P.laplace3d_27pt(9, gz=11), 1, 4, 5, omega=0.7, omega_tri=0.8)


@pytest.mark.parametrize("path", ["tsell", "csr"])
def test_manteuffel_shift(path, monkeypatch):
    """Option 'Shift' (reading R9) on both layouts."""
    if path == "csr":
        monkeypatch.setenv("FASTILU_NO_TSELL", "1")
    f = full_check(P.laplace3d_27pt(10), 1, 3, 4, shift=0.25)
    assert f.info().startswith(f"path={path}")


@pytest.mark.parametrize("kind,g,k", [("27pt", 10, 2), ("27pt", 9, 1), ("7pt", 12, 2)])
def test_warmup(kind, g, k):
    """Option 'Warm up' (reading R10): bitwise equal to the oracle's warm-up."""
    a = P.make(kind, g)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    f.compute_warmup(2)
    fo = oracle.compute_warmup(a, k, 2)
    assert np.array_equal(f.factors()[0], fo.vals)
    np.testing.assert_allclose(f.residual_history(), fo.resid, rtol=RTOL_RESID)


@pytest.mark.parametrize("nt", [1, 2])
def test_few_trisweeps(nt):
    full_check(P.laplace3d_7pt(12), 0, 2, nt)


@pytest.mark.parametrize("kind,k,ns,nt", [("7pt", 0, 2, 5), ("aniso7pt", 0, 2, 1),
                                           ("7pt", 0, 3, 2)])
def test_solve_host_register_pivot_path(kind, k, ns, nt):
    """Narrow templates (7-pt ILU(0), W = 7) pipeline through the register-pivot sweeps (iterate
    0 stored by the init kernel, diagonal schedule): solve_host's x and factors are bitwise those
    of compute + apply and the oracle's."""
    a = P.make(kind, 40, 90)
    b = P.rhs_positive(a.n)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    x1 = f.solve_host(a.values, ns, b, nt)
    v1, _ = f.factors()
    f.compute(ns)
    assert np.array_equal(x1, f.apply_host(b, nt))
    assert np.array_equal(v1, f.factors()[0])
    fo = oracle.compute(a, k, ns)
    assert np.array_equal(v1, fo.vals)
    assert np.array_equal(x1, oracle.apply(fo, b, nt))


@pytest.mark.parametrize("om_tri", [1.0, 0.7])
def test_one_trisweep_fused(om_tri):
    """ntri = 1 runs the first L and U sweeps as one pass (first_LU_kernel): x bitwise the
    oracle's one-sweep apply, damped or not, on the template and the CSR path."""
    full_check(P.laplace3d_27pt(9), 1, 3, 1, omega_tri=om_tri)
    full_check(P.random_sparse(300, 0.03, seed=5), 1, 3, 1, omega_tri=om_tri)


def test_zero_and_many_sweeps():
    full_check(P.laplace3d_27pt(6), 1, 0, 3)
    full_check(P.laplace3d_27pt(6), 1, 40, 30)  # converged to the exact ILU


def test_sweeps_reach_exact_ilu_on_gpu():
    a = P.laplace3d_7pt(6)
    f, vals, s, _ = gpu_run(a, 0, 60)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 0)
    _, ahat, _ = oracle.scale_init(a, pat)
    assert np.array_equal(vals, oracle.exact_ilu(pat, ahat))


@pytest.mark.parametrize("kind,g,k", [("27pt", 10, 1), ("27pt", 8, 2), ("7pt", 12, 0)])
def test_sweeps_to_convergence(kind, g, k):
    """BASELINE config 3 semantics ("sweeps to convergence", reading G15) at small size: the GPU
    stops at the same sweep s* as the oracle and its factors are bitwise equal."""
    a = P.make(kind, g)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    s_gpu = f.compute_tol(1e-10, 100)
    fo, s_or = oracle.compute_tol(a, k, 1e-10, 100)
    assert s_gpu == s_or and 5 < s_gpu < 100
    vals, _ = f.factors()
    assert np.array_equal(vals, fo.vals)
    np.testing.assert_allclose(f.residual_history(), fo.resid, rtol=RTOL_RESID)


def test_alias_and_host_apply():
    a = P.laplace3d_27pt(8)
    b = P.rhs_positive(a.n)
    f, _, _, x1 = gpu_run(a, 1, 3, 5, b)
    _, _, _, x2 = gpu_run(a, 1, 3, 5, b, alias=True)
    assert np.array_equal(x1, x2)
    assert np.array_equal(f.apply_host(b, 5), x1)


def test_signed_rhs_componentwise():
    a = P.laplace3d_27pt(9)
    b = P.rhs_signed(a.n)
    f, vals, s, x = gpu_run(a, 1, 3, 5, b)
    fo = oracle.compute(a, 1, 3)
    xo = oracle.apply(fo, b, 5)
    # componentwise bound for signed data
    assert np.abs(x - xo).max() <= 1e-12 * np.abs(xo).max()


def test_determinism_and_set_values():
    a = P.laplace3d_27pt(10)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
    f.compute(3)
    v1, _ = f.factors()
    f.compute(3)
    v2, _ = f.factors()
    assert np.array_equal(v1, v2)
    a2v = a.values * np.linspace(1.0, 2.0, a.nnz)
    a2 = P.Csr(a.row_ptr, a.col_idx, a2v)
    f.set_values(a2v)
    f.compute(3)
    v3, _ = f.factors()
    assert_rel(v3, oracle.compute(a2, 1, 3).vals)
    tv = torch.tensor(a.values, device="cuda")
    f.set_values_device(tv)
    f.compute(3)
    assert np.array_equal(f.factors()[0], v1)


def test_timings_before_any_apply():
    """fastilu_get_timings before the first apply must not leave a CUDA error behind that a
    later launch check would report (regression)."""
    a = P.laplace3d_27pt(6)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
    for _ in range(3):
        f.compute(2)
        t = f.timings()
        assert t["apply_ms"] == 0.0 and t["sweeps_ms"] > 0.0


def test_tiny_and_diagonal():
    full_check(P.Csr([0, 1], [0], [4.0]), 0, 2, 2)
    n = 37
    full_check(P.Csr(np.arange(n + 1), np.arange(n), np.linspace(-3, 5, n) + 0.5), 0, 1, 1)
    full_check(P.tridiagonal(300), 1, 5, 5)


def test_empty_matrix():
    """n = 0 (degenerate case): create, compute and apply succeed and do nothing; the oracle
    agrees (empty pattern, empty x)."""
    a = P.Csr(np.zeros(1), np.zeros(0), np.zeros(0))
    fo = oracle.compute(a, 1, 3)
    assert fo.pattern.nnz == 0 and len(oracle.apply(fo, np.zeros(0), 5)) == 0
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
    f.compute(3)
    b = torch.empty(0, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    f.apply(b, x, 5)
    torch.cuda.synchronize()
    rp, ci, _ = f.pattern()
    assert list(rp) == [0] and len(ci) == 0
    f.close()


def test_errors():
    a = P.laplace3d_7pt(4)
    v = a.values.copy()
    s, e = a.row_ptr[9], a.row_ptr[10]
    v[s + int(np.searchsorted(a.col_idx[s:e], 9))] = 0.0
    f = F.FastILU(a.row_ptr, a.col_idx, v, 0)
    with pytest.raises(F.FastILUError) as ei:
        f.compute(1)
    assert ei.value.status == "ZERO_DIAG" and ei.value.index == 9
    tb = torch.ones(a.n, dtype=torch.float64, device="cuda")
    with pytest.raises(F.FastILUError) as ei:
        f.apply(tb, tb, 1)
    assert ei.value.status == "STATE"
    z = P.Csr([0, 2, 4], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0])
    g = F.FastILU(z.row_ptr, z.col_idx, z.values, 0)
    g.compute(0)
    with pytest.raises(F.FastILUError) as ei:
        g.compute(1)
    assert ei.value.status == "ZERO_PIVOT" and ei.value.index == 1
    with pytest.raises(oracle.OracleError) as eo:
        oracle.compute(z, 0, 1)
    assert eo.value.index == 1


def test_config2_full_size_7pt_128_ilu0():
    """BASELINE configs[1] at full size (n = 2,097,152), element by element."""
    full_check(P.laplace3d_7pt(128), 0, 3, 5)


# ------------------------------------------------------------ asynchronous in-place sweeps
def test_async_reaches_the_fixed_point():
    """in-place (asynchronous) sweeps are non-deterministic but share the
    synchronous sweeps' fixed point: after enough sweeps the factors equal the exact ILU(k)."""
    a = P.laplace3d_27pt(8)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
    f.compute_async(80)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 1)
    _, ahat, _ = oracle.scale_init(a, pat)
    np.testing.assert_allclose(f.factors()[0], oracle.exact_ilu(pat, ahat), rtol=1e-13,
                               atol=1e-15)


def test_async_quality_vs_synchronous():
    """Gauss-Seidel-like updates: the defect ||(Ahat - LU)|_S|| of the factors after two
    asynchronous sweeps (evaluated by the oracle) is not worse than after two synchronous ones."""
    a = P.laplace3d_27pt(16)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
    f.compute_async(2)
    va = f.factors()[0]
    f.compute(2)
    vs = f.factors()[0]
    pat = oracle.symbolic(a.row_ptr, a.col_idx, 1)
    _, ahat, _ = oracle.scale_init(a, pat)
    ra = oracle.sweep(pat, ahat, va)[1]
    rs = oracle.sweep(pat, ahat, vs)[1]
    assert ra <= rs * 1.05, (ra, rs)


@pytest.mark.parametrize("kind,g,k,omega", [("27pt", 10, 1, 1.0), ("27pt", 9, 2, 0.7),
                                             ("7pt", 12, 1, 1.0)])
def test_first_sweep_kernel_equals_full_sweep(kind, g, k, omega, monkeypatch):
    """Sweep 1 from iterate 0 runs a kernel restricted to the terms whose operands lie on A's
    sub-template (fill entries of iterate 0 are exactly +0.0); it must equal the full sweep."""
    a = P.make(kind, g)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k, omega=omega)
    f.compute(2)
    monkeypatch.setenv("FASTILU_NO_FIRST_SWEEP", "1")
    h = F.FastILU(a.row_ptr, a.col_idx, a.values, k, omega=omega)
    h.compute(2)
    assert f.info().startswith("path=tsell") and h.info().startswith("path=tsell")
    assert np.array_equal(f.factors()[0], h.factors()[0])
    np.testing.assert_array_equal(f.residual_history(), h.residual_history())


# every template-path kernel variant computes exactly the oracle's factors and x
_VARIANTS = [
    ("register-pivot sweep", {"FASTILU_TSELL_STAGED": "0"}, None),
    ("staged sweep forced on", {"FASTILU_TSELL_STAGED": "1"}, "staged=1"),
    ("iterate 0 stored by the init", {"FASTILU_NO_FUSED_INIT": "1"}, None),
    ("shifted tiles (smaller TMA box)", {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_ST_OPTS": "64"},
     "staged=1"),
    ("3-stage ring", {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_STAGES": "3",
                      "FASTILU_TSELL_ST_OPTS": "256"}, "st_stages=3"),
    ("3-stage ring, 192-row tiles, last-arriver producer",
     {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_STAGES": "3", "FASTILU_TSELL_ST_THREADS": "384",
      "FASTILU_TSELL_ST_OPTS": "1792"}, None),
    ("thread-0 producer", {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_ST_OPTS": "768"}, "staged=1"),
    ("generic scale / init kernels", {"FASTILU_NO_JIT_PREP": "1"}, None),
    ("generic Jacobi kernels", {"FASTILU_NO_JIT_JACOBI": "1"}, None),
    ("loads-first Jacobi kernels", {"FASTILU_JIT_JACOBI_MODE": "1"}, None),
    ("128-row tiles", {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_ST_THREADS": "256"}, None),
    ("one part-warp per slice, 320-row tiles (full sweep)",
     {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_ST_PARTS": "1", "FASTILU_TSELL_ST_THREADS": "320"},
     None),
    ("init-fused sweep 1 with the full sweep's block shape",
     {"FASTILU_TSELL_INIT_PARTS": "2", "FASTILU_TSELL_INIT_THREADS": "512"}, None),
    ("init-fused sweep 1 with 128-row tiles (more tiles than the full sweep)",
     {"FASTILU_TSELL_INIT_PARTS": "1", "FASTILU_TSELL_INIT_THREADS": "128"}, None),
    ("two part-warps per slice, 256-row tiles",
     {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_ST_PARTS": "2", "FASTILU_TSELL_ST_THREADS": "512"},
     None),
    ("divisions through __ddiv_rn", {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_ST_OPTS": "0"},
     "staged=1"),
    ("column-major boxes", {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_ST_OPTS": "5888"},
     "staged=1"),
    ("column-major boxes, no presence select on l_it / u_jj",
     {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_ST_OPTS": "14080"}, "staged=1"),
    ("no presence select, row-major boxes",
     {"FASTILU_TSELL_STAGED": "1", "FASTILU_TSELL_ST_OPTS": "9984"}, "staged=1"),
]


@pytest.mark.parametrize("name,env,marker", _VARIANTS, ids=[v[0] for v in _VARIANTS])
@pytest.mark.parametrize("kind,g,gz,k,ns,nt", [("27pt", 12, 11, 1, 3, 5), ("27pt", 9, 10, 2, 2, 3),
                                               ("7pt", 20, 17, 0, 3, 4), ("27pt", 11, 9, 0, 1, 1)])
def test_template_kernel_variants(name, env, marker, kind, g, gz, k, ns, nt, monkeypatch):
    """Ragged grids (n not a multiple of the tile): factors, residual history and x of each
    kernel variant are bitwise the oracle's."""
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    a = P.make(kind, g, gz)
    b = P.rhs_positive(a.n)
    f, vals, _, x = gpu_run(a, k, ns, nt, b)
    assert f.info().startswith("path=tsell")
    if marker and not (k == 2 and "FASTILU_TSELL_STAGES" in env):  # 3 x 87 KB > 227 KB:
        assert marker in f.info(), f.info()  # ILU(2) then keeps the register-pivot kernel
    fo = oracle.compute(a, k, ns)
    assert np.array_equal(vals, fo.vals)
    np.testing.assert_allclose(f.residual_history(), fo.resid,
                               rtol=RTOL_RESID)
    assert np.array_equal(x, oracle.apply(fo, b, nt))


@pytest.mark.parametrize("offsets,k", [((-40, -33, 33, 40), 1), ((-70, -3, 2, 65), 0),
                                       ((-100, -64, 64, 100), 0), ((-100, -64, 64, 100), 1),
                                       ((-100, -64, -1, 1, 64, 100), 1)])
@pytest.mark.parametrize("staged", ["0", "1"])
def test_banded_templates(offsets, k, staged, monkeypatch):
    """Template patterns whose pivot groups lie away from the row (the last group's TMA box then
    misses the tile's own rows, and pivots span several slices): both sweep kernels, factors and
    x bitwise the oracle's."""
    monkeypatch.setenv("FASTILU_TSELL_STAGED", staged)
    a = P.banded(3001, offsets)
    b = P.rhs_positive(a.n)
    f, vals, _, x = gpu_run(a, k, 3, 4, b)
    assert f.info().startswith("path=tsell"), f.info()
    assert ("staged=1" in f.info()) == (staged != "0"), f.info()
    fo = oracle.compute(a, k, 3)
    assert np.array_equal(vals, fo.vals)
    assert np.array_equal(x, oracle.apply(fo, b, 4))


@pytest.mark.parametrize("kind,g,gz,k,ns", [("27pt", 24, 70, 1, 3), ("27pt", 20, 41, 2, 2),
                                            ("7pt", 40, 90, 0, 4), ("27pt", 24, 70, 1, 1)])
def test_compute_host_pipelined(kind, g, gz, k, ns):
    """fastilu_compute_host (values uploaded in row chunks, sweeps advanced chunk by chunk along
    a diagonal) equals set_values + compute bitwise (factors, x), and the oracle."""
    a = P.make(kind, g, gz)
    b = P.rhs_positive(a.n)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    f.compute_host(a.values, ns)
    v1, _ = f.factors()
    r1 = f.residual_history()
    tb = torch.tensor(b, dtype=torch.float64, device="cuda")
    tx = torch.empty_like(tb)
    f.apply(tb, tx, 3)
    torch.cuda.synchronize()
    x1 = tx.cpu().numpy()
    f.set_values(a.values)
    f.compute(ns)
    v2, _ = f.factors()
    f.apply(tb, tx, 3)
    torch.cuda.synchronize()
    assert np.array_equal(v1, v2)
    assert np.array_equal(x1, tx.cpu().numpy())
    fo = oracle.compute(a, k, ns)
    assert np.array_equal(v1, fo.vals)
    np.testing.assert_allclose(r1, fo.resid, rtol=RTOL_RESID)


def test_compute_host_new_values_and_errors():
    """compute_host with scaled values gives the factors of the scaled matrix (the old values are
    fully replaced), and a zero diagonal is reported like compute's."""
    a = P.laplace3d_27pt(24, gz=70)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
    f.compute(2)
    v2 = a.values * 3.0
    f.compute_host(v2, 2)
    g = F.FastILU(a.row_ptr, a.col_idx, v2, 1)
    g.compute(2)
    assert np.array_equal(f.factors()[0], g.factors()[0])
    z = a.values.copy()
    r = 24 * 24 * 50 + 3
    z[a.row_ptr[r] + int(np.searchsorted(a.col_idx[a.row_ptr[r]:a.row_ptr[r + 1]], r))] = 0.0
    with pytest.raises(F.FastILUError) as ei:
        f.compute_host(z, 2)
    assert ei.value.status == "ZERO_DIAG" and ei.value.index == r


@pytest.mark.parametrize("nt,om_tri", [(4, 1.0), (1, 1.0), (2, 0.8)])
@pytest.mark.parametrize("pipe", [False, True, "tail"])
def test_solve_host_equals_compute_and_apply(nt, om_tri, pipe, monkeypatch):
    """fastilu_solve_host (values + b uploaded on the copy stream in chunks, the last one cut into
    pieces of at least the band) = compute + apply, bitwise.  Default: the apply runs chunk by
    chunk inside the upload pipeline (a chunk's L sweeps as soon as its factors are final, the U
    sweeps along their dependency cone right behind, one buffer per Jacobi iterate, x copied
    back per chunk); FASTILU_SOLVE_NOPIPE=1 runs it after the compute; "tail" uses 8 tail
    pieces."""
    if pipe is False:
        monkeypatch.setenv("FASTILU_SOLVE_NOPIPE", "1")
    if pipe == "tail":
        monkeypatch.setenv("FASTILU_SOLVE_TAIL", "8")
    a = P.laplace3d_27pt(24, gz=70)
    b = P.rhs_positive(a.n)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1, omega_tri=om_tri)
    x1 = f.solve_host(a.values, 3, b, nt)
    f.compute(3)
    x2 = f.apply_host(b, nt)
    assert np.array_equal(x1, x2)
    fo = oracle.compute(a, 1, 3)
    assert np.array_equal(x1, oracle.apply(fo, b, nt, om_tri))
