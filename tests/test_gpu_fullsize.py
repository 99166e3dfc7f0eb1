"""Full-size parity at BASELINE.json's sizes, in the launch configuration bench.py times.

The whole path runs on the GPU at full size; the oracle recomputes sampled planes exactly with
its windowed mode: rows and columns of a slab of planes around the
sample, margins of nsweeps + ntri + k + 4 planes below and ntri + 2 above (pinned bitwise in
tests/test_oracle_numeric.py::test_windowed_equals_global_interior).  Sampled factors must be
bitwise equal and sampled x within 1e-12 per entry (in practice bitwise too)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2506_05793_b200 as F
import problems as P

pytestmark = pytest.mark.gpu


def run_full(kind, g, k, ns, nt):
    a = P.make(kind, g)
    b = P.rhs_positive(a.n)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    f.compute(ns)
    tb = torch.tensor(b, device="cuda")
    tx = torch.empty_like(tb)
    f.apply(tb, tx, nt)
    torch.cuda.synchronize()
    vals, s = f.factors()
    rp, ci, _ = f.pattern()
    return a, b, f, vals, s, rp, ci, tx.cpu().numpy()


@pytest.fixture(autouse=True)
def oracle_threads():
    """The windowed oracle on all host cores (bitwise the 1-thread oracle)."""
    import os
    oracle.set_threads(len(os.sched_getaffinity(0)))
    yield
    oracle.set_threads(1)


def check_planes(a, b, kind, g, k, ns, nt, planes, vals, rp, ci, x):
    plane = g * g
    for z in planes:
        lo_p = max(0, z - (ns + nt + k + 4))
        hi_p = min(g, z + nt + 3)
        lo, hi, fw, xw = oracle.windowed(a, plane, lo_p, hi_p, k, ns, b_full=b, ntri=nt)
        r0, r1 = z * plane, (z + 1) * plane
        wrp = fw.pattern.row_ptr
        g_vals = vals[rp[r0]:rp[r1]]
        o_vals = fw.vals[wrp[r0 - lo]:wrp[r1 - lo]]
        assert np.array_equal(ci[rp[r0]:rp[r1]], fw.pattern.col_idx[wrp[r0 - lo]:wrp[r1 - lo]] + lo)
        assert np.array_equal(g_vals, o_vals), f"plane {z}: factors differ"
        xo = xw[r0 - lo:r1 - lo]
        xg = x[r0:r1]
        assert np.all(np.abs(xg - xo) <= 1e-12 * np.abs(xo)), f"plane {z}: x differs"


@pytest.mark.parametrize("k", [1, 2])
def test_config3_27pt_128(k):
    g, ns, nt = 128, 3, 5
    a, b, f, vals, s, rp, ci, x = run_full("27pt", g, k, ns, nt)
    assert f.info().startswith("path=tsell")
    check_planes(a, b, "27pt", g, k, ns, nt, [1, 64, 126], vals, rp, ci, x)


def test_config3_to_convergence_128():
    """Config 3 'sweeps to convergence' at full size (reading G15): the stopping rule
    r(s*-1) <= 1e-10 ||Ahat|_S||_F < r(s*-2) and a monotone residual history.  ||Ahat|_S||_F is
    computed here from its definition, sum over A of a_ij^2 / (|a_ii| |a_jj|)."""
    a = P.laplace3d_27pt(128)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 1)
    s_star = f.compute_tol(1e-10, 100)
    h = f.residual_history()
    assert len(h) == s_star and 10 < s_star < 100
    assert np.all(np.diff(h) < 0)
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    d = np.zeros(a.n)
    d[rows[a.col_idx == rows]] = np.abs(a.values[a.col_idx == rows])
    norm = np.sqrt(np.sum(a.values ** 2 / (d[rows] * d[a.col_idx])))
    thr = 1e-10 * norm
    assert h[-1] <= thr * (1 + 1e-9) and h[-2] > thr * (1 - 1e-9)


def test_config3_to_convergence_128_windowed_oracle():
    """Config 3a 'to convergence' (reading G15) at full size: the GPU's factors at its stopping
    sweep s* and x after 5 + 5 Jacobi sweeps equal the windowed oracle's at the same s*, bitwise,
    on the middle plane (margins: s* + ntri + k + 4 planes below)."""
    g, k, nt = 128, 1, 5
    a = P.laplace3d_27pt(g)
    b = P.rhs_positive(a.n)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    s_star = f.compute_tol(1e-10, 100)
    tb = torch.tensor(b, device="cuda")
    tx = torch.empty_like(tb)
    f.apply(tb, tx, nt)
    torch.cuda.synchronize()
    vals, _ = f.factors()
    rp, ci, _ = f.pattern()
    check_planes(a, b, "27pt", g, k, s_star, nt, [64], vals, rp, ci, tx.cpu().numpy())


def test_config4_27pt_256():
    g, k, ns, nt = 256, 1, 3, 5
    a, b, f, vals, s, rp, ci, x = run_full("27pt", g, k, ns, nt)
    assert f.info().startswith("path=tsell")
    # first and last planes (TMA zero-fill below plane 0, the last tile's tail) and the middle
    check_planes(a, b, "27pt", g, k, ns, nt, [0, 128, 255], vals, rp, ci, x)
    # the e2e entry bench.py times (fastilu_solve_host: values + b uploaded in chunks, the sweeps,
    # the Jacobi L sweeps and the U cone pipelined behind the upload, x copied back per chunk)
    # returns the same x, bitwise, and leaves the same factors
    av = torch.from_numpy(a.values).pin_memory().numpy()
    bh = torch.from_numpy(b).pin_memory().numpy()
    xh = torch.empty(a.n, dtype=torch.float64).pin_memory().numpy()
    f.solve_host(av, ns, bh, nt, out=xh)
    assert np.array_equal(xh, x)
    v2, _ = f.factors()
    assert np.array_equal(v2, vals)


def test_config2_7pt_128_exact():
    g, k, ns, nt = 128, 0, 3, 5
    a, b, f, vals, s, rp, ci, x = run_full("7pt", g, k, ns, nt)
    check_planes(a, b, "7pt", g, k, ns, nt, [0, 77, 127], vals, rp, ci, x)


def test_config5_aniso7pt_256():
    """BASELINE configs[4] at full size: anisotropic 7-pt 256^3 ILU(0), 2 sweeps + 5/5 Jacobi
    (the register-pivot template path), sampled planes bitwise against the windowed oracle."""
    g, k, ns, nt = 256, 0, 2, 5
    a, b, f, vals, s, rp, ci, x = run_full("aniso7pt", g, k, ns, nt)
    assert f.info().startswith("path=tsell")
    check_planes(a, b, "aniso7pt", g, k, ns, nt, [0, 131, 255], vals, rp, ci, x)
