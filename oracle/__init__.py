"""FastILU CPU oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 implementation of what the FastILU hot
path computes (arXiv 2506.05793 Section 5), used to prove
parity of the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package; the product
package (paper_2506_05793_b200) never does, and this package never imports
the product.  Arithmetic lives in fastilu_oracle.c (compiled -O2
-ffp-contract=off; single thread by default, `set_threads(T)` runs its per-row
loops with OpenMP, bitwise equal to one thread); this file only marshals arrays
(and, for the warm-up, places level L-1's values into S_L).

Pins (tests/test_oracle_*.py, `-m "not gpu"`):
  * symbolic ILU(k): the ten nnz/n values printed in tab:fastilu_nx16/32
    (PAPER.md:596, 660); brute-force fill-path levels on tiny graphs; closed
    forms; k=0 => S = pattern(A); tridiagonal => no fill; dense => dense.
  * exact ILU: tridiagonal ILU(0) == Thomas LU bitwise; dense KIJ elimination
    with dropping == IKJ bitwise; k >= n => LAPACK getrf within 1e-14.
  * sweeps: reach the exact ILU bitwise within the dependency-DAG depth;
    residual non-increasing above the roundoff floor; diagonal A immediate;
    the residual's exact sum == math.fsum bitwise.
  * damped sweeps / Jacobi (omega < 1, reading R1 of PAPER.md:546-548): hand-derived
    iterates of a 3x3 tridiagonal example (tests/golden/damped_3x3.json), a 2x2
    closed form, omega = 0 is the identity, the update is affine in omega.
  * warm-up (R10): an independent dense embedding of S_{L-1} into S_L;
    a pattern with no fill (S_0 = S_1) makes FastILU(0) then FastILU(1) equal to
    one FastILU(0) run of twice the sweeps.
  * trisolve: == substitution after nlevels sweeps (bitwise), T = I, 1 sweep
    = D^-1 b; substitution == scipy solve_triangular.
  * gmres (NEXT row f1): A = I converges in one iteration; an exact LU preconditioner in at
    most two; unpreconditioned SPD systems within n iterations to numpy.linalg.solve;
    iteration counts of SURVEY.md G18's independent computation on the anisotropic problem.
Functions here are all pinned; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fastilu_oracle.c")
_LIB = os.path.join(_HERE, "build", "libfastilu_oracle.so")

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "BAD_MATRIX", 3: "MISSING_DIAG",
          4: "ZERO_DIAG", 5: "ZERO_PIVOT", 9: "OOM"}


class OracleError(RuntimeError):
    def __init__(self, code, index):
        super().__init__(f"oracle status {STATUS.get(code, code)} at index {index}")
        self.code = code
        self.status = STATUS.get(code, str(code))
        self.index = index


def build(force: bool = False) -> str:
    """Compile the oracle C library with gcc (plain -O2, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(_LIB), exist_ok=True)
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)
F64P = C.POINTER(C.c_double)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_validate.argtypes = [C.c_int64, I64P, I32P, I64P]
        L.orc_symbolic.argtypes = [C.c_int64, I64P, I32P, C.c_int, C.POINTER(I64P),
                                   C.POINTER(I32P), C.POINTER(I32P), I64P]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_set_threads.restype = C.c_int
        L.orc_fsum.argtypes = [C.c_int64, F64P]
        L.orc_fsum.restype = C.c_double
        L.orc_scale_init.argtypes = [C.c_int64, I64P, I32P, F64P, I64P, I32P, C.c_double, F64P,
                                     F64P, F64P, I64P]
        L.orc_bad_diagonal.argtypes = [C.c_int64, I64P, I32P, F64P]
        L.orc_bad_diagonal.restype = C.c_int64
        L.orc_sweep.argtypes = [C.c_int64, I64P, I32P, F64P, F64P, F64P, C.c_double, F64P]
        L.orc_sweep.restype = None
        L.orc_compute.argtypes = [C.c_int64, I64P, I32P, F64P, I64P, I32P, C.c_int, C.c_double,
                                  C.c_double, F64P, F64P, F64P, F64P, I64P]
        L.orc_exact_ilu.argtypes = [C.c_int64, I64P, I32P, F64P, F64P, I64P]
        for f in ("orc_jacobi_lower", "orc_jacobi_upper"):
            getattr(L, f).argtypes = [C.c_int64, I64P, I32P, F64P, F64P, C.c_int, C.c_double, F64P]
            getattr(L, f).restype = None
        L.orc_apply.argtypes = [C.c_int64, I64P, I32P, F64P, F64P, F64P, C.c_int, C.c_double, F64P]
        L.orc_apply.restype = None
        for f in ("orc_subst_lower", "orc_subst_upper"):
            getattr(L, f).argtypes = [C.c_int64, I64P, I32P, F64P, F64P, F64P]
            getattr(L, f).restype = None
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Pattern:
    """ILU(k) pattern S: row_ptr int64, col_idx int32, level int32 (row-wise, sorted)."""

    def __init__(self, row_ptr, col_idx, level):
        self.row_ptr, self.col_idx, self.level = row_ptr, col_idx, level
        self.n = row_ptr.shape[0] - 1

    @property
    def nnz(self):
        return int(self.row_ptr[-1])


def set_threads(t: int) -> int:
    """OpenMP threads for the oracle's per-row loops (1 = sequential, the default).  Results are
    bitwise independent of t (per-entry arithmetic is sequential; the residual sum is exact)."""
    return int(lib().orc_set_threads(int(t)))


def fsum(x) -> float:
    """Exactly rounded sum (the oracle's residual accumulator; pinned against math.fsum)."""
    x = _f64(x)
    return float(lib().orc_fsum(x.shape[0], _p(x, F64P)))


def validate(row_ptr, col_idx):
    rp, ci = _i64(row_ptr), _i32(col_idx)
    bad = C.c_int64(-1)
    st = lib().orc_validate(rp.shape[0] - 1, _p(rp, I64P), _p(ci, I32P), C.byref(bad))
    return st, bad.value


def symbolic(row_ptr, col_idx, k: int) -> Pattern:
    """Symbolic ILU(k) by the sum rule, row-wise, ascending pivots (reading R7)."""
    rp, ci = _i64(row_ptr), _i32(col_idx)
    n = rp.shape[0] - 1
    orp, oci, olev = I64P(), I32P(), I32P()
    bad = C.c_int64(-1)
    st = lib().orc_symbolic(n, _p(rp, I64P), _p(ci, I32P), int(k), C.byref(orp), C.byref(oci),
                            C.byref(olev), C.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    nnz = orp[n]
    srp = np.ctypeslib.as_array(orp, shape=(n + 1,)).copy()
    sci = np.ctypeslib.as_array(oci, shape=(max(nnz, 1),))[:nnz].copy()
    slev = np.ctypeslib.as_array(olev, shape=(max(nnz, 1),))[:nnz].copy()
    for p in (orp, oci, olev):
        lib().orc_free(C.cast(p, C.c_void_p))
    return Pattern(srp, sci, slev)


def scale_init(a, pat: Pattern, shift: float = 0.0):
    """Returns (s, ahat_S, vals0_S) -- readings R4, R5 (R9: Manteuffel shift)."""
    rp, ci, av = _i64(a.row_ptr), _i32(a.col_idx), _f64(a.values)
    n = a.n
    s = np.empty(n)
    ahat = np.empty(pat.nnz)
    vals = np.empty(pat.nnz)
    bad = C.c_int64(-1)
    st = lib().orc_scale_init(n, _p(rp, I64P), _p(ci, I32P), _p(av, F64P), _p(pat.row_ptr, I64P),
                              _p(pat.col_idx, I32P), float(shift), _p(s, F64P), _p(ahat, F64P),
                              _p(vals, F64P), C.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    return s, ahat, vals


def sweep(pat: Pattern, ahat, old, omega: float = 1.0):
    """One synchronous sweep; returns (new, r(s-1))."""
    ahat, old = _f64(ahat), _f64(old)
    out = np.empty_like(old)
    r = C.c_double(0.0)
    lib().orc_sweep(pat.n, _p(pat.row_ptr, I64P), _p(pat.col_idx, I32P), _p(ahat, F64P),
                    _p(old, F64P), _p(out, F64P), float(omega), C.byref(r))
    return out, r.value


def bad_diagonal(pat: Pattern, vals) -> int:
    vals = _f64(vals)
    return int(lib().orc_bad_diagonal(pat.n, _p(pat.row_ptr, I64P), _p(pat.col_idx, I32P),
                                      _p(vals, F64P)))


class Factors:
    def __init__(self, pat, s, ahat, vals, resid):
        self.pattern, self.s, self.ahat, self.vals, self.resid = pat, s, ahat, vals, resid


def compute(a, k: int, nsweeps: int, omega: float = 1.0, pat: Pattern | None = None,
            shift: float = 0.0) -> Factors:
    """Symbolic + scale/init + nsweeps synchronous sweeps (whole FastILU compute); shift is the
    Manteuffel shift of reading R9."""
    if pat is None:
        pat = symbolic(a.row_ptr, a.col_idx, k)
    rp, ci, av = _i64(a.row_ptr), _i32(a.col_idx), _f64(a.values)
    n = a.n
    s = np.empty(n)
    ahat = np.empty(pat.nnz)
    vals = np.empty(pat.nnz)
    hist = np.zeros(max(nsweeps, 1))
    bad = C.c_int64(-1)
    st = lib().orc_compute(n, _p(rp, I64P), _p(ci, I32P), _p(av, F64P), _p(pat.row_ptr, I64P),
                           _p(pat.col_idx, I32P), int(nsweeps), float(omega), float(shift),
                           _p(s, F64P),
                           _p(ahat, F64P), _p(vals, F64P), _p(hist, F64P), C.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    return Factors(pat, s, ahat, vals, hist[:nsweeps].copy())


def compute_tol(a, k: int, rtol: float, max_sweeps: int = 100, omega: float = 1.0):
    """Sweeps to convergence (reading G15): sweep s yields r(s-1); stop after the first
    s with r(s-1) <= rtol * ||Ahat|_S||_F, or after max_sweeps.  Returns (Factors, s)."""
    pat = symbolic(a.row_ptr, a.col_idx, k)
    s, ahat, vals = scale_init(a, pat)
    thr = rtol * float(np.sqrt(np.sum(ahat * ahat)))
    hist = []
    sw = 0
    for sw in range(1, max_sweeps + 1):
        vals, r = sweep(pat, ahat, vals, omega)
        hist.append(r)
        if r <= thr:
            break
    return Factors(pat, s, ahat, vals, np.array(hist)), sw


def compute_warmup(a, k: int, nsweeps: int, omega: float = 1.0, shift: float = 0.0):
    """Option "Warm up" (R10): FastILU(L) for L = 0..k, nsweeps each;
    the factors of level L-1 initialise the entries of S_{L-1} inside S_L, new fill entries
    start at +0.0, level 0 starts from the initial guess (R4).  Residual history concatenated."""
    hist = []
    prev = None
    for L in range(k + 1):
        pat = symbolic(a.row_ptr, a.col_idx, L)
        s, ahat, vals = scale_init(a, pat, shift)
        if prev is not None:
            ppat, pvals = prev
            key = np.repeat(np.arange(pat.n, dtype=np.int64), np.diff(pat.row_ptr)) * pat.n \
                + pat.col_idx
            pkey = np.repeat(np.arange(ppat.n, dtype=np.int64), np.diff(ppat.row_ptr)) * ppat.n \
                + ppat.col_idx
            pos = np.searchsorted(key, pkey)
            assert np.array_equal(key[pos], pkey)  # S_{L-1} is contained in S_L
            vals = np.zeros(pat.nnz)
            vals[pos] = pvals
        for _ in range(nsweeps):
            vals, r = sweep(pat, ahat, vals, omega)
            hist.append(r)
        prev = (pat, vals)
    return Factors(pat, s, ahat, vals, np.array(hist))


def exact_ilu(pat: Pattern, ahat):
    ahat = _f64(ahat)
    vals = np.empty_like(ahat)
    bad = C.c_int64(-1)
    st = lib().orc_exact_ilu(pat.n, _p(pat.row_ptr, I64P), _p(pat.col_idx, I32P), _p(ahat, F64P),
                             _p(vals, F64P), C.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    return vals


def jacobi_lower(pat: Pattern, vals, y, ntri: int, omega: float = 1.0):
    vals, y = _f64(vals), _f64(y)
    z = np.empty(pat.n)
    lib().orc_jacobi_lower(pat.n, _p(pat.row_ptr, I64P), _p(pat.col_idx, I32P), _p(vals, F64P),
                           _p(y, F64P), int(ntri), float(omega), _p(z, F64P))
    return z


def jacobi_upper(pat: Pattern, vals, z, ntri: int, omega: float = 1.0):
    vals, z = _f64(vals), _f64(z)
    w = np.empty(pat.n)
    lib().orc_jacobi_upper(pat.n, _p(pat.row_ptr, I64P), _p(pat.col_idx, I32P), _p(vals, F64P),
                           _p(z, F64P), int(ntri), float(omega), _p(w, F64P))
    return w


def apply(f: Factors, b, ntri: int, omega_tri: float = 1.0):
    """x = s o U^-1 L^-1 (s o b) with ntri Jacobi sweeps per factor (R5, R6)."""
    b = _f64(b)
    s = _f64(f.s)
    x = np.empty(f.pattern.n)
    p = f.pattern
    lib().orc_apply(p.n, _p(p.row_ptr, I64P), _p(p.col_idx, I32P), _p(_f64(f.vals), F64P),
                    _p(s, F64P), _p(b, F64P), int(ntri), float(omega_tri), _p(x, F64P))
    return x


def subst_lower(pat: Pattern, vals, y):
    vals, y = _f64(vals), _f64(y)
    z = np.empty(pat.n)
    lib().orc_subst_lower(pat.n, _p(pat.row_ptr, I64P), _p(pat.col_idx, I32P), _p(vals, F64P),
                          _p(y, F64P), _p(z, F64P))
    return z


def subst_upper(pat: Pattern, vals, z):
    vals, z = _f64(vals), _f64(z)
    w = np.empty(pat.n)
    lib().orc_subst_upper(pat.n, _p(pat.row_ptr, I64P), _p(pat.col_idx, I32P), _p(vals, F64P),
                          _p(z, F64P), _p(w, F64P))
    return w


def spmv(a, v):
    """y = A v for a CSR matrix (plain loop over rows in numpy, row sums left to right)."""
    v = _f64(v)
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    return np.bincount(rows, weights=a.values * v[a.col_idx], minlength=a.n)


def gmres(a, b, precond, restart: int = 60, rtol: float = 1e-6, max_iters: int = 1000):
    """Restarted GMRES(m), right preconditioning x = M^-1 y, modified Gram-Schmidt, Givens
    rotations, x0 = 0, converged when ||b - A x|| / ||b|| <= rtol (the paper's
    protocol: GMRES(60), six orders of magnitude).  `precond(v)` applies M^-1.
    Returns (x, inner iterations, final relative residual)."""
    b = _f64(b)
    n = b.shape[0]
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return x, 0, 0.0
    r = b.copy()
    beta = bnorm
    total = 0
    while beta / bnorm > rtol and total < max_iters:
        V = np.zeros((restart + 1, n))
        Hm = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        V[0] = r / beta
        j = 0
        while j < restart and total < max_iters:
            w = spmv(a, precond(V[j]))
            for q in range(j + 1):  # modified Gram-Schmidt
                Hm[q, j] = float(np.dot(V[q], w))
                w = w - Hm[q, j] * V[q]
            Hm[j + 1, j] = float(np.linalg.norm(w))
            if Hm[j + 1, j] > 0.0:
                V[j + 1] = w / Hm[j + 1, j]
            for q in range(j):
                t = cs[q] * Hm[q, j] + sn[q] * Hm[q + 1, j]
                Hm[q + 1, j] = -sn[q] * Hm[q, j] + cs[q] * Hm[q + 1, j]
                Hm[q, j] = t
            rr = float(np.hypot(Hm[j, j], Hm[j + 1, j]))
            cs[j], sn[j] = (Hm[j, j] / rr, Hm[j + 1, j] / rr) if rr > 0 else (1.0, 0.0)
            Hm[j, j], Hm[j + 1, j] = rr, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            j += 1
            if abs(g[j]) <= rtol * bnorm or Hm[j, j - 1] == 0.0 and rr == 0.0:
                break
        y = np.zeros(j)
        for q in range(j - 1, -1, -1):
            y[q] = (g[q] - np.dot(Hm[q, q + 1:j], y[q + 1:j])) / Hm[q, q]
        x = x + precond(V[:j].T @ y)
        r = b - spmv(a, x)
        beta = float(np.linalg.norm(r))
    return x, total, beta / bnorm


def fastilu_preconditioner(f: "Factors", ntri: int, omega_tri: float = 1.0):
    """M^-1 v = s o U^-1 L^-1 (s o v) with ntri Jacobi sweeps per factor (the FastILU apply)."""
    return lambda v: apply(f, v, ntri, omega_tri)


def exact_preconditioner(f: "Factors"):
    """M^-1 v = s o U^-1 L^-1 (s o v) by exact substitution (config 5 arm C)."""
    def pre(v):
        z = subst_lower(f.pattern, f.vals, f.s * _f64(v))
        return f.s * subst_upper(f.pattern, f.vals, z)
    return pre


def windowed(a_full, plane: int, lo_plane: int, hi_plane: int, k: int, nsweeps: int,
             b_full=None, ntri: int = 0, omega: float = 1.0, omega_tri: float = 1.0):
    """Windowed oracle for stencil problems in natural z-plane order (DESIGN.md "windowed
    oracle"): runs the whole path on rows/cols of planes [lo_plane, hi_plane) of `a_full`
    and returns (row_lo, row_hi) of the window plus the Factors / x for the window.
    Callers compare only planes far enough from the cut (margins in DESIGN.md)."""
    from problems import submatrix  # data slicing only, no method arithmetic
    lo, hi = lo_plane * plane, hi_plane * plane
    sub = submatrix(a_full, lo, hi)
    f = compute(sub, k, nsweeps, omega)
    x = None
    if b_full is not None:
        x = apply(f, np.asarray(b_full)[lo:hi], ntri, omega_tri)
    return lo, hi, f, x
