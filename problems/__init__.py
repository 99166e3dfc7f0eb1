"""Seeded synthetic inputs shared by the oracle side and the product side.

This module holds NO arithmetic of the FastILU method: it only assembles the
model matrices in CSR form and draws the seeded vectors.  Both the oracle
(oracle/) and the CUDA path (paper_2506_05793_b200/) are fed from here; neither
imports the other.

Workloads (BASELINE.json `configs`; recipe in DESIGN.md "Inputs"):
  * 3D 7-point Laplacian on a g^3 grid, natural (lexicographic, x fastest)
    ordering, Dirichlet truncation: diagonal 2(cx+cy+cz), off-diagonals -c_axis
    (isotropic: 6 / -1; anisotropic config 5: (cx,cy,cz) = (1, 0.01, 0.01)).
  * 3D 27-point Laplacian: diagonal 26, the 26 neighbours -1 (HPCG convention).
  * 3-dof-per-node 27-point pattern (the paper's "3D Elasticity problem on a
    27-point stencil"): dense 3x3 node blocks.  Only its pattern
    is pinned by the paper (nnz/n rows of tab:fastilu_nx16/32, PAPER.md:596,
    660); values are diagonally dominant placeholders.
  * right-hand sides: b ~ U[0.5, 1.5) (positive, see DESIGN.md tolerance
    reading) from numpy.random.default_rng(20250605); GMRES x_true ~ U[0,1).
"""
from __future__ import annotations

import numpy as np

SEED = 20250605


class Csr:
    """Plain CSR triple: row_ptr int64[n+1], col_idx int32[nnz], values f64[nnz]."""

    __slots__ = ("n", "row_ptr", "col_idx", "values")

    def __init__(self, row_ptr, col_idx, values):
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.n = int(self.row_ptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n, self.n))
        for i in range(self.n):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            d[i, self.col_idx[s:e]] = self.values[s:e]
        return d


def _stencil(g: int, offsets, weights, diag: float, gz: int | None = None,
             planes: tuple[int, int] | None = None) -> Csr:
    """Assemble a 3D stencil operator on a g x g x gz grid (x fastest).

    offsets: list of (dx, dy, dz); weights: value of each off-diagonal entry.
    Out-of-grid neighbours are dropped (Dirichlet truncation).
    planes=(z0, z1): only the rows of planes z0..z1-1, with GLOBAL column indices (a row block
    of the global matrix, used by the multi-GPU row partition).
    """
    gz = g if gz is None else gz
    z0, z1 = (0, gz) if planes is None else planes
    n = g * g * (z1 - z0)
    ents = [((0, 0, 0), diag)] + list(zip(offsets, weights))
    # increasing column order == increasing linear offset dz*g^2 + dy*g + dx
    ents.sort(key=lambda e: e[0][2] * g * g + e[0][1] * g + e[0][0])
    rows = np.arange(n, dtype=np.int64) + z0 * g * g
    x = rows % g
    y = (rows // g) % g
    z = rows // (g * g)
    masks = []
    for (dx, dy, dz), _w in ents:
        m = np.ones(n, dtype=bool)
        if dx:
            m &= (x + dx >= 0) & (x + dx < g)
        if dy:
            m &= (y + dy >= 0) & (y + dy < g)
        if dz:
            m &= (z + dz >= 0) & (z + dz < gz)
        masks.append(m)
    counts = np.zeros(n, dtype=np.int64)
    for m in masks:
        counts += m
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    nnz = int(rp[-1])
    ci = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    fill = rp[:-1].copy()
    for ((dx, dy, dz), w), m in zip(ents, masks):
        off = dz * g * g + dy * g + dx
        r = rows[m]
        pos = fill[m]
        ci[pos] = (r + off).astype(np.int32)
        vals[pos] = w
        fill[m] += 1
    return Csr(rp, ci, vals)


AXIS6 = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
CUBE26 = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
          if (dx, dy, dz) != (0, 0, 0)]


def laplace3d_7pt(g: int, coeffs=(1.0, 1.0, 1.0), gz: int | None = None, planes=None) -> Csr:
    cx, cy, cz = coeffs
    w = [-cx, -cx, -cy, -cy, -cz, -cz]
    return _stencil(g, AXIS6, w, 2.0 * (cx + cy + cz), gz, planes)


def laplace3d_27pt(g: int, gz: int | None = None, planes=None) -> Csr:
    return _stencil(g, CUBE26, [-1.0] * 26, 26.0, gz, planes)


ANISO_COEFFS = (1.0, 0.01, 0.01)


def aniso3d_7pt(g: int, gz: int | None = None, planes=None) -> Csr:
    return laplace3d_7pt(g, ANISO_COEFFS, gz, planes)


def elasticity_pattern_3dof(g: int) -> Csr:
    """3 dofs per node, dense 3x3 blocks on the 27-point node graph.

    Dof d of node v is row 3v+d.  Values: 80 on the diagonal, -1 elsewhere
    (diagonally dominant placeholder; only the pattern is pinned by the paper).
    """
    node = laplace3d_27pt(g)
    nn = node.n
    cnt = np.diff(node.row_ptr)
    rp = np.zeros(3 * nn + 1, dtype=np.int64)
    np.cumsum(np.repeat(cnt * 3, 3), out=rp[1:])
    ci = np.empty(int(rp[-1]), dtype=np.int32)
    vals = np.full(int(rp[-1]), -1.0)
    for v in range(nn):
        cols = node.col_idx[node.row_ptr[v]:node.row_ptr[v + 1]].astype(np.int64)
        blk = (3 * cols[:, None] + np.arange(3)[None, :]).ravel()
        for d in range(3):
            r = 3 * v + d
            s = rp[r]
            ci[s:s + blk.size] = blk
            vals[s + np.searchsorted(blk, r)] = 80.0
    return Csr(rp, ci, vals)


def multi_dof_pattern(g: int, dofs: int, seed: int | None = None) -> Csr:
    """`dofs` unknowns per node, dense dofs x dofs blocks on the 27-point node graph (as
    elasticity_pattern_3dof, any block size).  Off-diagonal values -1, or, with a seed,
    -U[0.5, 1.5); diagonal 27 dofs + 1 + (seeded: U[0, 1)), so rows are strictly dominant."""
    node = laplace3d_27pt(g)
    nn = node.n
    cnt = np.diff(node.row_ptr)
    rp = np.zeros(dofs * nn + 1, dtype=np.int64)
    np.cumsum(np.repeat(cnt * dofs, dofs), out=rp[1:])
    ci = np.empty(int(rp[-1]), dtype=np.int32)
    rng = np.random.default_rng(seed) if seed is not None else None
    vals = -rng.uniform(0.5, 1.5, size=int(rp[-1])) if rng is not None else np.full(int(rp[-1]), -1.0)
    for v in range(nn):
        cols = node.col_idx[node.row_ptr[v]:node.row_ptr[v + 1]].astype(np.int64)
        blk = (dofs * cols[:, None] + np.arange(dofs)[None, :]).ravel()
        for d in range(dofs):
            r = dofs * v + d
            s = rp[r]
            ci[s:s + blk.size] = blk
            vals[s + np.searchsorted(blk, r)] = 27.0 * dofs + 1.0 + (rng.uniform() if rng else 0.0)
    return Csr(rp, ci, vals)


def tridiagonal(n: int, seed: int = SEED) -> Csr:
    """Random diagonally dominant tridiagonal matrix (values seeded)."""
    rng = np.random.default_rng(seed)
    rp = [0]
    ci = []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                ci.append(j)
        rp.append(len(ci))
    vals = -rng.uniform(0.1, 1.0, size=len(ci))
    rp = np.array(rp, dtype=np.int64)
    ci = np.array(ci, dtype=np.int32)
    for i in range(n):
        s, e = rp[i], rp[i + 1]
        d = s + int(np.searchsorted(ci[s:e], i))
        vals[d] = 3.0 + rng.uniform(0.0, 1.0)
    return Csr(rp, ci, vals)


def banded(n: int, offsets, seed: int = SEED) -> Csr:
    """Diagonally dominant matrix with the given column offsets j - i (0 included; entries
    outside [0, n) dropped), off-diagonal values -U[0.1, 1.0) (seeded): a template pattern whose
    pivots need not lie next to the row (edge cases of the template-SELL kernels)."""
    offs = sorted(set(int(o) for o in offsets) | {0})
    rng = np.random.default_rng(seed)
    rp = [0]
    ci = []
    for i in range(n):
        ci.extend(i + o for o in offs if 0 <= i + o < n)
        rp.append(len(ci))
    rp = np.array(rp, dtype=np.int64)
    ci = np.array(ci, dtype=np.int32)
    vals = -rng.uniform(0.1, 1.0, size=ci.size)
    for i in range(n):
        s, e = rp[i], rp[i + 1]
        vals[s + int(np.searchsorted(ci[s:e], i))] = float(len(offs)) + rng.uniform(0.0, 1.0)
    return Csr(rp, ci, vals)


def random_sparse(n: int, density: float, seed: int = SEED, dominant: bool = True) -> Csr:
    """Random sparse matrix with a full diagonal; M-matrix-like when dominant."""
    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, True)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(1), out=rp[1:])
    ci = np.nonzero(mask)[1].astype(np.int32)
    vals = -rng.uniform(0.0, 1.0, size=ci.size)
    for i in range(n):
        s, e = rp[i], rp[i + 1]
        d = s + int(np.searchsorted(ci[s:e], i))
        vals[d] = (float(e - s) + 1.0) if dominant else rng.uniform(0.5, 1.5)
    return Csr(rp, ci, vals)


def submatrix(a: Csr, lo: int, hi: int) -> Csr:
    """Rows and columns [lo, hi) of `a` (plain CSR slicing, used for windows)."""
    rp = a.row_ptr
    s, e = int(rp[lo]), int(rp[hi])
    ci = a.col_idx[s:e].astype(np.int64)
    vals = a.values[s:e]
    keep = (ci >= lo) & (ci < hi)
    rows = np.repeat(np.arange(hi - lo), np.diff(rp[lo:hi + 1]))
    cnt = np.bincount(rows[keep], minlength=hi - lo)
    nrp = np.zeros(hi - lo + 1, dtype=np.int64)
    np.cumsum(cnt, out=nrp[1:])
    return Csr(nrp, (ci[keep] - lo).astype(np.int32), vals[keep])


def bandwidth(kind: str, g: int) -> int:
    """Half bandwidth max |i - j| of the stencil matrices in natural order."""
    return g * g + (g + 1 if kind == "27pt" else 0)


def row_block(a: Csr, r0: int, r1: int) -> Csr:
    """Rows [r0, r1) of `a` with their global column indices (plain CSR slicing)."""
    s, e = int(a.row_ptr[r0]), int(a.row_ptr[r1])
    return Csr(a.row_ptr[r0:r1 + 1] - s, a.col_idx[s:e], a.values[s:e])


def rhs_positive(n: int, seed: int = SEED) -> np.ndarray:
    """b ~ U[0.5, 1.5) (positive b keeps Jacobi terms one-signed)."""
    return np.random.default_rng(seed).uniform(0.5, 1.5, size=n)


def rhs_signed(n: int, seed: int = SEED) -> np.ndarray:
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=n)


def x_true(n: int, seed: int = SEED) -> np.ndarray:
    """GMRES exact solution ~ U[0,1) ("solution is a vector of random variables")."""
    return np.random.default_rng(seed).uniform(0.0, 1.0, size=n)


WORKLOADS = {
    # name: (generator, grid, level k, nsweeps, ntrisweeps)   BASELINE.json configs
    "c1_7pt_10_ilu0": ("7pt", 10, 0, 3, 5),
    "c2_7pt_128_ilu0": ("7pt", 128, 0, 3, 5),
    "c3a_27pt_128_ilu1": ("27pt", 128, 1, 3, 5),
    "c3b_27pt_128_ilu2": ("27pt", 128, 2, 3, 5),
    "c4_27pt_256_ilu1": ("27pt", 256, 1, 3, 5),
    "c5_aniso7pt_256_ilu0": ("aniso7pt", 256, 0, 2, 5),
    # the paper's own FastILU(3) problem of tab:fastilu_sweep: 3-dof 27-pt
    # pattern on 32^3 nodes (n = 98,304, nnz(S) = 45,729,504); context workload only
    "t6_3dof_32_ilu3": ("3dof", 32, 3, 3, 5),
}


def make(kind: str, g: int, gz: int | None = None, planes=None) -> Csr:
    if kind == "3dof" and (gz is not None or planes is not None):
        raise ValueError("the 3-dof pattern is generated on full g^3 grids only")
    if kind == "7pt":
        return laplace3d_7pt(g, gz=gz, planes=planes)
    if kind == "27pt":
        return laplace3d_27pt(g, gz=gz, planes=planes)
    if kind == "aniso7pt":
        return aniso3d_7pt(g, gz=gz, planes=planes)
    if kind == "3dof":
        return elasticity_pattern_3dof(g)
    raise ValueError(kind)
