"""Pins for the oracle's symbolic ILU(k) (reading R7), independent of the oracle itself.

* values the paper prints: nnz/n of ILU(k), k=0..4, on the 3-dof 27-point pattern at 16^3 and
  32^3 (tests/golden/paper_nnz_per_n.json);
* brute force: Hysom-Pothen fill-path levels (shortest path through lower-numbered vertices)
  computed by BFS on tiny random directed graphs;
* closed forms: 7-pt ILU(0) = 7g^3 - 6g^2, 27-pt ILU(0) = (3g-2)^3, plus the ILU(1)/ILU(2)
  polynomials of SURVEY.md Sec. 8(a) (fitted there by an independent script);
* special cases: k=0 => S = pattern(A); tridiagonal => no fill at any k; dense => dense.
"""
import json
import os
from collections import deque

import numpy as np
import pytest

import oracle
import problems as P

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_nnz_per_n.json")


def _rows(pat):
    return [pat.col_idx[pat.row_ptr[i]:pat.row_ptr[i + 1]].tolist() for i in range(pat.n)]


def test_paper_nnz_per_n_16():
    gold = json.load(open(GOLD))
    tol = gold["printed_precision"]
    e = P.elasticity_pattern_3dof(16)
    assert e.n == gold["grids"]["16"]["n"]
    for k, want in enumerate(gold["grids"]["16"]["nnz_per_n"]):
        pat = oracle.symbolic(e.row_ptr, e.col_idx, k)
        got = pat.nnz / e.n
        assert abs(got - want) <= tol, (k, got, want)
        assert round(got, 1) == pytest.approx(want), (k, got, want)


def _block_expand_count(node_pat):
    return 9 * node_pat.nnz


def test_block_expansion_equivalence_16():
    """Scalar ILU(k) of the dense-3x3-block matrix == block expansion of the node-graph
    ILU(k), entry by entry and level by level (checked directly at 16^3, k = 0..4)."""
    e = P.elasticity_pattern_3dof(16)
    node = P.laplace3d_27pt(16)
    for k in range(5):
        ps = oracle.symbolic(e.row_ptr, e.col_idx, k)
        pn = oracle.symbolic(node.row_ptr, node.col_idx, k)
        cnt = np.diff(pn.row_ptr)
        rp = np.zeros(3 * node.n + 1, dtype=np.int64)
        np.cumsum(np.repeat(3 * cnt, 3), out=rp[1:])
        assert np.array_equal(rp, ps.row_ptr)
        for v in (0, 1, 17, 300, 2000, node.n - 1):
            cols = pn.col_idx[pn.row_ptr[v]:pn.row_ptr[v + 1]].astype(np.int64)
            levs = pn.level[pn.row_ptr[v]:pn.row_ptr[v + 1]]
            blk = (3 * cols[:, None] + np.arange(3)[None, :]).ravel()
            blev = np.repeat(levs, 3)
            for d in range(3):
                r = 3 * v + d
                s, t = ps.row_ptr[r], ps.row_ptr[r + 1]
                assert np.array_equal(ps.col_idx[s:t], blk)
                assert np.array_equal(ps.level[s:t], blev)


def test_paper_nnz_per_n_32():
    gold = json.load(open(GOLD))
    tol = gold["printed_precision"]
    node = P.laplace3d_27pt(32)
    n3 = 3 * node.n
    assert n3 == gold["grids"]["32"]["n"]
    for k, want in enumerate(gold["grids"]["32"]["nnz_per_n"]):
        pn = oracle.symbolic(node.row_ptr, node.col_idx, k)
        got = _block_expand_count(pn) / n3
        assert abs(got - want) <= tol, (k, got, want)
    e = P.elasticity_pattern_3dof(32)
    for k in (0, 1):
        ps = oracle.symbolic(e.row_ptr, e.col_idx, k)
        want = gold["grids"]["32"]["nnz_per_n"][k]
        assert abs(ps.nnz / e.n - want) <= tol


def _bfs_levels(dense_pattern, K):
    """Fill-path theorem (Hysom & Pothen): lev(i,j) = (length of the shortest directed path
    i -> j in the graph of A whose intermediate vertices are all < min(i,j)) - 1."""
    n = dense_pattern.shape[0]
    adj = [np.nonzero(dense_pattern[u])[0].tolist() for u in range(n)]
    lev = {}
    for i in range(n):
        for j in range(n):
            if i == j:
                lev[(i, j)] = 0
                continue
            m = min(i, j)
            dist = {i: 0}
            dq = deque([i])
            found = None
            while dq:
                u = dq.popleft()
                for v in adj[u]:
                    if v == j:
                        found = dist[u] + 1
                        break
                    if v < m and v not in dist:
                        dist[v] = dist[u] + 1
                        dq.append(v)
                if found is not None:
                    break
            if found is not None and found - 1 <= K:
                lev[(i, j)] = found - 1
    return lev


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("K", [0, 1, 2, 3])
def test_bruteforce_fill_paths(seed, K):
    a = P.random_sparse(24, 0.08, seed=seed)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, K)
    d = a.to_dense() != 0
    want = _bfs_levels(d, K)
    got = {}
    for i in range(pat.n):
        for p in range(pat.row_ptr[i], pat.row_ptr[i + 1]):
            got[(i, int(pat.col_idx[p]))] = int(pat.level[p])
    assert got == want


@pytest.mark.parametrize("g", [3, 4, 5, 6, 7, 9])
def test_closed_forms(g):
    a7 = P.laplace3d_7pt(g)
    assert oracle.symbolic(a7.row_ptr, a7.col_idx, 0).nnz == 7 * g**3 - 6 * g**2
    a27 = P.laplace3d_27pt(g)
    assert oracle.symbolic(a27.row_ptr, a27.col_idx, 0).nnz == (3 * g - 2) ** 3
    assert oracle.symbolic(a27.row_ptr, a27.col_idx, 1).nnz == 63 * g**3 - 194 * g**2 + 204 * g - 72
    if g >= 4:
        assert oracle.symbolic(a27.row_ptr, a27.col_idx, 2).nnz == \
            115 * g**3 - 474 * g**2 + 648 * g - 288


@pytest.mark.parametrize("seed", [5, 6])
def test_k0_is_pattern_of_A_and_levels(seed):
    a = P.random_sparse(60, 0.05, seed=seed)
    p0 = oracle.symbolic(a.row_ptr, a.col_idx, 0)
    assert np.array_equal(p0.row_ptr, a.row_ptr)
    assert np.array_equal(p0.col_idx, a.col_idx)
    assert np.all(p0.level == 0)
    prev = _rows(p0)
    for k in (1, 2, 3):
        pk = oracle.symbolic(a.row_ptr, a.col_idx, k)
        rows = _rows(pk)
        assert all(set(r0) <= set(r1) for r0, r1 in zip(prev, rows))  # S_k grows with k
        assert pk.level.max() <= k
        prev = rows


@pytest.mark.parametrize("k", [0, 1, 2, 5])
def test_tridiagonal_has_no_fill(k):
    # tridiagonal LU creates no fill (SPEC.md:362's "pentadiagonal" example is wrong)
    a = P.tridiagonal(17)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, k)
    assert np.array_equal(pat.row_ptr, a.row_ptr) and np.array_equal(pat.col_idx, a.col_idx)


def test_dense_stays_dense():
    a = P.random_sparse(12, 1.0)
    for k in (0, 3):
        pat = oracle.symbolic(a.row_ptr, a.col_idx, k)
        assert pat.nnz == 144 and np.all(pat.level == 0)


def test_arrow_fill_full_at_k1():
    # arrow matrix with the dense row/col FIRST: eliminating vertex 0 fills everything at level 1
    n = 8
    d = np.eye(n, dtype=bool)
    d[0, :] = True
    d[:, 0] = True
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(d.sum(1), out=rp[1:])
    ci = np.nonzero(d)[1].astype(np.int32)
    p1 = oracle.symbolic(rp, ci, 1)
    assert p1.nnz == n * n
    lev = np.full((n, n), -1)
    for i in range(n):
        for p in range(p1.row_ptr[i], p1.row_ptr[i + 1]):
            lev[i, p1.col_idx[p]] = p1.level[p]
    want = np.where(d, 0, 1)
    assert np.array_equal(lev, want)
    assert oracle.symbolic(rp, ci, 0).nnz == d.sum()


def test_validation_errors():
    a = P.laplace3d_7pt(3)
    st, bad = oracle.validate(a.row_ptr, a.col_idx)
    assert st == 0
    # drop the diagonal of row 4
    rp, ci = a.row_ptr.copy(), a.col_idx.copy()
    s, e = rp[4], rp[5]
    d = s + int(np.searchsorted(ci[s:e], 4))
    ci2 = np.delete(ci, d)
    rp2 = rp.copy()
    rp2[5:] -= 1
    st, bad = oracle.validate(rp2, ci2)
    assert (oracle.STATUS[st], bad) == ("MISSING_DIAG", 4)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.symbolic(rp2, ci2, 1)
    assert ei.value.status == "MISSING_DIAG" and ei.value.index == 4
    # unsorted row 2
    ci3 = ci.copy()
    s = rp[2]
    ci3[s], ci3[s + 1] = ci3[s + 1], ci3[s]
    st, bad = oracle.validate(rp, ci3)
    assert (oracle.STATUS[st], bad) == ("BAD_MATRIX", 2)
    # column out of range
    ci4 = ci.copy()
    ci4[-1] = a.n
    st, bad = oracle.validate(rp, ci4)
    assert (oracle.STATUS[st], bad) == ("BAD_MATRIX", a.n - 1)
