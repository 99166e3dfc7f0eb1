"""GPU parity of the block sweep (csrc/bsr.cu): block-dense ILU(k) patterns -- the paper's 3-dof
27-point problems and 2-/4-dof variants -- against
the oracle, bitwise (the block terms are the scalar terms in the oracle's ascending-k order)."""
import numpy as np
import pytest

import oracle
import paper_2506_05793_b200 as F
import problems as P
from test_gpu_parity import full_check

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def no_template(monkeypatch):
    """Small block patterns also fit the template-SELL layout (W <= 128); take the block path."""
    monkeypatch.setenv("FASTILU_NO_TSELL", "1")


@pytest.mark.parametrize("g,k,ns,nt", [(4, 0, 3, 3), (4, 1, 3, 5), (5, 2, 2, 4), (6, 3, 3, 3),
                                       (8, 3, 3, 5)])
def test_3dof_block_path(g, k, ns, nt):
    f = full_check(P.elasticity_pattern_3dof(g), k, ns, nt)
    assert f.info().startswith("path=bsr3"), f.info()


@pytest.mark.parametrize("dofs,g,k", [(2, 5, 2), (4, 4, 1), (4, 3, 2)])
def test_other_block_sizes(dofs, g, k):
    f = full_check(P.multi_dof_pattern(g, dofs, seed=7), k, 3, 4)
    assert f.info().startswith(f"path=bsr{dofs}"), f.info()


def test_block_damping_and_shift():
    a = P.multi_dof_pattern(4, 3, seed=3)
    f = full_check(a, 2, 4, 3, omega=0.6, omega_tri=0.9)
    assert f.info().startswith("path=bsr3")
    full_check(a, 1, 3, 3, shift=0.3)


def test_block_sweeps_to_convergence():
    a = P.elasticity_pattern_3dof(5)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 2)
    s_gpu = f.compute_tol(1e-10, 100)
    fo, s_or = oracle.compute_tol(a, 2, 1e-10, 100)
    assert f.info().startswith("path=bsr3")
    assert s_gpu == s_or
    assert np.array_equal(f.factors()[0], fo.vals)


def test_block_zero_pivot():
    """A dense 2x2 all-ones matrix is block-dense (bs 2): u_11 = 1 - 1 * 1 = 0 after sweep 1."""
    z = P.Csr([0, 2, 4], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0])
    g = F.FastILU(z.row_ptr, z.col_idx, z.values, 0)
    assert g.info().startswith("path=bsr2")
    g.compute(0)
    with pytest.raises(F.FastILUError) as ei:
        g.compute(1)
    assert ei.value.status == "ZERO_PIVOT" and ei.value.index == 1


def test_table6_problem_block_vs_scalar_kernel(monkeypatch):
    """The paper's Table-6 problem at full size (3-dof 32^3, ILU(3), 45.7 M entries): the block
    sweep equals the scalar CSR sweep bitwise (both are pinned to the oracle at small sizes
    above; the oracle itself needs minutes here)."""
    a = P.elasticity_pattern_3dof(32)
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 3)
    assert f.info().startswith("path=bsr3")
    f.compute(3)
    v1, _ = f.factors()
    h1 = f.residual_history()
    f.close()
    monkeypatch.setenv("FASTILU_NO_BSR", "1")
    g = F.FastILU(a.row_ptr, a.col_idx, a.values, 3)
    assert g.info().startswith("path=csr")
    g.compute(3)
    v2, _ = g.factors()
    assert v1.size == 45729504
    assert np.array_equal(v1, v2)
    np.testing.assert_allclose(h1, g.residual_history(), rtol=1e-9)


def test_handles_with_different_smem_configs(monkeypatch):
    """The dynamic shared-memory limit is per kernel function: a handle configured later with
    less shared memory must not break an earlier handle's launches (regression)."""
    a = P.elasticity_pattern_3dof(6)
    monkeypatch.setenv("FASTILU_BSR_SMEM_KB", "32")
    f = F.FastILU(a.row_ptr, a.col_idx, a.values, 2)
    monkeypatch.setenv("FASTILU_BSR_SMEM_KB", "8")
    g = F.FastILU(a.row_ptr, a.col_idx, a.values, 2)
    for h in (f, g, f):
        h.compute(3)
    assert np.array_equal(f.factors()[0], g.factors()[0])
