"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/fastilu.h declares,
and its host-side setup (validation + the product's own symbolic ILU(k), an independent
implementation: sorted linked lists, chunk-parallel windows) matches the oracle bit-exactly.
No compute call needs a GPU here."""
import ctypes as C

import numpy as np
import pytest

import oracle
import paper_2506_05793_b200 as F
import problems as P


def test_library_exports_every_header_symbol():
    L = F.lib()
    names = F.header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    assert set(F._SIGS) == set(names)


def test_status_strings_and_defaults():
    assert F.fastilu_status_string(0) == "FASTILU_OK"
    assert F.fastilu_status_string(5) == "FASTILU_ERR_ZERO_PIVOT"
    o = F.fastilu_default_options()
    assert (o.omega, o.omega_tri, o.device, o.nranks) == (1.0, 1.0, -1, 1)
    assert F.fastilu_required_lead_rows(10, 1) == 40


def _same_pattern(a, k, threads=0):
    rp, ci, lev = F.fastilu_symbolic(a.row_ptr, a.col_idx, k, threads)
    pat = oracle.symbolic(a.row_ptr, a.col_idx, k)
    assert np.array_equal(rp, pat.row_ptr)
    assert np.array_equal(ci, pat.col_idx)
    assert np.array_equal(lev.astype(np.int32), pat.level)


@pytest.mark.parametrize("kind,g,k", [("7pt", 10, 0), ("7pt", 9, 2), ("27pt", 7, 1),
                                       ("27pt", 6, 2), ("27pt", 5, 3), ("aniso7pt", 8, 1),
                                       ("3dof", 5, 2)])
def test_symbolic_matches_oracle(kind, g, k):
    _same_pattern(P.make(kind, g), k)


@pytest.mark.parametrize("seed,k", [(1, 0), (2, 1), (3, 2), (4, 4)])
def test_symbolic_matches_oracle_random(seed, k):
    _same_pattern(P.random_sparse(300, 0.01, seed=seed), k)


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_symbolic_chunk_parallel_exact(threads):
    # n = 110,592 > 65,536: the chunked windows are used; their rows must be exact
    _same_pattern(P.laplace3d_27pt(48), 1, threads)


def test_symbolic_chunk_parallel_exact_ilu2_ragged():
    # 40 x 40 x 45 grid (ragged in z), ILU(2): several chunks with 6 (K+1) bandwidth margins
    _same_pattern(P.laplace3d_27pt(40, gz=45), 2, 5)


def test_symbolic_errors():
    a = P.laplace3d_7pt(4)
    rp, ci = a.row_ptr.copy(), a.col_idx.copy()
    s, e = rp[7], rp[8]
    d = s + int(np.searchsorted(ci[s:e], 7))
    ci2 = np.delete(ci, d)
    rp2 = rp.copy()
    rp2[8:] -= 1
    with pytest.raises(F.FastILUError) as ei:
        F.fastilu_symbolic(rp2, ci2, 1)
    assert ei.value.status == "MISSING_DIAG" and ei.value.index == 7
    ci3 = ci.copy()
    ci3[rp[3]], ci3[rp[3] + 1] = ci3[rp[3] + 1], ci3[rp[3]]
    with pytest.raises(F.FastILUError) as ei:
        F.fastilu_symbolic(rp, ci3, 0)
    assert ei.value.status == "BAD_MATRIX" and ei.value.index == 3
    with pytest.raises(F.FastILUError) as ei:
        F.fastilu_symbolic(rp, ci, -1)
    assert ei.value.status == "INVALID_ARG"


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    a = P.laplace3d_7pt(3)
    with pytest.raises(F.FastILUError) as ei:
        F.FastILU(a.row_ptr, a.col_idx, a.values, 0)
    assert ei.value.status == "CUDA"


def test_bench_block_flop_count_matches_survey():
    """bench.py's flop count for the block path reproduces SURVEY Sec. 8(d)'s independent count
    for the Table-6 problem (3,537,519,556 terms per sweep) from the block-term total that the
    library reports for it (129,330,412 pivot-block terms over 5,081,056 blocks)."""
    import bench
    info = "path=bsr3 blocks=5081056 terms=129330412 threads=256"
    r = bench.bsr_roofline(info, 98304, 1.0)
    assert r["terms_per_sweep"] == 3537519556
    assert r["bound"] == "alu" and r["unit"] == "TFLOP/s"


def test_bench_smem_port_bytes():
    """bench.py's shared-memory-port figure of the staged sweep: one 8-byte
    LDS per term and row plus the TMA box writes, counted from the kernel configuration the
    library reports (c4: 587 terms, 65,536 tiles of 256 rows, 7 boxes of 32 x 32 x 10 doubles)."""
    import bench
    info = ("path=tsell W=63 c0=31 WA=27 terms=587 staged=1 st_threads=512 st_parts=2 "
            "st_rows=256 st_shift=0 st_groups=7 st_box=32x32x10 st_stages=2")
    n = 256 ** 3
    r = bench.smem_port(info, n, 1.0, 1000.0, 100)
    assert r["lds_bytes"] == n * 587 * 8
    assert r["tma_bytes"] == (n // 256) * 7 * 32 * 32 * 10 * 8
    assert abs(r["peak"] - 128 * 100 * 1000e6 / 1e9) < 1e-9
    assert abs(r["achieved"] - (r["lds_bytes"] + r["tma_bytes"]) / 1e-3 / 1e9) < 1e-6
    assert bench.smem_port("path=tsell W=7 terms=3", n, 1.0, 1000.0) is None
    # with the generator's exact counts (distinct LDS per row over both part-warps, TMA bytes
    # per tile incl. the own-row boxes) those replace the lower bound, which is kept alongside
    r2 = bench.smem_port(info + " st_lds=712 st_tma=645120", n, 1.0, 1000.0, 100)
    assert r2["lds_bytes"] == n * 712 * 8 and r2["tma_bytes"] == (n // 256) * 645120
    assert r2["lower_bound"]["bytes_per_launch"] == r["bytes_per_launch"]
    assert r2["frac"] > r["frac"]


def test_binding_argument_checks():
    """The binding checks length, dtype, device and contiguity before any pointer reaches the C
    side (which reads / writes a fixed count): ADVICE r1."""
    import torch
    v = F._host_in([1, 2, 3], 3, "v")
    assert v.dtype == np.float64 and v.flags.c_contiguous
    with pytest.raises(ValueError):
        F._host_in(np.zeros(4), 3, "v")
    with pytest.raises(ValueError):
        F._host_in(np.zeros((3, 1)), 3, "v")
    assert F._host_out(None, 5, "o").shape == (5,)
    for bad in (np.zeros(5, dtype=np.float32), np.zeros(4), np.zeros(10)[::2],
                np.zeros(5).reshape(5, 1)):
        with pytest.raises(ValueError):
            F._host_out(bad, 5, "o")
    ro = np.zeros(5)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        F._host_out(ro, 5, "o")
    assert F._dev_arg(12345, 5, 0, "b") == 12345  # raw pointers pass through
    with pytest.raises(ValueError):  # float32
        F._dev_arg(torch.zeros(5, dtype=torch.float32), 5, 0, "b")
    with pytest.raises(ValueError):  # not on a GPU
        F._dev_arg(torch.zeros(5, dtype=torch.float64), 5, 0, "b")
