"""Multi-rank CUDA path on ONE B200: P ranks as threads of this process (FASTILU_COMM_LOCAL), each
with its own handle, stream and z-slab of rows, halos exchanged by the library (factor rows of
the lower neighbour per sweep; z / w vector halos per trisolve sweep; s once).  Synchronous
sweeps make every result independent of the partition: factors and x must be BITWISE equal to
the single-GPU run (and therefore to the oracle's factors)."""
import threading

import numpy as np
import pytest
import torch

import oracle
import paper_2506_05793_b200 as F
import problems as P

pytestmark = pytest.mark.gpu


def split_planes(gz, world):
    return [(gz * r // world, gz * (r + 1) // world) for r in range(world)]


def run_partitioned(kind, g, gz, k, ns, nt, world, omega=1.0, omega_tri=1.0, tol=None, info=None):
    plane = g * g
    global_n = plane * gz
    b = P.rhs_positive(global_n)
    grp = F.fastilu_group_create(world)
    out = [None] * world
    errs = [None] * world

    def worker(r):
        try:
            torch.cuda.set_device(0)
            z0, z1 = split_planes(gz, world)[r]
            need = F.fastilu_required_lead_rows(P.bandwidth(kind, g), k)
            lp = min(z0, -(-need // plane))
            blk = P.make(kind, g, gz, planes=(z0 - lp, z1))
            f = F.FastILU(blk.row_ptr, blk.col_idx, blk.values, k, omega=omega,
                          omega_tri=omega_tri, rank=r, nranks=world, comm_kind=F.COMM_LOCAL,
                          group=grp, global_n=global_n, row_begin=z0 * plane,
                          n_lead=lp * plane, n=(z1 - z0) * plane)
            if tol is not None:
                assert f.compute_tol(tol, 100) > 0
            else:
                f.compute(ns)
            if info is not None:
                info[r] = f.info()
            vals, s = f.factors()
            tb = torch.tensor(b[z0 * plane:z1 * plane], device="cuda")
            tx = torch.empty_like(tb)
            f.apply(tb, tx, nt)
            torch.cuda.synchronize()
            # the end-to-end entry bench.py times at N > 1 (host values + b in, x out)
            xh = (f.solve_host(blk.values, ns, b[z0 * plane:z1 * plane], nt)
                  if tol is None else None)
            out[r] = (vals, s, tx.cpu().numpy(), f.residual_history(), f.pattern(), xh)
            f.close()
        except Exception as e:  # surfaced below
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "rank threads hung"
    F.fastilu_group_destroy(grp)
    for e in errs:
        if e is not None:
            raise e
    return out, b


@pytest.mark.parametrize("kind,g,gz,k,ns,nt,world", [
    ("27pt", 10, 16, 1, 3, 5, 2),
    ("27pt", 8, 24, 2, 3, 4, 3),
    ("7pt", 16, 20, 0, 3, 5, 4),
    ("27pt", 12, 30, 1, 2, 3, 4),
])
def test_partition_bitwise_equal_single_gpu(kind, g, gz, k, ns, nt, world):
    a = P.make(kind, g, gz)
    b = P.rhs_positive(a.n)
    f1 = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    f1.compute(ns)
    v1, s1 = f1.factors()
    tb = torch.tensor(b, device="cuda")
    tx = torch.empty_like(tb)
    f1.apply(tb, tx, nt)
    torch.cuda.synchronize()
    x1 = tx.cpu().numpy()
    out, _ = run_partitioned(kind, g, gz, k, ns, nt, world)
    vP = np.concatenate([o[0] for o in out])
    sP = np.concatenate([o[1] for o in out])
    xP = np.concatenate([o[2] for o in out])
    assert np.array_equal(np.concatenate([o[4][1] for o in out]), f1.pattern()[1])
    assert np.array_equal(sP, s1)
    assert np.array_equal(vP, v1), "partitioned factors differ from the single-GPU run"
    assert np.array_equal(xP, x1), "partitioned x differs from the single-GPU run"
    assert np.array_equal(np.concatenate([o[5] for o in out]), x1), "solve_host on P ranks"
    for o in out:  # residual: rank-ordered sum of the same per-row terms
        np.testing.assert_allclose(o[3], f1.residual_history(), rtol=1e-12)
    fo = oracle.compute(a, k, ns)
    assert np.array_equal(vP, fo.vals)


def test_partition_damped():
    kind, g, gz, k, ns, nt = "27pt", 8, 18, 1, 3, 3
    a = P.make(kind, g, gz)
    b = P.rhs_positive(a.n)
    out, _ = run_partitioned(kind, g, gz, k, ns, nt, 3, omega=0.8, omega_tri=0.9)
    fo = oracle.compute(a, k, ns, 0.8)
    assert np.array_equal(np.concatenate([o[0] for o in out]), fo.vals)
    xo = oracle.apply(fo, b, nt, 0.9)
    xP = np.concatenate([o[2] for o in out])
    assert np.all(np.abs(xP - xo) <= 1e-12 * np.abs(xo))


def test_partition_fused_first_sweep_and_tolerance():
    """Template path on 2 ranks: sweep 1 runs the init-fused staged kernel on every rank (the
    lower ghost rows' ahat is computed locally), and the stopping sweep of compute_tol (norm of
    ahat over owned rows, residual summed over ranks) equals the single-GPU one."""
    kind, g, gz, k, nt = "27pt", 16, 16, 1, 3
    a = P.make(kind, g, gz)
    f1 = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    s1 = f1.compute_tol(1e-10, 100)
    v1 = f1.factors()[0]
    info = [None, None]
    out, _ = run_partitioned(kind, g, gz, k, 0, nt, 2, tol=1e-10, info=info)
    assert all("staged=1" in i and "st_init=1" in i for i in info), info
    for o in out:
        assert len(o[3]) == s1
        np.testing.assert_allclose(o[3], f1.residual_history(), rtol=1e-12)
    assert np.array_equal(np.concatenate([o[0] for o in out]), v1)


@pytest.mark.parametrize("overlap", ["1", "0"])
def test_partition_128_four_ranks_bitwise(overlap, monkeypatch):
    """27-pt 128^3 ILU(1) (config 3a) on 4 in-process ranks of 32 planes: the ghost
    region (one plane + a line, ~16.6k rows) spans whole TMA boxes of the staged sweep, the
    packed factor halo moves only the diagonal + upper columns, and the interior rows are swept
    while it flies (overlap "1"; "0": FASTILU_NO_HALO_OVERLAP, halo first).  Factors and x are
    bitwise the single-GPU run's."""
    if overlap == "0":
        monkeypatch.setenv("FASTILU_NO_HALO_OVERLAP", "1")
    kind, g, gz, k, ns, nt, world = "27pt", 128, 128, 1, 3, 5, 4
    a = P.make(kind, g, gz)
    b = P.rhs_positive(a.n)
    f1 = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    f1.compute(ns)
    v1 = f1.factors()[0]
    tb = torch.tensor(b, device="cuda")
    tx = torch.empty_like(tb)
    f1.apply(tb, tx, nt)
    torch.cuda.synchronize()
    x1 = tx.cpu().numpy()
    r1 = f1.residual_history()
    f1.close()
    del a
    info = [None] * world
    out, _ = run_partitioned(kind, g, gz, k, ns, nt, world, info=info)
    assert all("staged=1" in i and "halo_bytes=" in i for i in info), info
    assert np.array_equal(np.concatenate([o[0] for o in out]), v1)
    assert np.array_equal(np.concatenate([o[2] for o in out]), x1)
    assert np.array_equal(np.concatenate([o[5] for o in out]), x1)  # solve_host
    for o in out:
        np.testing.assert_allclose(o[3], r1, rtol=1e-12)
    # the packed halo: diagonal + upper columns (32 of W = 63) of the ghost rows
    hb = [int(i.split("halo_bytes=")[1].split()[0]) for i in info]
    assert hb[-1] == 0 and all(h == hb[0] for h in hb[:-1])
    assert hb[0] == 128 * 128 * 32 * 8, hb  # G = one plane (the lowest neighbour is -g^2)


def test_partition_256_two_ranks_x_bitwise():
    """The bench workload (c4: 27-pt 256^3 ILU(1), 3 sweeps + 5/5 Jacobi sweeps) split into two
    in-process ranks of 128 planes: x (which depends on every factor entry) and the residual
    history equal the single-GPU run's bitwise / to rounding of the rank-ordered sum.  Only x
    and the histories come back to the host (the factors are 8 GB)."""
    kind, g, gz, k, ns, nt, world = "27pt", 256, 256, 1, 3, 5, 2
    a = P.make(kind, g, gz)
    b = P.rhs_positive(a.n)
    f1 = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    f1.compute(ns)
    tb = torch.tensor(b, device="cuda")
    tx = torch.empty_like(tb)
    f1.apply(tb, tx, nt)
    torch.cuda.synchronize()
    x1 = tx.cpu().numpy()
    r1 = f1.residual_history()
    f1.close()
    del a, tb, tx
    torch.cuda.empty_cache()
    plane = g * g
    grp = F.fastilu_group_create(world)
    out, errs = [None] * world, [None] * world

    def worker(r):
        try:
            torch.cuda.set_device(0)
            z0, z1 = split_planes(gz, world)[r]
            need = F.fastilu_required_lead_rows(P.bandwidth(kind, g), k)
            lp = min(z0, -(-need // plane))
            blk = P.make(kind, g, gz, planes=(z0 - lp, z1))
            f = F.FastILU(blk.row_ptr, blk.col_idx, blk.values, k, rank=r, nranks=world,
                          comm_kind=F.COMM_LOCAL, group=grp, global_n=plane * gz,
                          row_begin=z0 * plane, n_lead=lp * plane, n=(z1 - z0) * plane)
            del blk
            f.compute(ns)
            xb = torch.tensor(b[z0 * plane:z1 * plane], device="cuda")
            xr = torch.empty_like(xb)
            f.apply(xb, xr, nt)
            torch.cuda.synchronize()
            out[r] = (xr.cpu().numpy(), f.residual_history(), f.info())
            f.close()
        except Exception as e:  # surfaced below
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not any(t.is_alive() for t in th), "rank threads hung"
    F.fastilu_group_destroy(grp)
    for e in errs:
        if e is not None:
            raise e
    assert all("staged=1" in o[2] for o in out)
    assert np.array_equal(np.concatenate([o[0] for o in out]), x1)
    for o in out:
        np.testing.assert_allclose(o[1], r1, rtol=1e-12)


def test_nccl_two_processes():
    """The NCCL transport across two GPUs (one process per GPU, torchrun): factors and x of a
    2-rank run are bitwise the single-GPU run's.  Skips on a box with fewer than 2 GPUs."""
    import os
    import subprocess
    import sys
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29611",
                        os.path.join(root, "tests", "nccl_worker.py")],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert '"ok": true' in r.stdout, r.stdout[-2000:]


def test_partition_gmres():
    """Config 5's GMRES(60) on 3 in-process ranks (SpMV vector halos, dot products summed over
    ranks, FastILU apply with trisolve halos): the iteration count equals the single-GPU run's
    (+-1: the dot products are summed rank by rank) and both reach the 1e-6 relative residual."""
    kind, g, gz, k, ns, nt, world = "aniso7pt", 16, 24, 0, 2, 5, 3
    a = P.make(kind, g, gz)
    xt = P.x_true(a.n)
    b = oracle.spmv(a, xt)
    f1 = F.FastILU(a.row_ptr, a.col_idx, a.values, k)
    f1.compute(ns)
    tb = torch.tensor(b, device="cuda")
    tx = torch.zeros_like(tb)
    it1, rr1 = f1.gmres(tb, tx, 60, 1e-6, 2000, nt)
    plane = g * g
    grp = F.fastilu_group_create(world)
    res = [None] * world
    errs = [None] * world

    def worker(r):
        try:
            torch.cuda.set_device(0)
            z0, z1 = split_planes(gz, world)[r]
            need = F.fastilu_required_lead_rows(P.bandwidth(kind, g), k)
            lp = min(z0, -(-need // plane))
            blk = P.make(kind, g, gz, planes=(z0 - lp, z1))
            f = F.FastILU(blk.row_ptr, blk.col_idx, blk.values, k, rank=r, nranks=world,
                          comm_kind=F.COMM_LOCAL, group=grp, global_n=a.n,
                          row_begin=z0 * plane, n_lead=lp * plane, n=(z1 - z0) * plane)
            f.compute(ns)
            tbr = torch.tensor(b[z0 * plane:z1 * plane], device="cuda")
            txr = torch.zeros_like(tbr)
            res[r] = f.gmres(tbr, txr, 60, 1e-6, 2000, nt) + (txr.cpu().numpy(),)
            f.close()
        except Exception as e:
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    F.fastilu_group_destroy(grp)
    for e in errs:
        if e is not None:
            raise e
    its = {r[0] for r in res}
    assert len(its) == 1, its  # every rank ran the same iterations
    itP, rrP = res[0][0], res[0][1]
    assert rr1 <= 1e-6 and rrP <= 1e-6 and abs(itP - it1) <= 1, (itP, it1)
    x = np.concatenate([r[2] for r in res])
    assert np.linalg.norm(b - oracle.spmv(a, x)) <= 1e-6 * np.linalg.norm(b) * (1 + 1e-9)
