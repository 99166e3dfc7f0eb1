#!/usr/bin/env python
"""FastILU benchmark (BASELINE.json metric: FastILU sweep nnz-updates/s and trisolve GB/s vs HBM
peak).  One step = one pass of the whole hot path on one synthetic matrix: fastilu_compute
(scale + init + nsweeps synchronous sweeps) then fastilu_apply (ntri Jacobi sweeps for L and
for U).  Inputs (A, b) are resident in HBM before the timed region; the working set (tens of GB)
exceeds the 126 MB L2, so no explicit flush is needed between steps for the default workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `value` = nnz(S) * nsweeps * N / (device time of one step, max
over ranks).  Extra keys: sweep-only rate, trisolve and composite GB/s, the dominant kernel's
roofline, e2e through host buffers, and the oracle timed on a bounded sample (cpu_baseline).
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import problems as P  # noqa: E402

METRIC = "FastILU sweep nnz-updates/s and trisolve GB/s vs HBM peak, 1/2/4/8 B200"
UNIT = "nnz-updates/s"
SV, SI = 8, 4


# FP64 lane throughput of one B200: 148 SMs x 64 FP64 lanes x 1.965 GHz.  The
# sweep's rounded product and rounded difference are separate instructions (no FMA, for the
# oracle's bitwise order), so one flop per lane-cycle.
FP64_LANE_TFLOPS = 148 * 64 * 1.965e9 / 1e12


def bsr_roofline(info, n, sweep_ms):
    """Block path: flops per sweep from the term count.  Each pivot-block term is BS^3 rounded
    multiply-subtracts; each off-diagonal target block adds BS^2 (BS-1)/2 tail terms inside block
    min(I,J), each diagonal block sum_{d,e} min(d,e) (3,537,519,556 terms per
    sweep for the Table-6 problem)."""
    import re
    bs = int(re.search(r"path=bsr(\d)", info).group(1))
    nterms = int(re.search(r"terms=(\d+)", info).group(1))
    nblk = int(re.search(r"blocks=(\d+)", info).group(1))
    nb = n // bs
    tail = bs * bs * (bs - 1) // 2 * (nblk - nb) + sum(min(d, e) for d in range(bs)
                                                        for e in range(bs)) * nb
    terms = bs ** 3 * nterms + tail
    achieved = 2 * terms / (sweep_ms * 1e-3) / 1e12
    return {"bound": "alu", "kernel": "bsr_sweep_kernel", "achieved": achieved,
            "peak": FP64_LANE_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_LANE_TFLOPS,
            "peak_source": "derived: 148 SMs x 64 FP64 lanes x 1.965 GHz, one rounded mul or sub "
                           "per lane-cycle (no FMA)", "traffic": None, "terms_per_sweep": terms}


def smem_port(info, n, launch_ms, sm_mhz, sms=148):
    """Staged template sweep: shared-memory port bytes per launch against
    128 B/clk/SM (B300_MICROARCH.md LDS/STS table) x SMs x the SM clock measured in the timed
    region.  Bytes = the distinct 8-byte shared-memory loads the generated kernel issues per row
    (st_lds: pivot values u_kj, divisors u_jj, own l_it and own old u_ij, counted by the generator
    over all part-warps) x n + the TMA bytes written into shared memory per tile (st_tma: pivot
    boxes + own-row boxes) x tiles.  `lower_bound` keeps round 1's figure (one LDS per term + the
    pivot boxes only)."""
    import re
    kv = dict(re.findall(r"(\w+)=(\S+)", info))
    if kv.get("staged") != "1" or launch_ms <= 0:
        return None
    terms, rows = int(kv["terms"]), int(kv["st_rows"])
    bx, by, bz = (int(v) for v in kv["st_box"].split("x"))
    tiles = -(-n // rows)
    lds_lb = n * terms * 8
    tma_lb = tiles * int(kv["st_groups"]) * bx * by * bz * 8
    lds = n * int(kv["st_lds"]) * 8 if "st_lds" in kv else lds_lb
    tma = tiles * int(kv["st_tma"]) if "st_tma" in kv else tma_lb
    mhz = sm_mhz or 1965.0
    peak = 128 * sms * mhz * 1e6 / 1e9
    ach = (lds + tma) / (launch_ms * 1e-3) / 1e9
    return {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "bytes_per_launch": lds + tma, "lds_bytes": lds, "tma_bytes": tma,
            "lds_per_row": int(kv.get("st_lds", terms)),
            "lower_bound": {"bytes_per_launch": lds_lb + tma_lb,
                            "frac": (lds_lb + tma_lb) / (launch_ms * 1e-3) / 1e9 / peak},
            "peak_source": f"128 B/clk/SM x {sms} SMs x {mhz:.0f} MHz (median SM clock, timed region)"}


def byte_model(n, nnz_A, nnz_S, nnz_Ls, ns, nt):
    """Algorithmic bytes."""
    sp = 4 if nnz_S < 2**31 else 8
    B_f = nnz_S * (2 * SV + SI) + nnz_A * SV + 2 * (n + 1) * sp
    B_L = nnz_Ls * (SV + SI) + (n + 1) * sp + 3 * n * SV
    B_U = B_L + n * SV
    B_init = nnz_A * (SV + SI) + nnz_S * SV + n * SV
    # first L sweep (z0 = 0): y = s o b, z1 = w y -> 4 n words; first U sweep: w1 = z / u_ii
    B_apply = (nt - 1) * (B_L + B_U) + 4 * n * SV + 3 * n * SV
    return dict(B_f=B_f, B_L=B_L, B_U=B_U, B_init=B_init, B_apply=B_apply)


def layout_model(info, n, nnz_A, nnz_S, nnz_Ls, ns, nt):
    """Bytes the kernels of this handle's layout must move at least once:
    the template-SELL layout stores W value slots per row (padded to 32-row slices), Ahat on A's
    WA template columns and a presence mask, and NO column indices -- so it moves less than the
    SURVEY Sec. 8(d) CSR model, which charges 4 index bytes per entry.  Per launch:
      full sweep   read + write the W slots, read Ahat (WA) + mask, write u_ii
      sweep 1      (init fused) read Ahat + mask, write the W slots + u_ii
      init         scale: a_ii in, s + ahat_ii out; Ahat: A's WA slots + mask in, WA slots out
      Jacobi L     the c0 strict-lower slots + mask, rhs, x_old (compulsory), x_new out
      Jacobi U     the W-c0-1 strict-upper slots + mask, rhs, x_old, u_ii, x_new out
      first L / U  b, s in, y, z out / z, u_ii in, w out
    Non-template paths (CSR, block): the SURVEY model (they do move index bytes)."""
    import re
    kv = dict(re.findall(r"(\w+)=(\S+)", info))
    if not info.startswith("path=tsell"):
        bm = byte_model(n, nnz_A, nnz_S, nnz_Ls, ns, nt)
        return dict(kind="survey (CSR / block path)", B_f=bm["B_f"], B_f1=bm["B_f"],
                    B_init=bm["B_init"], B_L=bm["B_L"], B_U=bm["B_U"], B_apply=bm["B_apply"])
    W, c0, WA = int(kv["W"]), int(kv["c0"]), int(kv["WA"])
    words = (W + 63) // 64
    npad = -(-n // 32) * 32
    B_f = npad * 8 * (2 * W + WA + words) + 8 * n
    B_init = 24 * n + npad * 8 * (2 * WA + words) + 8 * n
    if kv.get("st_init") == "1":  # sweep 1 derives iterate 0 from Ahat: it reads no W slots
        B_f1 = npad * 8 * (W + WA + words) + 8 * n
    else:  # the init stores iterate 0 (W slots + u_ii) and sweep 1 is a full sweep
        B_f1 = B_f
        B_init += npad * 8 * W + 8 * n
    B_L = npad * 8 * (c0 + words) + 24 * n
    B_U = npad * 8 * (W - c0 - 1 + words) + 32 * n
    B_apply = 32 * n + (nt - 1) * B_L + 32 * n + (nt - 1) * B_U
    return dict(kind="template-SELL layout (no index bytes)", B_f=B_f, B_f1=B_f1, B_init=B_init,
                B_L=B_L, B_U=B_U, B_apply=B_apply)


def cpu_info():
    """Host cores the oracle may use and the CPU model (lscpu / /proc/cpuinfo)."""
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cores, model


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling (B200_PROFILING.md clocks line).  Started before the warm-up (the tool
    needs ~0.3 s to start); samples carry wall-clock stamps and only those inside the timed
    window [mark_start, mark_stop] are summarised (all samples if the window caught < 3)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.t0 = self.t1 = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                      text=True, bufsize=1)
            import threading
            self.rows = []
            self.th = threading.Thread(target=self._reader, daemon=True)
            self.th.start()
        except Exception:
            self.p = None

    def _reader(self):
        for line in self.p.stdout:
            self.rows.append((time.time(), line.strip()))

    def wait_ready(self, timeout=5.0):
        """Block until nvidia-smi delivered its first sample (its start-up takes ~0.3-1 s, longer
        than a short timed region)."""
        t = time.time()
        while self.p is not None and not self.rows and time.time() - t < timeout:
            time.sleep(0.02)

    def mark_start(self):
        self.t0 = time.time()

    def mark_stop(self):
        self.t1 = time.time()

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.p.terminate()
        self.p.wait()
        self.th.join(timeout=1)
        os.unlink(self.f.name)
        rows = self.rows
        win = [r for r in rows if self.t0 and self.t1 and self.t0 <= r[0] <= self.t1 + 0.05]
        scope = "timed region"
        if len(win) < 3:
            win, scope = rows, "whole run (timed region too short for the sampler)"
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, line in win:
            r = line.split(",")
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
                for nm, v in zip(names, r[4:8]):
                    if v.strip().lower() in ("active", "1"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm), "scope": scope}


def build_matrix(kind, g):
    t = time.perf_counter()
    a = P.make(kind, g)
    return a, time.perf_counter() - t


def cpu_sample(kind, g, k, ns, nt, planes, threads=1):
    """Oracle on a bounded sample of the workload: a g x g x planes slab of the same stencil,
    its per-row loops on `threads` OpenMP threads (bitwise the 1-thread oracle)."""
    import oracle
    sub = P.make(kind, g, gz=planes)
    pat = oracle.symbolic(sub.row_ptr, sub.col_idx, k)
    b = P.rhs_positive(sub.n)
    used = oracle.set_threads(threads)
    try:
        t0 = time.perf_counter()
        f = oracle.compute(sub, k, ns, pat=pat)
        oracle.apply(f, b, nt)
        dt = time.perf_counter() - t0
    finally:
        oracle.set_threads(1)
    return dict(value=pat.nnz * ns / dt, seconds=dt, nnz_S=pat.nnz, n=sub.n, threads=used,
                sample=f"{kind} {g}x{g}x{planes} slab of the workload, ILU({k}), {ns} sweeps + "
                       f"{nt}/{nt} trisweeps, scale/init+sweeps+apply timed (symbolic excluded), "
                       f"{used} OpenMP threads")


def cpu_planes_for(kind, g, k, ns, nt, threads, target_s=8.0, cap=64):
    """Slab thickness giving ~target_s seconds of oracle time on `threads` cores (probe with a
    2-plane slab); capped so the sample's host memory stays bounded."""
    probe = cpu_sample(kind, g, k, ns, nt, 2, threads)
    per_plane = probe["seconds"] / 2
    return int(max(2, min(cap, g, target_s / max(per_plane, 1e-6))))


def run_reference(args, wl):
    """The reference arm of this tier: the oracle as it stands, on all host cores, on a bounded
    slab of the workload (rank 0 only; other ranks exit without work)."""
    kind, g, k, ns, nt = wl
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores, model = cpu_info()
    planes = args.cpu_planes or cpu_planes_for(kind, g, k, ns, nt, cores, target_s=4.0)
    for _ in range(args.warmup):
        cpu_sample(kind, g, k, ns, nt, planes, cores)
    vals, secs = [], []
    for _ in range(args.steps):
        r = cpu_sample(kind, g, k, ns, nt, planes, cores)
        vals.append(r["value"])
        secs.append(r["seconds"])
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.median(secs)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "sample_planes": planes},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["threads"], "cpu": model,
                             "kind": "oracle", "sample": r["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _reorth(f):
    """Second Gram-Schmidt passes the last GMRES took (DGKS criterion)."""
    import re
    m = re.search(r"gmres_reorth=(\d+)", f.info())
    return int(m.group(1)) if m else None


def gmres_arms(args, f, a, ns, stream):
    """BASELINE configs[4] (config 5): FastILU-preconditioned GMRES(60) to a 1e-6 relative
    residual, x0 = 0, b = A x_true with x_true ~ U[0,1) (SURVEY 8(d) "Config 5
    comparison arms").  Device-timed (CUDA events on the handle's stream), per ntri = 1..5:
      A: FastILU factors (ns sweeps) + ntri Jacobi sweeps per apply   (compute + GMRES timed)
      B: the factors at the sweep map's fixed point (compute_tol(1e-14): the exact ILU(0) up to
         rounding, SURVEY 8(c) "Sweep map") + ntri Jacobi sweeps        (GMRES timed)
    Arm C (the CPU oracle's exact ILU(0) + exact substitution) is part of the cpu_baseline leg."""
    import torch
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    b = np.bincount(rows, weights=a.values * P.x_true(a.n)[a.col_idx], minlength=a.n)
    dev = torch.device("cuda", torch.cuda.current_device())
    tb = torch.tensor(b, device=dev)
    tx = torch.zeros_like(tb)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"restart": 60, "rtol": 1e-6, "nsweeps": ns, "arms": []}
    nts = args.gmres_ntri
    f.compute(ns)
    f.gmres(tb, tx, 60, 1e-6, 20, 1)  # warm-up (JIT, workspace)
    for nt in nts:
        torch.cuda.synchronize()
        e0.record(stream)
        f.compute(ns)
        it, rr = f.gmres(tb, tx, 60, 1e-6, 5000, nt)
        e1.record(stream)
        torch.cuda.synchronize()
        out["arms"].append({"arm": "A", "ntri": nt, "iterations": it, "relres": rr,
                            "time_to_solution_ms": e0.elapsed_time(e1),
                            "reorth_passes": _reorth(f)})
    torch.cuda.synchronize()
    e0.record(stream)
    s_fix = f.compute_tol(1e-14, 5000)
    e1.record(stream)
    torch.cuda.synchronize()
    out["arm_B_factors"] = {"sweeps": s_fix, "ms": e0.elapsed_time(e1),
                            "resid": float(f.residual_history()[-1])}
    for nt in nts:
        torch.cuda.synchronize()
        e0.record(stream)
        it, rr = f.gmres(tb, tx, 60, 1e-6, 5000, nt)
        e1.record(stream)
        torch.cuda.synchronize()
        out["arms"].append({"arm": "B", "ntri": nt, "iterations": it, "relres": rr,
                            "time_to_solution_ms": e0.elapsed_time(e1),
                            "reorth_passes": _reorth(f)})
    return out, b


def gmres_arm_c(a, b, cores):
    """Arm C (cpu_baseline leg): the oracle's exact ILU(0) + exact substitution as the
    preconditioner of the oracle's GMRES(60) (numpy), timed on the host."""
    import oracle
    used = oracle.set_threads(cores)
    try:
        t0 = time.perf_counter()
        fe = oracle.compute(a, 0, 0)
        fe.vals = oracle.exact_ilu(fe.pattern, fe.ahat)
        t1 = time.perf_counter()
        _, it, rr = oracle.gmres(a, b, oracle.exact_preconditioner(fe), 60, 1e-6, 5000)
        t2 = time.perf_counter()
    finally:
        oracle.set_threads(1)
    return {"arm": "C", "iterations": it, "relres": rr, "factor_s": t1 - t0, "gmres_s": t2 - t1,
            "threads": used}


def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2506_05793_b200 as F

    kind, g, k, ns, nt = wl
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    # a dedicated (non-default) stream: the library enqueues on it and every timing event is
    # recorded on it (the legacy default stream's handle 0 would make the library use its own)
    stream = torch.cuda.Stream(dev)

    t0 = time.perf_counter()
    if world == 1:
        a = P.make(kind, g)
        row_begin = 0
    else:
        # weak scaling: global g x g x (g * world) grid, rank r owns planes [g r, g (r + 1)),
        # plus the lead planes below it that reproduce its ghost rows' exact pattern
        z0, z1 = g * rank, g * (rank + 1)
        need = F.fastilu_required_lead_rows(P.bandwidth(kind, g), k)
        lp = min(z0, -(-need // (g * g)))
        a = P.make(kind, g, gz=g * world, planes=(z0 - lp, z1))
        row_begin = z0 * g * g
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    if world == 1:
        f = F.FastILU(a.row_ptr, a.col_idx, a.values, k, device=local, stream=stream.cuda_stream)
    else:
        uid = [F.fastilu_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        f = F.FastILU(a.row_ptr, a.col_idx, a.values, k, device=local,
                      stream=stream.cuda_stream, rank=rank, nranks=world,
                      comm_kind=F.COMM_NCCL, nccl_unique_id=uid[0],
                      global_n=g * g * g * world, row_begin=row_begin,
                      n_lead=lp * g * g, n=g * g * g)
    t_setup = time.perf_counter() - t0
    n, nnz_S, nnz_A = f.n, f.nnz_S, f.nnz_A
    nnz_S_total = nnz_S
    if world > 1:
        tt = torch.tensor([nnz_S], dtype=torch.float64, device=dev)
        dist.all_reduce(tt)
        nnz_S_total = int(tt.item())
    rp, ci, _ = f.pattern()
    rows = np.repeat(np.arange(n, dtype=np.int64) + row_begin, np.diff(rp))
    nnz_Ls = int(np.count_nonzero(ci < rows))
    del rows, rp, ci
    bm = byte_model(n, nnz_A, nnz_S, nnz_Ls, ns, nt)
    b = torch.tensor(P.rhs_positive(n), device=dev)
    x = torch.empty_like(b)
    torch.cuda.synchronize(dev)

    s_star = []

    def step():
        if args.tol is not None:  # config 3 "sweeps to convergence" (reading G15)
            s_star.append(f.compute_tol(args.tol, 100))
        else:
            f.compute(ns)
        f.apply(b, x, nt)

    clocks = Clocks(local)
    clocks.wait_ready()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if s_star:  # the stopping sweep is deterministic: every step runs the same s*
        ns = s_star[-1]
        bm = byte_model(n, nnz_A, nnz_S, nnz_Ls, ns, nt)
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_sweeps, t_apply, t_init, t_first, t_rest = [], [], [], [], []
    torch.cuda.synchronize()
    clocks.mark_start()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        tm = f.timings()  # library CUDA events on this stream (compute synchronised)
        t_sweeps.append(tm["sweeps_ms"])
        t_first.append(tm["sweep1_ms"])
        t_rest.append(tm["sweeps_rest_ms"])
        t_init.append(tm["init_ms"])
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.mark_stop()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    # apply alone (events inside the library), measured on the last step
    t_apply = f.timings()["apply_ms"]
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.barrier()
    sweep_ms = float(np.mean(t_sweeps))
    value = nnz_S_total * ns / (ms * 1e-3)
    peak, peak_src = peaks()
    # the dominant kernel is the full sweep (sweeps 2..ns); sweep 1 is a different kernel (the
    # initial guess fused in, A x A terms only), reported separately
    rest_ms = float(np.mean(t_rest)) if ns >= 2 else 0.0
    per_launch_ms = rest_ms / (ns - 1) if ns >= 2 and rest_ms > 0 else sweep_ms / max(ns, 1)
    info = f.info()
    lm = layout_model(info, n, nnz_A, nnz_S, nnz_Ls, ns, nt)
    achieved = lm["B_f"] / (per_launch_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.workload, {}).get("sweep_dram_bytes")

    # e2e through host buffers: H2D of A's values and b, compute, apply, D2H of x, every step
    e2e = None
    if not args.no_e2e:
        av = torch.from_numpy(a.values).pin_memory().numpy()
        bh = torch.from_numpy(P.rhs_positive(n)).pin_memory().numpy()
        xh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
        # the public entry for new values from the host: upload pipelined with the compute
        for _ in range(2):  # warm-up: first-call allocations (pipeline buffers), JIT, page-in
            f.solve_host(av, ns, bh, nt, out=xh)
        torch.cuda.synchronize()
        ke = max(1, min(args.steps, 5))
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(ke + 1)]
        evs[0].record(stream)
        for q in range(ke):
            f.solve_host(av, ns, bh, nt, out=xh)  # synchronous: returns with x on the host
            evs[q + 1].record(stream)
        torch.cuda.synchronize()
        ems = evs[0].elapsed_time(evs[ke]) / ke
        ems_steps = [evs[q].elapsed_time(evs[q + 1]) for q in range(ke)]
        if world > 1:
            tt = torch.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": nnz_S_total * ns / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(a.values.nbytes + 8 * n), "d2h_bytes_per_step": int(8 * n),
               "ms_per_step": ems, "ms_steps": ems_steps}
        # the e2e roofline: the step cannot end before its input bytes are on the device -- one
        # pinned copy of the same bytes (values + b) on an idle stream, measured here, after the
        # timed region (the best of 3)
        hb = torch.empty(int(a.values.nbytes // 8 + n), dtype=torch.float64).pin_memory()
        db = torch.empty_like(hb, device=dev)
        cs = torch.cuda.Stream()
        best = 1e30
        for _ in range(3):
            torch.cuda.synchronize()
            with torch.cuda.stream(cs):
                c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                c0.record(cs)
                db.copy_(hb, non_blocking=True)
                c1.record(cs)
            torch.cuda.synchronize()
            best = min(best, c0.elapsed_time(c1))
        del hb, db
        e2e["h2d_floor_ms"] = best
        e2e["h2d_gbs"] = (a.values.nbytes + 8 * n) / (best * 1e-3) / 1e9
        e2e["frac_of_h2d_floor"] = best / ems

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and kind != "3dof":
        cores, model = cpu_info()
        planes = args.cpu_planes or cpu_planes_for(kind, g, k, ns, nt, cores)
        r = cpu_sample(kind, g, k, ns, nt, planes, cores)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["threads"], "cpu": model,
               "kind": "oracle", "sample": r["sample"], "seconds": r["seconds"]}

    gm = None
    if kind == "aniso7pt" and world == 1 and not args.no_gmres:
        gm, b_gm = gmres_arms(args, f, a, ns, stream)
        if cpu is not None and args.arm_c:
            cpu["gmres_arm_c"] = gmres_arm_c(a, b_gm, cpu["cores"])
    launches_per_step = 2 + 2 * ns + 2 * nt + (3 if info.startswith("path=bsr") else 0)
    # the full sweep kernel (sweeps 2..ns) against the measured copy bandwidth, on the bytes its
    # layout moves (no index bytes on the template path); the SURVEY 8(d) CSR model alongside
    roof = {"bound": "hbm", "kernel": "fastilu_tsell_sweep_st" if "staged=1" in info
            else "sweep_kernel", "achieved": achieved, "peak": peak,
            "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "bytes_per_launch": lm["B_f"], "byte_model": lm["kind"],
            "survey_model": {"bytes_per_launch": bm["B_f"],
                             "achieved": bm["B_f"] / (per_launch_ms * 1e-3) / 1e9,
                             "frac": bm["B_f"] / (per_launch_ms * 1e-3) / 1e9 / peak,
                             "note": "SURVEY 8(d): 4 index bytes per entry the layout never "
                                     "loads; not a bandwidth"}}
    if traffic:
        roof["traffic_achieved"] = traffic / (per_launch_ms * 1e-3) / 1e9
        roof["traffic_frac"] = roof["traffic_achieved"] / peak
    if info.startswith("path=bsr"):
        roof = bsr_roofline(info, n, sweep_ms / max(ns, 1))
    else:  # the secondary bound of the staged sweep (its shared-memory port)
        roof["smem_port"] = smem_port(info, n, per_launch_ms, clk.get("sm_mhz"),
                                      torch.cuda.get_device_properties(dev).multi_processor_count)
    composite = lm["B_init"] + (lm["B_f1"] + (ns - 1) * lm["B_f"] if ns >= 1 else 0) + \
        lm["B_apply"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded stencil generator, b ~ U[0.5,1.5))",
            "config": {"workload": args.workload, "grid": g, "stencil": kind, "level_k": k,
                       "nsweeps": ns, "ntrisweeps": nt, "tol": args.tol, "n": n, "nnz_A": nnz_A, "nnz_S": nnz_S,
                       "parallelism": (f"row-block z-slabs x{world}, NCCL halos"
                                       if world > 1 else "1gpu"),
                       "comm": ({"nccl_ranks": world, "halo_bytes_per_sweep":
                                 int(dict(re.findall(r"(\w+)=(\S+)", info)).get(
                                     "halo_bytes", 0))} if world > 1 else None),
                       "global_grid": [g, g, g * world],
                       "l2": "working set >> 126 MB L2 (no flush needed)"},
            "sweep_nnz_updates_per_s": nnz_S * ns / (sweep_ms * 1e-3),
            "sweep_ms": sweep_ms, "sweep1_ms": float(np.mean(t_first)),
            "sweep_launch_ms": per_launch_ms, "init_ms": float(np.mean(t_init)), "apply_ms": t_apply,
            # bandwidths on the bytes the layout moves (layout_model), fraction of the measured
            # copy peak; the SURVEY model's figures (index bytes included) under "survey_model"
            "trisolve_gbs": lm["B_apply"] / (t_apply * 1e-3) / 1e9 if t_apply > 0 else None,
            "trisolve_frac": (lm["B_apply"] / (t_apply * 1e-3) / 1e9 / peak
                              if t_apply > 0 else None),
            "composite_gbs": composite / (ms * 1e-3) / 1e9,
            "composite_frac": composite / (ms * 1e-3) / 1e9 / peak,
            "bytes_per_step": {"layout": composite, "survey_model": (
                bm["B_init"] + ns * bm["B_f"] + bm["B_apply"]), "byte_model": lm["kind"]},
            "roofline": roof,
            "gmres": gm,
            "clocks": clk, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "cpu_baseline": cpu,
            "setup_s": {"generate": t_gen, "create": t_setup},
            "kernel_config": info,
        }
        print(json.dumps(line), flush=True)
    f.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4_27pt_256_ilu1", choices=sorted(P.WORKLOADS))
    ap.add_argument("--nsweeps", type=int, default=None)
    ap.add_argument("--ntri", type=int, default=None)
    ap.add_argument("--cpu-planes", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-gmres", action="store_true", help="config 5: skip the GMRES arms")
    ap.add_argument("--arm-c", action="store_true",
                    help="config 5: add arm C (CPU oracle exact ILU(0) + substitution; minutes)")
    ap.add_argument("--gmres-ntri", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--tol", type=float, default=None,
                    help="sweeps to convergence: stop at r(s-1) <= tol ||Ahat|_S||_F (config 3)")
    args = ap.parse_args()
    kind, g, k, ns, nt = P.WORKLOADS[args.workload]
    ns = args.nsweeps if args.nsweeps is not None else ns
    nt = args.ntri if args.ntri is not None else nt
    wl = (kind, g, k, ns, nt)
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # launched without torchrun: start one rank per GPU ourselves (same arguments), so that
        # `python bench.py --gpus N` runs N ranks instead of silently running one
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world is not None and int(world) != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; refusing to report",
              file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
