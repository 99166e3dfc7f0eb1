"""One rank of the CPU multi-rank checks (gloo, 127.0.0.1), launched by test_multirank_gloo.py.

Each rank owns a z-slab of a global stencil matrix and reproduces, from its row block plus the
`fastilu_required_lead_rows` rows below it, (1) the exact ILU(k) pattern of its owned rows and
of the ghost rows it reads from its lower neighbour (the product's host setup,
fastilu_symbolic_window), and (2) the oracle's factors and x of its owned rows from a windowed
oracle run.  Everything is gathered over gloo; every rank checks it against the neighbours and
rank 0 against the global single-rank computation.  Prints one JSON line {"ok": ...}.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import paper_2506_05793_b200 as F  # noqa: E402
import problems as P  # noqa: E402


def split_planes(gz, world):
    return [(gz * r // world, gz * (r + 1) // world) for r in range(world)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int)
    ap.add_argument("--world", type=int)
    ap.add_argument("--port", type=int)
    ap.add_argument("--kind", default="27pt")
    ap.add_argument("--g", type=int, default=5)
    ap.add_argument("--gz", type=int, default=14)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--ns", type=int, default=3)
    ap.add_argument("--nt", type=int, default=3)
    a = ap.parse_args()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{a.port}", rank=a.rank,
                            world_size=a.world)
    g, gz, k = a.g, a.gz, a.k
    plane = g * g
    global_n = plane * gz
    z0, z1 = split_planes(gz, a.world)[a.rank]
    row_begin, row_end = z0 * plane, z1 * plane
    bw = P.bandwidth(a.kind, g)
    need = F.fastilu_required_lead_rows(bw, k)
    lead_planes = min(z0, -(-need // plane))
    n_lead = lead_planes * plane
    blk = P.make(a.kind, g, gz, planes=(z0 - lead_planes, z1))
    row0 = row_begin - n_lead
    # pattern of [row_begin - (k+1) bw, row_end): owned rows + every possible ghost row
    gcap = min(n_lead, (k + 1) * bw)
    rp, ci, lev = F.fastilu_symbolic_window(blk.row_ptr, blk.col_idx, row0, global_n,
                                            row_begin - gcap, row_end, k)
    own = slice(int(rp[gcap]), int(rp[-1]))
    own_rp = rp[gcap:] - rp[gcap]
    own_ci, own_lev = ci[own], lev[own]
    # ghost rows: the lower rows my owned rows reference
    G = row_begin - int(min(own_ci.min(), row_begin)) if own_ci.size else 0
    Hh = int(max(own_ci.max(), row_end - 1)) - (row_end - 1) if own_ci.size else 0
    gs = int(rp[gcap - G])
    ghost = dict(rp=(rp[gcap - G:gcap + 1] - gs).tolist(), ci=ci[gs:int(rp[gcap])].tolist(),
                 lev=lev[gs:int(rp[gcap])].tolist())
    # windowed oracle for the owned planes (margins: DESIGN.md "windowed oracle")
    a_full = P.make(a.kind, g, gz)
    b = P.rhs_positive(global_n)
    lo_p = max(0, z0 - (a.ns + a.nt + k + 4))
    hi_p = min(gz, z1 + a.nt + 2)
    lo, hi, fw, xw = oracle.windowed(a_full, plane, lo_p, hi_p, k, a.ns, b_full=b, ntri=a.nt)
    wrp = fw.pattern.row_ptr
    fvals = fw.vals[wrp[row_begin - lo]:wrp[row_end - lo]]
    xown = xw[row_begin - lo:row_end - lo]
    mine = dict(rank=a.rank, row_begin=row_begin, row_end=row_end, G=G, H=Hh,
                own_rp=own_rp.tolist(), own_ci=own_ci.tolist(), own_lev=own_lev.tolist(),
                ghost=ghost, vals=fvals.tolist(), x=xown.tolist())
    allr = [None] * a.world
    dist.all_gather_object(allr, mine)
    ok, why = True, []
    # neighbour consistency: my ghost rows == the previous rank's last G owned rows
    if a.rank > 0:
        prev = allr[a.rank - 1]
        prp = np.array(prev["own_rp"])
        nprev = prp.size - 1
        if G > nprev:
            ok, why = False, why + ["ghost rows reach beyond the lower neighbour"]
        else:
            s = int(prp[nprev - G])
            want_rp = (prp[nprev - G:] - s).tolist()
            want_ci = prev["own_ci"][s:]
            want_lev = prev["own_lev"][s:]
            if want_rp != ghost["rp"] or want_ci != ghost["ci"] or want_lev != ghost["lev"]:
                ok, why = False, why + ["ghost pattern differs from the owner's rows"]
    if a.rank + 1 < a.world and Hh > allr[a.rank + 1]["row_end"] - allr[a.rank + 1]["row_begin"]:
        ok, why = False, why + ["upper halo beyond the upper neighbour"]
    if a.rank == 0:
        rpg, cig, levg = F.fastilu_symbolic(a_full.row_ptr, a_full.col_idx, k)
        cat_ci = np.concatenate([np.array(r["own_ci"], dtype=np.int32) for r in allr])
        cat_lev = np.concatenate([np.array(r["own_lev"], dtype=np.int8) for r in allr])
        cat_rp = [0]
        for r in allr:
            cat_rp += (np.array(r["own_rp"][1:]) + cat_rp[-1]).tolist()
        if not (np.array_equal(cat_ci, cig) and np.array_equal(cat_lev, levg)
                and np.array_equal(np.array(cat_rp), rpg)):
            ok, why = False, why + ["partitioned pattern != global pattern"]
        fg = oracle.compute(a_full, k, a.ns)
        xg = oracle.apply(fg, b, a.nt)
        cat_v = np.concatenate([np.array(r["vals"]) for r in allr])
        cat_x = np.concatenate([np.array(r["x"]) for r in allr])
        if not np.array_equal(cat_v, fg.vals):
            ok, why = False, why + ["partitioned oracle factors != global (bitwise)"]
        if not np.array_equal(cat_x, xg):
            ok, why = False, why + ["partitioned oracle x != global (bitwise)"]
    print(json.dumps({"rank": a.rank, "ok": ok, "why": why, "G": G, "H": Hh}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
