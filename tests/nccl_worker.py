"""One rank of tests/test_gpu_multirank.py::test_nccl_two_processes (torchrun, one GPU per rank):
27-pt ILU(1) on z-slabs with the library's NCCL halos; rank 0 compares the gathered factors and
x with a single-GPU run bitwise and prints {"ok": ...}."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2506_05793_b200 as F  # noqa: E402
import problems as P  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    kind, g, gz, k, ns, nt = "27pt", 32, 40, 1, 3, 5
    plane = g * g
    z0, z1 = gz * rank // world, gz * (rank + 1) // world
    need = F.fastilu_required_lead_rows(P.bandwidth(kind, g), k)
    lp = min(z0, -(-need // plane))
    blk = P.make(kind, g, gz, planes=(z0 - lp, z1))
    uid = [F.fastilu_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    f = F.FastILU(blk.row_ptr, blk.col_idx, blk.values, k, device=local, rank=rank,
                  nranks=world, comm_kind=F.COMM_NCCL, nccl_unique_id=uid[0],
                  global_n=plane * gz, row_begin=z0 * plane, n_lead=lp * plane,
                  n=(z1 - z0) * plane)
    f.compute(ns)
    b = P.rhs_positive(plane * gz)
    tb = torch.tensor(b[z0 * plane:z1 * plane], device=f"cuda:{local}")
    tx = torch.empty_like(tb)
    f.apply(tb, tx, nt)
    torch.cuda.synchronize()
    mine = (f.factors()[0], tx.cpu().numpy(), f.info())
    allr = [None] * world
    dist.all_gather_object(allr, mine)
    ok, why = True, []
    if rank == 0:
        a = P.make(kind, g, gz)
        f1 = F.FastILU(a.row_ptr, a.col_idx, a.values, k, device=local)
        f1.compute(ns)
        tb1 = torch.tensor(b, device=f"cuda:{local}")
        tx1 = torch.empty_like(tb1)
        f1.apply(tb1, tx1, nt)
        torch.cuda.synchronize()
        if not np.array_equal(np.concatenate([r[0] for r in allr]), f1.factors()[0]):
            ok, why = False, why + ["factors differ from 1 GPU"]
        if not np.array_equal(np.concatenate([r[1] for r in allr]), tx1.cpu().numpy()):
            ok, why = False, why + ["x differs from 1 GPU"]
        print(json.dumps({"ok": ok, "why": why, "info": [r[2] for r in allr]}), flush=True)
    f.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
