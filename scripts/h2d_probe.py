"""Host-to-device copy probe for the e2e path: one pinned copy of the c4 step's input bytes
(3.73 GB: A's values + b) as a single cudaMemcpyAsync, and as 16 chunks on one stream, timed with
CUDA events -- the PCIe ceiling that fastilu_solve_host's 76.5 ms/step is compared against.
    python scripts/h2d_probe.py [--gb 3.73]"""
import argparse

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--gb", type=float, default=3.729858496)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
n = int(args.gb * 1e9) // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ("single", "chunks16"):
    best = 1e30
    for _ in range(args.reps):
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            e0.record(s)
            if mode == "single":
                d.copy_(h, non_blocking=True)
            else:
                c = (n + 15) // 16
                for q in range(16):
                    d[q * c:(q + 1) * c].copy_(h[q * c:(q + 1) * c], non_blocking=True)
            e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{mode}: {best:.2f} ms for {8 * n / 1e9:.2f} GB = {8 * n / best / 1e6:.1f} GB/s")
