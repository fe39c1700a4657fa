"""One sweep row through zks_run_cells (the unit ncu profiles): K, n, gammas, R replicates.

    python tools/profile_row.py --n 1000 --k inf --gammas 1.5:3.5:0.1 --r 100000 --iters 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1000)
ap.add_argument("--k", default="inf")
ap.add_argument("--gammas", default="1.5:3.5:0.1")
ap.add_argument("--r", type=int, default=100000)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--chunk-gb", type=float, default=0.0)
args = ap.parse_args()
K = None if args.k == "inf" else int(args.k)
lo, hi, step = (float(x) for x in args.gammas.split(":"))
gammas = [round(g, 6) for g in np.arange(lo, hi + step / 2, step)]
eng = engine.get_engine()
if args.chunk_gb:
    eng.set_chunk_bytes(int(args.chunk_gb * 2**30))
tables = [eng.table(g, K, lambda g=g: sampling_cdf(g, Support(K))) for g in gammas]
outs = [(torch.empty(args.r, dtype=torch.float64, device="cuda"), torch.empty(args.r, dtype=torch.float64, device="cuda"),
         torch.empty(args.r, dtype=torch.uint8, device="cuda")) for _ in gammas]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(args.iters):
    ev[0].record()
    for j0 in range(0, len(gammas), 32):
        eng.run_cells(tables[j0 : j0 + 32], K, gammas[j0 : j0 + 32], args.n, 1, 0, 0, args.r, outs[j0 : j0 + 32])
    ev[1].record()
    torch.cuda.synchronize()
    print(f"iter {it}: {ev[0].elapsed_time(ev[1]):.3f} ms for {len(gammas)} cells x {args.r} (n={args.n}, K={args.k})",
          flush=True)
print("ok", float(outs[0][0].mean()), max(int(o[2].max()) for o in outs))
