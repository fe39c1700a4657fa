"""Bitwise determinism of the replicate kernels across launches and shard splits."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf

eng = engine.get_engine()
def run(K, g, n, first, count):
    t = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
    ks = torch.empty(count, dtype=torch.float64, device='cuda'); gh = torch.empty_like(ks); st = torch.empty(count, dtype=torch.uint8, device='cuda')
    eng.run_replicates(t, K, g, n, 1, 0, first, count, ks, gh, st)
    return ks.cpu().numpy(), gh.cpu().numpy()
for K, g, n in [(None, 1.5, 10), (None, 2.5, 100), (None, 1.5, 1000), (1000, 0.5, 100), (None, 2.0, 3000)]:
    R = 200000 if n <= 1000 else 20000
    a = run(K, g, n, 0, R)
    b = run(K, g, n, 0, R)
    parts = [run(K, g, n, s, e - s) for s, e in ((0, 777), (777, R // 2), (R // 2, R))]
    c = (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))
    d1 = np.flatnonzero(a[0] != b[0]); d2 = np.flatnonzero(a[0] != c[0]); d3 = np.flatnonzero(a[1] != c[1])
    print(K, g, n, "repeat-diff", d1.size, "shard-diff ks", d2.size, "gh", d3.size, d2[:5], (a[0][d2[:3]] - c[0][d2[:3]]) if d2.size else "")
