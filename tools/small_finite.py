"""Device time of small-n finite-support cells (lane-per-replicate kernel), 10^6 replicates each."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf

eng = engine.get_engine()
R = 1000000
ks = torch.empty(R, dtype=torch.float64, device='cuda'); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device='cuda')
tot = 0.0
for K, g, n in [(1000, 0.5, 100), (1000, 1.0, 100), (1000, 1.5, 100), (1000, 0.5, 20), (1000, 1.0, 50), (20, 0.5, 100), (5000, 0.5, 100), (None, 1.25, 100)]:
    t = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
    eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1); tot += ms
    print(f"K={K} g={g} n={n}: {ms:.2f} ms  ks-sum {float(ks.sum()):.12e}", flush=True)
print(f"total {tot:.2f} ms")
