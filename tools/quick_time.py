"""Per-cell device throughput probe (replicates/s) for a few cells."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf

eng = engine.get_engine()
R = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
cells = [(None, g, n) for g in (1.5, 2.5, 3.5) for n in (10, 100, 1000)] + [(1000, g, n) for g in (0.5, 1.0, 2.0) for n in (10, 100, 1000, 10000)] + [(None, 2.0, 100000)]
dev = 'cuda:0'
ks = torch.empty(R, dtype=torch.float64, device=dev); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device=dev)
for K, g, n in cells:
    r = R if n < 100000 else 2000
    t = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
    eng.run_replicates(t, K, g, n, 1, 0, 0, r, ks, gh, st)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); eng.run_replicates(t, K, g, n, 1, 0, 0, r, ks, gh, st); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"K={K} g={g} n={n}: {r/ms*1e3:,.0f} rep/s  ({ms:.2f} ms for {r})  max_status={int(st[:r].max())}", flush=True)
