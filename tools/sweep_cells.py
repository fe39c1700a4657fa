"""Per-cell device time of the config-2 sweep (10^6 replicates per cell): where the time goes."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf
import bench

eng = engine.get_engine()
R = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
K = None
ks = torch.empty(R, dtype=torch.float64, device='cuda'); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device='cuda')
rows = []
for g in bench.GAMMAS:
    t = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
    for n in bench.NS:
        eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st); e1.record(); torch.cuda.synchronize()
        rows.append((e0.elapsed_time(e1), g, n))
tot = sum(r[0] for r in rows)
print(f"total kernel time {tot:.1f} ms")
byn = {}
for ms, g, n in rows:
    byn[n] = byn.get(n, 0) + ms
print("by n:", {n: round(v, 1) for n, v in byn.items()})
for ms, g, n in sorted(rows, reverse=True)[:15]:
    print(f"  g={g} n={n}: {ms:.2f} ms  ({R/ms/1e3:.1f} M rep/s)")
