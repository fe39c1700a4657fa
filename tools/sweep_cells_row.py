"""Per-gamma device time of one n-row's cells (run_replicates, 10^6 replicates each)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf
import bench

eng = engine.get_engine()
R = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
ns = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (10, 100)
ks = torch.empty(R, dtype=torch.float64, device='cuda'); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device='cuda')
for n in ns:
    line, tot = [], 0.0
    for g in bench.GAMMAS:
        t = eng.table(g, None, lambda: sampling_cdf(g, Support(None)))
        eng.run_replicates(t, None, g, n, 1, 0, 0, R, ks, gh, st)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); eng.run_replicates(t, None, g, n, 1, 0, 0, R, ks, gh, st); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1); tot += ms
        line.append(f"{g}:{ms:.2f}")
    print(f"n={n} total {tot:.1f} ms  " + " ".join(line), flush=True)
