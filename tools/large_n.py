"""Device time of single cells at large n (configs 3 and 4 shapes): replicates/s per cell."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf

eng = engine.get_engine()
cells = [(1000, 1.0, 500, 200000), (1000, 1.0, 1000, 200000), (1000, 1.0, 2000, 100000), (1000, 1.0, 5000, 50000),
         (1000, 1.0, 10000, 20000), (1000, 0.5, 10000, 20000), (1000, 2.0, 10000, 20000),
         (None, 2.0, 1000, 200000), (None, 2.0, 2000, 100000), (None, 2.0, 10000, 20000),
         (None, 2.0, 30000, 10000), (None, 2.0, 65535, 4000), (1000, 1.0, 50000, 4000), (None, 2.0, 100000, 4000), (None, 2.0, 1000000, 400)]
for K, g, n, R in cells:
    ks = torch.empty(R, dtype=torch.float64, device='cuda'); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device='cuda')
    t = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
    eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st)
    eng.set_timing(True); eng.kernel_times()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st); e1.record(); torch.cuda.synchronize()
    kt = eng.kernel_times(); eng.set_timing(False)
    ms = e0.elapsed_time(e1)
    split = " ".join(f"{k} {v[0]:.2f}" for k, v in kt.items() if v[1])
    print(f"K={K} g={g} n={n} R={R}: {ms:.2f} ms -> {R / ms / 1e3:.2f} M rep/s, {R * n / ms / 1e6:.1f} G draws/s | {split} | max st {int(st.max())}", flush=True)
