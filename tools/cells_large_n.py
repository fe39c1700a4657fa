"""Heavy-tailed single cells (the paper's unbounded grid above n = 10^4): device time per cell and
the per-kind split (CUDA events around every launch).

    python tools/cells_large_n.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1305_6738_b200 import engine  # noqa: E402
from paper_1305_6738_b200.distribution import Support, sampling_cdf  # noqa: E402

eng = engine.get_engine()
CELLS = [(None, 1.25, 50000, 50000), (None, 1.5, 50000, 50000), (None, 2.0, 50000, 50000), (None, 4.0, 50000, 50000),
         (None, 1.25, 20000, 50000), (None, 1.25, 5000, 50000), (None, 1.25, 1000, 50000)]
for K, g, n, R in CELLS:
    ks = torch.empty(R, dtype=torch.float64, device="cuda")
    gh = torch.empty_like(ks)
    st = torch.empty(R, dtype=torch.uint8, device="cuda")
    t = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
    eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st)
    eng.set_timing(True)
    eng.kernel_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st)
    e1.record()
    torch.cuda.synchronize()
    kt = eng.kernel_times()
    eng.set_timing(False)
    ms = e0.elapsed_time(e1)
    split = " ".join(f"{k} {v[0]:.2f}" for k, v in kt.items() if v[1])
    print(f"K={K} g={g} n={n} R={R}: {ms:.2f} ms -> {R * n / ms / 1e6:.1f} G draws/s | {split}", flush=True)
