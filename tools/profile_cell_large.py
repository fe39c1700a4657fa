"""One heavy-tailed cell (K = inf, gamma = 1.25, n = 5x10^4, 5x10^4 replicates) run twice: the unit
ncu profiles long_tail_kernel with (the draw_stats -> fit_ks -> long_tail path above n = 16384)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1305_6738_b200 import engine  # noqa: E402
from paper_1305_6738_b200.distribution import Support, sampling_cdf  # noqa: E402

g, n, R = 1.25, 50000, 50000
eng = engine.get_engine()
t = eng.table(g, None, lambda: sampling_cdf(g, Support(None)))
ks = torch.empty(R, dtype=torch.float64, device="cuda")
gh = torch.empty_like(ks)
st = torch.empty(R, dtype=torch.uint8, device="cuda")
for _ in range(2):
    eng.run_replicates(t, None, g, n, 1, 0, 0, R, ks, gh, st)
torch.cuda.synchronize()
print("ok", float(ks.mean()), int(st.max()))
