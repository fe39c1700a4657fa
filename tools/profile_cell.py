"""Run one config-2 cell a few times (the unit ncu profiles): K=inf, gamma, n, R replicates."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf

g = float(sys.argv[1]) if len(sys.argv) > 1 else 2.5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
R = int(sys.argv[3]) if len(sys.argv) > 3 else 200000
K = None if len(sys.argv) <= 4 or sys.argv[4] == 'inf' else int(sys.argv[4])
eng = engine.get_engine()
dev = 'cuda:0'
ks = torch.empty(R, dtype=torch.float64, device=dev); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device=dev)
t = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
for _ in range(3):
    eng.run_replicates(t, K, g, n, 1, 0, 0, R, ks, gh, st)
torch.cuda.synchronize()
print("ok", float(ks[:R].mean()), int(st[:R].max()))
