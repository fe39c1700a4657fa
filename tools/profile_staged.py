"""One staged-uniform cell (the unit ncu profiles): K=inf, gamma, n in [128, 1024], R replicates."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf

g = float(sys.argv[1]) if len(sys.argv) > 1 else 2.5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
R = int(sys.argv[3]) if len(sys.argv) > 3 else 200000
eng = engine.get_engine()
ks = torch.empty(R, dtype=torch.float64, device='cuda'); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device='cuda')
u = torch.empty(R * eng.staging_stride(n), dtype=torch.int32, device='cuda')
t = eng.table(g, None, lambda: sampling_cdf(g, Support(None)))
eng.stage_uniforms(1, 0, 0, R, n, u)
for _ in range(3):
    eng.run_replicates_staged(t, None, g, n, 1, 0, 0, R, u, 0, R, ks, gh, st)
torch.cuda.synchronize()
print("ok", float(ks.mean()), int(st.max()))
