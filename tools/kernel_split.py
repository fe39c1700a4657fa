"""Time the draw and fit/KS kernels of one staged cell separately (CUDA events around each launch)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf

g = float(sys.argv[1]); n = int(sys.argv[2]); R = int(sys.argv[3]) if len(sys.argv) > 3 else 1000000
eng = engine.get_engine()
ks = torch.empty(R, dtype=torch.float64, device='cuda'); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device='cuda')
u = torch.empty(R * eng.staging_stride(n), dtype=torch.int32, device='cuda')
t = eng.table(g, None, lambda: sampling_cdf(g, Support(None)))
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for it in range(2):
    e[0].record(); eng.stage_uniforms(1, 0, 0, R, n, u); e[1].record()
    eng.run_replicates_staged(t, None, g, n, 1, 0, 0, R, u, 0, R, ks, gh, st); e[2].record()
    eng.run_replicates(t, None, g, n, 1, 0, 0, R, ks, gh, st); e[3].record()
    torch.cuda.synchronize()
print(f"g={g} n={n}: stage {e[0].elapsed_time(e[1]):.2f} ms, staged draw+fit {e[1].elapsed_time(e[2]):.2f} ms, philox draw+fit {e[2].elapsed_time(e[3]):.2f} ms")
