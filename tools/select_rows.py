"""Device time of one sweep row's batched selection: 21 arrays x 10^6 KS-like values, 4 ranks."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200.engine import get_engine

eng = get_engine()
R, A = 1000000, 21
g = torch.Generator(device='cuda').manual_seed(1)
vals = [torch.exp(torch.randn(R, device='cuda', dtype=torch.float64, generator=g) * 0.4 - 3.5) for _ in range(A)]
sts = [torch.zeros(R, dtype=torch.uint8, device='cuda') for _ in range(A)]
outs = [torch.empty(4, dtype=torch.float64, device='cuda') for _ in range(A)]
worst = [torch.zeros(1, dtype=torch.uint8, device='cuda') for _ in range(A)]
ranks = [int(R * q) for q in (0.9, 0.95, 0.99, 0.999)]
for label, jobs in (("with status", [(v, ranks, o, s, w) for v, o, s, w in zip(vals, outs, sts, worst)]),
                    ("values only", [(v, ranks, o) for v, o in zip(vals, outs)])):
    for _ in range(3):
        eng.select_many(jobs)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        eng.select_many(jobs)
    e1.record(); torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per row", flush=True)
want = [torch.sort(v).values[ranks] for v in vals[:3]]
print("exact:", all(torch.equal(o, w) for o, w in zip(outs[:3], want)))
