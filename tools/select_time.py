import sys, time
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200.engine import get_engine
eng = get_engine()
for R in (100000, 1000000, 10000000):
    v = torch.rand(R, dtype=torch.float64, device='cuda') * 0.1
    out = torch.empty(4, dtype=torch.float64, device='cuda')
    ranks = [int(R * q) for q in (0.9, 0.95, 0.99, 0.999)]
    for _ in range(3): eng.select_ranks(v, ranks, out=out)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): eng.select_ranks(v, ranks, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    m = v.max(); torch.cuda.synchronize()
    e0.record()
    for _ in range(50): v.max()
    e1.record(); torch.cuda.synchronize()
    print(f"R={R}: select {ms*1e3:.1f} us per call; torch max {e0.elapsed_time(e1)/50*1e3:.1f} us", flush=True)
