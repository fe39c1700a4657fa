"""Device time per n-row of the config-2 sweep through the grouped (staged-uniform) path."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1305_6738_b200 as zk
from paper_1305_6738_b200 import montecarlo as mc
from paper_1305_6738_b200.engine import get_engine
import bench

eng = get_engine()
R = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
sup = zk.Support.unbounded()
tot = 0.0
for n in bench.NS:
    plans = lambda: [mc._CellPlan(zk.SimulationConfig(n=n, support=sup, gamma=g, base_seed=1, replicates=R, repetitions=1)) for g in bench.GAMMAS]
    mc._enqueue_plans(eng, plans()); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ev = []
    e0.record(); mc._enqueue_plans(eng, plans(), kernel_events=ev); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1); kms = sum(a.elapsed_time(b) for a, b in ev)
    tot += ms
    print(f"n={n}: row {ms:.1f} ms, replicate kernels {kms:.1f} ms ({len(ev)} launches)", flush=True)
print(f"total {tot:.1f} ms -> {len(bench.NS) * len(bench.GAMMAS) * R / tot * 1e3 / 1e6:.1f} M rep/s")
if len(sys.argv) > 2:
    n = int(sys.argv[2])
    plans = [mc._CellPlan(zk.SimulationConfig(n=n, support=sup, gamma=g, base_seed=1, replicates=R, repetitions=1)) for g in bench.GAMMAS]
    ev = []
    mc._enqueue_plans(eng, plans, kernel_events=ev); torch.cuda.synchronize()
    per = {}
    for i, (a, b) in enumerate(ev):
        g = bench.GAMMAS[i % len(bench.GAMMAS)]
        per[g] = per.get(g, 0) + a.elapsed_time(b)
    print(" ".join(f"{g}:{v:.1f}" for g, v in per.items()))
