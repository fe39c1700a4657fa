"""Device time per n-row of the config-2 sweep (grouped path), with the per-kernel-kind split."""
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
kinds_total = {}
for n in bench.NS:
    plans = lambda: [mc._CellPlan(zk.SimulationConfig(n=n, support=sup, gamma=g, base_seed=1, replicates=R, repetitions=1)) for g in bench.GAMMAS]
    mc._enqueue_plans(eng, plans()); torch.cuda.synchronize()
    eng.set_timing(True); eng.kernel_times()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); mc._enqueue_plans(eng, plans()); e1.record(); torch.cuda.synchronize()
    kt = eng.kernel_times(); eng.set_timing(False)
    ms = e0.elapsed_time(e1)
    tot += ms
    split = " ".join(f"{k} {v[0]:.1f}/{v[1]}" for k, v in kt.items() if v[1])
    for k, v in kt.items():
        kinds_total[k] = kinds_total.get(k, 0.0) + v[0]
    print(f"n={n}: row {ms:.1f} ms | {split}", flush=True)
print(f"total {tot:.1f} ms -> {len(bench.NS) * len(bench.GAMMAS) * R / tot * 1e3 / 1e6:.1f} M rep/s | "
      + " ".join(f"{k} {v:.1f}" for k, v in kinds_total.items() if v))
