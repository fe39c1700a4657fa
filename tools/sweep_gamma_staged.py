"""Per-gamma split of the staged two-kernel path (draw / fit / retry) for one n of the config-2 sweep."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1305_6738_b200 import engine
from paper_1305_6738_b200.distribution import Support, sampling_cdf
import bench

eng = engine.get_engine()
R = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
ns = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (1000,)
ks = torch.empty(R, dtype=torch.float64, device='cuda'); gh = torch.empty_like(ks); st = torch.empty(R, dtype=torch.uint8, device='cuda')
for n in ns:
    ub = torch.empty(R * eng.staging_stride(n), dtype=torch.int32, device='cuda')
    eng.stage_uniforms(1, 0, 0, R, n, ub)
    torch.cuda.synchronize()
    tot = {}
    for g in bench.GAMMAS:
        t = eng.table(g, None, lambda: sampling_cdf(g, Support(None)))
        eng.run_replicates_staged(t, None, g, n, 1, 0, 0, R, ub, 0, R, ks, gh, st)
        torch.cuda.synchronize()
        eng.set_timing(True); eng.kernel_times()
        eng.run_replicates_staged(t, None, g, n, 1, 0, 0, R, ub, 0, R, ks, gh, st)
        kt = eng.kernel_times(); eng.set_timing(False)
        parts = {k: v[0] for k, v in kt.items() if v[1]}
        for k, v in parts.items():
            tot[k] = tot.get(k, 0.0) + v
        print(f"n={n} g={g:.1f} " + " ".join(f"{k} {v:.3f}" for k, v in parts.items()), flush=True)
    print(f"n={n} total " + " ".join(f"{k} {v:.2f}" for k, v in tot.items()), flush=True)
