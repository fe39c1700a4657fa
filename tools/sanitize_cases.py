"""Every engine kernel path once, on small shapes: the program compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck, one tool per process):

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py

row_draw_kernel (list tails, dense per-draw and all-cut counts), fit_ks_kernel with page
compaction, retry_kernel, lane_row_kernel (lane tails, warp tails, retries, double
failures), draw_stats_kernel (16384 < n <= 65535), replicate_kernel (overflow slab, direct-sum
MLE), the cooperative selection and the distributed selection steps, user-sample fits, series,
solves, uniforms, draws, the fast stream.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_6738_b200 as zk  # noqa: E402
from paper_1305_6738_b200 import engine  # noqa: E402
from paper_1305_6738_b200.distribution import Support, sampling_cdf  # noqa: E402


def cell(eng, K, g, n, R, seed=3):
    t = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
    ks = torch.empty(R, dtype=torch.float64, device="cuda")
    gh = torch.empty_like(ks)
    st = torch.empty(R, dtype=torch.uint8, device="cuda")
    eng.run_replicates(t, K, g, n, seed, 0, 0, R, ks, gh, st)
    torch.cuda.synchronize()
    return ks, gh, st


def main():
    eng = engine.get_engine()
    # row kernel + fit + retry + batched selection (unbounded list tails; dense K = 1000 both ways)
    zk.build_table(ns=(150, 700), gammas=(1.3, 2.0, 3.0), support=zk.Support.unbounded(), base_seed=2, replicates=256,
                   repetitions=1)
    zk.build_table(ns=(300, 5000), gammas=(0.5, 1.5), support=zk.Support.finite(1000), base_seed=2, replicates=128,
                   repetitions=1)
    # heavy tails: fit_ks_kernel's page passes with in-place compaction
    cell(eng, None, 1.1, 12000, 64)
    # lane kernel: lane tails, warp tails, retries and double failures
    cell(eng, None, 1.1, 127, 256)
    cell(eng, None, 2.5, 37, 512)
    cell(eng, 20, -30.0, 3, 256)
    cell(eng, 1000, 0.25, 10, 256)
    # two-kernel path above the row kernel, large-n kernel with its overflow slab
    cell(eng, None, 1.5, 20000, 32)
    cell(eng, None, 1.3, 70000, 8)
    # direct-sum MLE (replicate_kernel at every n)
    eng.set_mle_mode(True)
    cell(eng, None, 2.0, 200, 64)
    cell(eng, 50, 1.0, 40, 64)
    eng.set_mle_mode(False)
    # fast stream
    zk.set_rng("philox4x32")
    zk.build_table(ns=(20, 300), gammas=(1.7, 2.4), support=zk.Support.unbounded(), base_seed=9, replicates=256,
                   repetitions=1)
    zk.set_rng("numpy")
    # selection: single array (signed keys), batched
    rng = np.random.default_rng(1)
    zk.order_quantiles(rng.standard_normal(100_000), (0.1, 0.5, 0.9, 0.999))
    # user samples, series, solves, uniforms, draws
    samples = [zk.sample(zk.ZipfModel(2.0, zk.Support.unbounded()), 300, zk.RandomStream.for_replicate(5, 0, i))
               for i in range(4)]
    zk.fit_samples([s.observations for s in samples], zk.Support.unbounded())
    zk.zeta_log_moments(2.5)
    zk.finite_log_moments(1.0, 1000)
    zk.mle_gamma(samples[0], zk.Support.unbounded())
    zk.ks_statistic(samples[0], zk.ZipfModel(2.0, zk.Support.unbounded()))
    zk.cdf(zk.ZipfModel(2.0, zk.Support.unbounded()), 5000)
    zk.RandomStream([1, 2, 3, 4]).uniforms(17)
    torch.cuda.synchronize()
    # determinism under contention: the row kernel's bucketing order varies between runs (shared
    # atomics), its outputs must not; three runs of mixed rows, every replicate bitwise
    from paper_1305_6738_b200 import montecarlo as mc

    def row(K, n, gammas):
        plans = [mc._CellPlan(zk.SimulationConfig(n=n, support=zk.Support(K), gamma=g, base_seed=4, replicates=4096,
                                                  repetitions=1)) for g in gammas]
        keep = {}
        mc._enqueue_plans(eng, plans, keep=keep)
        torch.cuda.synchronize()
        return {k: tuple(t.cpu().numpy() for t in v) for k, v in keep.items()}

    for K, n, gammas in ((None, 700, (1.2, 1.6, 2.4, 3.3)), (1000, 2500, (0.5, 1.0, 1.8)), (None, 60, (1.1, 2.0))):
        runs = [row(K, n, gammas) for _ in range(3)]
        for other in runs[1:]:
            for key in runs[0]:
                for a, b in zip(runs[0][key], other[key]):
                    assert np.array_equal(a, b), ("nondeterministic", K, n, key)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
