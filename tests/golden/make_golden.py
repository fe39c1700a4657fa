"""Generate golden vectors from the reference ``zipfks`` package itself.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports the UNMODIFIED reference from ``/root/reference/pkg/src`` and
records, per stream / replicate, exactly what the reference computes.  The
output ``tests/golden/golden.npz`` is committed; nothing at test time (and
nothing on the GPU box) reads ``/root/reference``.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

# (support K or 0 for unbounded, gamma, n, base_seed, repetition, replicates)
CELLS = [
    (0, 2.5, 100, 1, 0, 64),        # BASELINE config 1
    (0, 1.5, 10, 1, 0, 64),
    (0, 1.5, 1000, 1, 0, 32),
    (0, 3.5, 50, 7, 1, 64),
    (0, 1.25, 400, 3, 0, 32),       # sparse KS path (kmax > 4096) almost always
    (0, 1.05, 50, 11, 0, 32),       # smallest admissible unbounded exponent
    (0, 2.0, 100000, 1, 0, 4),      # BASELINE config 4 (large n)
    (1000, 0.5, 100, 1, 0, 64),     # BASELINE config 3
    (1000, 1.0, 10, 5, 2, 64),
    (1000, 2.0, 10000, 1, 0, 8),
    (20, 1.0, 1000, 20240001, 0, 32),
    (2, 1.0, 10, 9, 0, 64),
    (5000, 1.5, 500, 4, 0, 16),     # finite support above the 4096 seam
    (20, 0.25, 20, 2, 3, 64),
    (20, -30.0, 3, 101, 0, 16),     # estimator failures: retries and double failures
]

SAMPLE_KEEP = 4  # store the drawn integers of the first few replicates per cell

STREAMS = [
    (1, 0, 0), (1, 0, 5), (0, 0, 0), (2**64 - 1, 3, 2**32 + 7), (20240001, 9, 49999),
    (1, 0, 2**32 + 3), (12345678901234, 7, 0), (77, 2**31, 2**40 + 1),
]


def main() -> None:
    sys.path.insert(0, REF)
    import zipfks
    from zipfks import distribution as D
    from zipfks import estimate as E
    from zipfks import gof as G
    from zipfks import montecarlo as M

    assert zipfks.__version__ == "1.0.0"
    out: dict[str, np.ndarray] = {}

    # streams: raw uint64 words and uniforms straight from numpy as the reference uses it
    for i, (s, r, x) in enumerate(STREAMS):
        gen = np.random.Generator(np.random.Philox(np.random.SeedSequence([s, r, x])))
        bg = gen.bit_generator
        out[f"stream{i}_key"] = np.asarray([s, r, x], dtype=np.uint64)
        out[f"stream{i}_philox_key"] = bg.state["state"]["key"].copy()
        out[f"stream{i}_u"] = D.RandomStream.for_replicate(s, r, x).uniforms(37)
        raw = np.random.Generator(np.random.Philox(np.random.SeedSequence([s, r, x])))
        out[f"stream{i}_raw"] = raw.bit_generator.random_raw(9)

    cell_rows = []
    for ci, (k, gamma, n, seed, rep, count) in enumerate(CELLS):
        support = D.Support(k=None if k == 0 else k)
        cfg = M.SimulationConfig(n=n, support=support, gamma=gamma, base_seed=seed,
                                 replicates=max(count, 100), repetitions=rep + 1)
        model = M._generating_model(gamma, support.k)
        out[f"cell{ci}_cdf_head"] = model._sampling_cdf[:64].copy()
        out[f"cell{ci}_cdf_tail"] = model._sampling_cdf[-8:].copy()
        ks = np.full(count, np.nan)
        gh = np.full(count, np.nan)
        target = np.full(count, np.nan)
        status = np.zeros(count, dtype=np.uint8)
        for idx in range(count):
            got = None
            for attempt, stream_index in enumerate((idx, idx + M._RETRY_OFFSET)):
                stream = D.RandomStream.for_replicate(seed, rep, stream_index)
                drawn = D.sample(model, n, stream)
                t = E.log_mean(drawn)
                if support.is_finite and int(drawn.observations.min()) == support.k:
                    t -= (np.log(support.k) - np.log(support.k - 1)) / n
                target[idx] = t
                if attempt == 0 and idx < SAMPLE_KEEP:
                    out[f"cell{ci}_sample{idx}"] = drawn.observations.astype(np.int32)
                try:
                    g = E.mle_gamma(drawn, support, E.DEFAULT_SETTINGS)
                except E.NoRootError:
                    continue
                fitted = D.ZipfModel(gamma=g, support=support)
                got = (G.ks_statistic(drawn, fitted).statistic, g, attempt)
                break
            if got is None:
                status[idx] = 2
            else:
                ks[idx], gh[idx], status[idx] = got
                # cross-check against the reference's own replicate driver
                o = M.run_replicate(cfg, idx, rep)
                assert (o.ks, o.gamma_hat) == (got[0], got[1])
        out[f"cell{ci}_ks"] = ks
        out[f"cell{ci}_gamma_hat"] = gh
        out[f"cell{ci}_target"] = target
        out[f"cell{ci}_status"] = status
        cell_rows.append([k, gamma, n, seed, rep, count])
        print(f"cell {ci}: K={k or 'inf'} gamma={gamma} n={n}: status counts "
              f"{np.bincount(status, minlength=3).tolist()}", flush=True)
    out["cells"] = np.asarray(cell_rows, dtype=np.float64)

    # whole-repetition quantiles through the reference's run_simulation
    sims = [
        (20, 1.5, 50, 101, 400, 2),
        (0, 2.5, 100, 1, 1000, 1),
        (1000, 1.0, 200, 3, 300, 3),
    ]
    for si, (k, gamma, n, seed, reps_r, reps) in enumerate(sims):
        support = D.Support(k=None if k == 0 else k)
        cfg = M.SimulationConfig(n=n, support=support, gamma=gamma, base_seed=seed,
                                 replicates=reps_r, repetitions=reps)
        pairs = M.run_simulation(cfg, workers=1)
        out[f"sim{si}_cutoffs"] = np.asarray([c for _, c in pairs])
        ks0, gh0 = M.run_repetition(cfg, 0, None)
        out[f"sim{si}_rep0_ks"] = ks0
        out[f"sim{si}_rep0_gamma_hat"] = gh0
    out["sims"] = np.asarray(sims, dtype=np.float64)

    # series known values at a gamma grid (tier-2 inputs of the MLE / KS)
    grid_u = np.linspace(1.05, 20.0, 97)
    out["zeta_grid"] = grid_u
    out["zeta_moments"] = np.asarray([zipfks.series.zeta_log_moments(g) for g in grid_u])
    out["zeta_value"] = np.asarray([zipfks.series.zeta_value(g) for g in grid_u])
    grid_f = np.linspace(-20.0, 20.0, 81)
    out["finite_grid"] = grid_f
    out["finite_moments_1000"] = np.asarray([zipfks.series.finite_log_moments(g, 1000) for g in grid_f])
    logs = zipfks.series.natural_logs(65536).copy()
    import hashlib
    out["logs_65536_sha256"] = np.frombuffer(hashlib.sha256(logs.tobytes()).digest(), dtype=np.uint8)
    out["logs_sample_idx"] = np.arange(0, 65537, 97)
    out["logs_sample"] = logs[::97].copy()

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **out)

    known = {
        "normalization_1_K2": D.normalization(1.0, D.Support.finite(2)),
        "mle_112_K2": E.mle_gamma(D.Sample([1, 1, 2]), D.Support.finite(2)),
        "mle_222_K2": E.mle_gamma(D.Sample([2, 2, 2]), D.Support.finite(2)),
        "mle_22_K10": E.mle_gamma(D.Sample([2, 2]), D.Support.finite(10)),
        "mle_41_K10": E.mle_gamma(D.Sample([4, 1]), D.Support.finite(10)),
        "mle_short_tail_K20": E.mle_gamma(D.Sample([17, 19, 20, 20, 16]), D.Support.finite(20)),
        "mle_ones10_K20": E.mle_gamma(D.Sample([1] * 10), D.Support.finite(20)),
        "mle_ones50_inf": E.mle_gamma(D.Sample([1] * 50), D.Support.unbounded()),
        "ks_112_K2": G.ks_statistic(D.Sample([1, 1, 2]), D.ZipfModel(1.0, D.Support.finite(2))).statistic,
        "ks_222_K2": G.ks_statistic(D.Sample([2, 2, 2]), D.ZipfModel(1.0, D.Support.finite(2))).statistic,
        "ks_sparse_5000_6000": G._ks_sparse(np.array([5000, 6000]), D.ZipfModel(1.5, D.Support.unbounded()), 6000).statistic,
        "log_mean_124": E.log_mean(D.Sample([1, 2, 4])),
        "log_mean_ones10": E.log_mean(D.Sample([1] * 10)),
        "quantiles_r100_q029": M.order_quantiles(np.arange(100) / 100.0, [0.29]),
    }
    with open(os.path.join(OUT, "known.json"), "w") as fh:
        json.dump(known, fh, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
