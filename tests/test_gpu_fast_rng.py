"""The opt-in fast stream (set_rng("philox4x32")): tier-3 parity only.

Its samples differ from numpy's streams, its law does not: per cell, the cutoffs of 10
repetitions in each mode agree within Monte Carlo error (z = delta / sqrt(s1^2 + s2^2), s the
standard error of a 10-repetition mean from the per-repetition spread), over the paths the
stream feeds: the small-n kernel, the row kernel (128 <= n <= 16384), the two-kernel path above
it and the large-n kernel (n > 65535).
"""
import math

import numpy as np
import pytest


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

# (K, gamma, n, replicates per repetition)
CELLS = [(None, 1.5, 10, 50000), (None, 2.5, 100, 50000), (None, 2.0, 300, 50000), (None, 3.5, 1000, 50000),
         (1000, 1.0, 50, 50000), (1000, 0.5, 2000, 20000), (None, 2.0, 20000, 5000), (None, 2.0, 100000, 1000)]


def per_rep_quantiles(zk, K, g, n, R, seed, kind):
    from paper_1305_6738_b200 import montecarlo as mc

    eng = mc._engine()
    zk.set_rng(kind)
    try:
        plan = mc._CellPlan(zk.SimulationConfig(n=n, support=zk.Support(K), gamma=g, base_seed=seed, replicates=R,
                                                repetitions=10))
        mc._enqueue_plans(eng, [plan])
        mc._fetch_plans([plan])
        assert plan.host[1].max() < 2
        return np.asarray(plan.host[0])
    finally:
        zk.set_rng("numpy")


@pytest.mark.parametrize("K,g,n,R", CELLS)
def test_fast_stream_cutoffs_within_mc_error(K, g, n, R):
    import paper_1305_6738_b200 as zk

    exact = per_rep_quantiles(zk, K, g, n, R, 41, "numpy")
    fast = per_rep_quantiles(zk, K, g, n, R, 41, "philox4x32")
    assert not np.array_equal(exact, fast)  # a different stream
    s = np.sqrt(exact.var(axis=0, ddof=1) / 10 + fast.var(axis=0, ddof=1) / 10)
    z = (fast.mean(axis=0) - exact.mean(axis=0)) / np.maximum(s, 1e-9)
    assert np.all(np.abs(z) <= 5.0), (z, exact.mean(axis=0), fast.mean(axis=0))


def test_fast_stream_is_deterministic_and_sweep_consistent():
    import paper_1305_6738_b200 as zk

    zk.set_rng("philox4x32")
    try:
        kw = dict(ns=(20, 400), gammas=(1.7, 2.4), support=zk.Support.unbounded(), base_seed=9, replicates=3000,
                  repetitions=1)
        t1, t2 = zk.build_table(**kw), zk.build_table(**kw)
        assert t1.cells == t2.cells
        for (g, n), row in t1.cells.items():  # a sweep row equals its cells run alone
            cfg = zk.SimulationConfig(n=n, support=zk.Support.unbounded(), gamma=g, base_seed=9, replicates=3000,
                                      repetitions=1)
            assert row == tuple(c for _, c in zk.run_simulation(cfg))
    finally:
        zk.set_rng("numpy")
    with pytest.raises(ValueError):
        zk.set_rng("mt19937")
