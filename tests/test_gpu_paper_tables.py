"""Tier 3 over the paper's whole published grid (tests/golden/paper_tables.json).

Every support the paper tabulates (K = inf x 8 gammas, K in {20, 50, 100, 500, 1000} x 12 gammas;
pkg/src/zipfks/cli.py:24-26) at every n <= 10^4, with the paper's own protocol: 50,000
replicates x 10 repetitions averaged (the reference's defaults).  Both the published numbers and
ours carry that protocol's Monte Carlo error; it is measured from our per-repetition spread
(sigma_MC = std / sqrt(10)), so z = delta / sqrt(2 sigma_MC^2 + sigma_round^2) with the 4-decimal
rounding sigma_round = 0.5e-4 / sqrt(3).  sigma_MC is itself estimated from 10 repetitions, so
z is roughly t-distributed with 9 degrees of freedom (P(|t_9| <= 3) = 0.985).

Cells where the KS law has atoms (n <= 50 with gamma >= 2.5: most draws are 1 or 2, the
statistic takes few values and a quantile sits on an atom, where the per-repetition spread says
nothing about the error) are held to the fraction test only.  profiles/r02_config5/vs_paper.json
has the same comparison at 10^7 replicates per cell.
"""
import json
import math
import os

import numpy as np
import pytest


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

HERE = os.path.dirname(os.path.abspath(__file__))
NS = (10, 20, 30, 40, 50, 100, 500, 1000, 2000, 3000, 4000, 5000, 10000)
SIGMA_ROUND = 0.5e-4 / math.sqrt(3.0)


def _grid(zk, support, gammas, seed):
    from paper_1305_6738_b200 import montecarlo as mc

    eng = mc._engine()
    plans = [mc._CellPlan(mc.SimulationConfig(n=n, support=support, gamma=g, base_seed=seed, replicates=50000,
                                              repetitions=10)) for g in gammas for n in NS]
    mc._enqueue_plans(eng, plans)
    mc._fetch_plans(plans)
    out = {}
    for p in plans:
        cut = [c for _, c in mc._finish_cell(eng, p)]
        per_rep = np.asarray(p.host[0])
        out[(p.config.gamma, p.config.n)] = (cut, np.std(per_rep, axis=0, ddof=1) / math.sqrt(per_rep.shape[0]))
    return out


@pytest.mark.parametrize("label", ["inf", "20", "50", "100", "500", "1000"])
def test_paper_grid_within_mc_error(label):
    import paper_1305_6738_b200 as zk
    from paper_1305_6738_b200 import cli

    with open(os.path.join(HERE, "golden", "paper_tables.json")) as fh:
        paper = json.load(fh)["tables"][label]
    support = zk.Support.unbounded() if label == "inf" else zk.Support.finite(int(label))
    gammas = cli.REFERENCE_GAMMAS_UNBOUNDED if label == "inf" else cli.REFERENCE_GAMMAS_FINITE
    ours = _grid(zk, support, gammas, seed=20240001)
    z_all, worst = [], []
    for (g, n), (cut, sig) in ours.items():
        pub = paper[f"{g},{n}"]
        atom = n <= 50 and g >= 2.5
        for i in range(4):
            z = (cut[i] - pub[i]) / math.sqrt(2.0 * sig[i] ** 2 + SIGMA_ROUND ** 2)
            z_all.append(abs(z))
            if not atom:
                worst.append((abs(z), g, n, i, cut[i], pub[i]))
    z_all = np.asarray(z_all)
    assert len(z_all) == 4 * len(gammas) * len(NS)
    assert np.mean(z_all <= 3.0) >= 0.95, np.mean(z_all <= 3.0)
    assert np.mean(z_all <= 2.0) >= 0.88, np.mean(z_all <= 2.0)
    worst.sort(reverse=True)
    assert worst[0][0] <= 6.0, worst[:3]
