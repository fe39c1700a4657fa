"""``fit --bespoke`` on the device: fit a user sample, then calibrate the KS
cutoffs for exactly its (gamma_hat, n, support) by Monte Carlo and judge the fit.

Mirrors the bespoke branch of cli._cmd_fit (pkg/src/zipfks/cli.py:197-262) without the CLI:
mle_gamma -> ZipfModel(gamma_hat) -> ks_statistic -> SimulationConfig(n, gamma_hat) ->
run_simulation -> judge per level.  The reference spends minutes of CPU on the default
50,000 x 10 calibration; here it is one queued batch of replicate kernels.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

from .distribution import Sample, Support, ZipfModel
from .estimate import mle_gamma
from .gof import Verdict, judge, ks_statistic
from .montecarlo import DEFAULT_LEVELS, SimulationConfig, run_simulation


@dataclass(frozen=True)
class FitReport:
    """Result of testing one dataset against the Zipf family (reporting.py:10-24)."""

    n: int
    support: Support
    gamma_hat: float
    ks: float
    ks_argmax: int
    cutoff_source: str
    verdicts: tuple[Verdict, ...]

    def rejected_at(self, level: float) -> bool:
        for verdict in self.verdicts:
            if verdict.level == level:
                return verdict.rejected
        raise ValueError(f"no verdict at level {level}")


def fit_bespoke(sample: Sample, support: Support, base_seed: int, replicates: int = 50000, repetitions: int = 10,
                quantiles: Sequence[float] = DEFAULT_LEVELS) -> FitReport:
    """Fit, score and judge ``sample`` with bespoke simulated cutoffs (NoRootError propagates)."""
    if not isinstance(sample, Sample):
        sample = Sample(sample)
    if not support.contains(sample.observations):
        raise ValueError(f"observations exceed the declared support 1..{support}")
    gamma_hat = mle_gamma(sample, support)
    ks = ks_statistic(sample, ZipfModel(gamma=gamma_hat, support=support))
    config = SimulationConfig(n=sample.n, support=support, gamma=gamma_hat, base_seed=base_seed,
                              replicates=replicates, repetitions=repetitions, quantiles=tuple(quantiles))
    pairs = run_simulation(config)
    verdicts = tuple(judge(ks.statistic, cutoff, level) for level, cutoff in pairs)
    source = f"bespoke simulation (replicates={replicates}, repetitions={repetitions}, seed={base_seed})"
    return FitReport(n=sample.n, support=support, gamma_hat=gamma_hat, ks=ks.statistic, ks_argmax=ks.argmax_k,
                     cutoff_source=source, verdicts=verdicts)
