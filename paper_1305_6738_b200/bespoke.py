"""``fit`` on the device: fit a user sample, then calibrate the KS cutoffs for
exactly its (gamma_hat, n, support) by Monte Carlo (``--bespoke``) or look them up in a table file
(``--table``), and judge the fit; plus the command's observation files and reports.

Mirrors the bespoke branch of cli._cmd_fit (pkg/src/zipfks/cli.py:197-262) without the CLI:
mle_gamma -> ZipfModel(gamma_hat) -> ks_statistic -> SimulationConfig(n, gamma_hat) ->
run_simulation -> judge per level.  The reference spends minutes of CPU on the default
50,000 x 10 calibration; here it is one queued batch of replicate kernels.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

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


# ---------------------------------------------------------------------------
# the `fit` command's host side: observation files and reports (observations.py, reporting.py)

class ObservationParseError(ValueError):
    """An observation file that is not whitespace-separated positive integers (observations.py:11-12);
    the message names the line and token."""


def parse_observations(path) -> Sample:
    """Every integer of a UTF-8 file in file order (observations.py:15-34)."""
    values: list[int] = []
    with open(path, "r", encoding="utf-8") as fh:
        for line_no, line in enumerate(fh, start=1):
            for token_no, token in enumerate(line.split(), start=1):
                if not token.isdigit() or int(token) < 1:
                    raise ObservationParseError(
                        f"{path}: line {line_no}, token {token_no}: {token!r} is not a positive integer")
                values.append(int(token))
    if not values:
        raise ObservationParseError(f"{path}: no observations found")
    return Sample(np.asarray(values, dtype=np.int64))


def write_observations(sample: Sample, path) -> None:
    """One observation per line, readable by parse_observations (observations.py:37-42)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(f"{int(v)}\n" for v in sample.observations)


def format_human(report: FitReport) -> str:
    """The human-readable report (reporting.py:27-40)."""
    support = "unbounded" if report.support.k is None else f"1..{report.support.k}"
    out = [f"observations:  {report.n}", f"support:       {support}", f"gamma_hat:     {report.gamma_hat:.4f}",
           f"ks_statistic:  {report.ks:.4f} (attained at k={report.ks_argmax})",
           f"cutoffs from:  {report.cutoff_source}"]
    out += [f"  level {v.level:<5}  cutoff {v.cutoff:.4f}  {'REJECTED' if v.rejected else 'not rejected'}"
            for v in report.verdicts]
    return "\n".join(out)


def _level_tag(level: float) -> str:
    """0.9 -> '90', 0.95 -> '95', 0.999 -> '999' (reporting.py:43-46)."""
    digits = repr(float(level)).replace("0.", "", 1)
    return digits + "0" if len(digits) == 1 else digits


def format_machine(report: FitReport) -> str:
    """key=value lines at full precision (reporting.py:49-62)."""
    out = [f"n={report.n}", f"k_support={report.support}", f"gamma_hat={report.gamma_hat!r}", f"ks={report.ks!r}",
           f"ks_argmax={report.ks_argmax}", f"cutoff_source={report.cutoff_source}"]
    for v in report.verdicts:
        tag = _level_tag(v.level)
        out += [f"cutoff_q{tag}={v.cutoff!r}", f"rejected_q{tag}={str(v.rejected).lower()}"]
    return "\n".join(out)
