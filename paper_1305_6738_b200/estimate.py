"""Maximum-likelihood estimation of the Zipf exponent (reference ``estimate.py``), on the device.

The Newton / bisection solve runs in ``libzks_b200.so``: inside the replicate kernels for the
Monte Carlo (always with DEFAULT_SETTINGS, as the reference does, montecarlo.py:93) and in
``zks_fit_samples`` / ``zks_solve_exponents`` for user samples (the calls below).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .distribution import MIN_UNBOUNDED_GAMMA, Sample, Support

MAX_UNBOUNDED_GAMMA = 20.0  # estimate.py:21


@dataclass(frozen=True)
class MleSettings:
    """Newton-Raphson controls (estimate.py:24-47)."""

    initial_guess: float = 0.5
    absolute_tolerance: float = 1e-5
    max_iterations: int = 200
    bracket: tuple[float, float] = (-20.0, 20.0)

    def __post_init__(self) -> None:
        if self.absolute_tolerance <= 0:
            raise ValueError("absolute_tolerance must be positive")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        low, high = self.bracket
        if not low < self.initial_guess < high:
            raise ValueError("bracket must satisfy low < initial_guess < high")


DEFAULT_SETTINGS = MleSettings()


class NoRootError(ValueError):
    """The estimating equation has no root inside the admissible range (estimate.py:55)."""


def _search_range(support: Support, settings: MleSettings = DEFAULT_SETTINGS) -> tuple[float, float]:
    low, high = settings.bracket
    if not support.is_finite:
        low, high = max(low, MIN_UNBOUNDED_GAMMA), min(high, MAX_UNBOUNDED_GAMMA)
    return low, high


def _no_root(target: float, low: float, high: float) -> NoRootError:
    return NoRootError(f"estimating equation has no root in [{low}, {high}] (mean log of data: {target:.6g})")


def _fit_one(sample: Sample, support: Support | None, mode: int, settings=None, gamma=None, norm=None) -> dict:
    from .gof import fit_samples_device

    return fit_samples_device([sample.observations], support, mode, settings, gamma, norm, single=True)


def log_mean(sample: Sample) -> float:
    """(sum ln x_i) / n with the all-ones nudge (estimate.py:59-73), on the device."""
    r = _fit_one(sample, Support.unbounded(), 0)
    return float(r["log_mean"][0])


def _mean_log_and_slope(gamma: float, support: Support) -> tuple[float, float]:
    """Model mean of ln X and its variance (estimate.py:76-83), by the reference's sums."""
    from .series import _series_rows

    s0, s1, s2, _ = _series_rows([gamma], support)[0]
    if not math.isfinite(s0):
        raise ValueError(f"series diverges for gamma <= 1, got {gamma}")
    mean = s1 / s0
    return mean, s2 / s0 - mean * mean


def _solve(targets, support: Support, settings: MleSettings, bisect_only: bool, low=None, high=None):
    import torch

    from .engine import get_engine

    eng = get_engine()
    t = torch.as_tensor(np.asarray(targets, dtype=np.float64)).to(f"cuda:{eng.device}")
    s = settings
    if bisect_only:
        s = MleSettings(initial_guess=0.5 * (low + high), absolute_tolerance=1e-5, max_iterations=1,
                        bracket=(low, high))
    g, st = eng.solve(support.k, t, s, bisect_only)
    return g.cpu().numpy(), st.cpu().numpy()


def _bisect(target: float, support: Support, low: float, high: float) -> float:
    """Bisection on [low, high] (estimate.py:94-112)."""
    g, st = _solve([target], support, DEFAULT_SETTINGS, True, low, high)
    if st[0] == _native.SAMPLE_NOROOT:
        raise _no_root(target, low, high)
    return float(g[0])


def mle_gamma(sample: Sample, support: Support, settings: MleSettings = DEFAULT_SETTINGS) -> float:
    """Exponent estimate for the sample over the declared support (estimate.py:115-146)."""
    if not support.contains(sample.observations):
        raise ValueError(f"observations exceed the declared support 1..{support}")
    r = _fit_one(sample, support, _native.FIT_EXPONENT, None if settings == DEFAULT_SETTINGS else settings)
    status = int(r["status"][0])
    if status == _native.SAMPLE_NOROOT:
        low, high = _search_range(support, settings)
        target = float(r["log_mean"][0])
        obs = sample.observations
        if support.is_finite and int(obs.min()) == support.k:
            target -= (math.log(support.k) - math.log(support.k - 1)) / sample.n
        raise _no_root(target, low, high)
    if status != _native.SAMPLE_OK:
        raise ValueError(f"observations exceed the declared support 1..{support}")
    return float(r["gamma"][0])
