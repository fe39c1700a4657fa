"""Exponent-estimator settings and errors (reference ``estimate.py``).

The Newton / bisection solve itself runs on the device inside the replicate kernel
(csrc/zks_replicate.cuh: fit_exponent, bisect_root), always with DEFAULT_SETTINGS as the
reference's Monte Carlo does (montecarlo.py:93).
"""
from __future__ import annotations

from dataclasses import dataclass

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
