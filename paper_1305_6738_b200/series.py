"""Host-side tables shared with the device (reference ``series.py``).

Only the ln-k table lives here: it is built with numpy exactly as the reference's
``natural_logs`` (pkg/src/zipfks/series.py:31-44) and uploaded once per engine, so the
device forms every term ``exp(-gamma * ln k)`` from the same ln k values the reference
uses.  All power sums (finite moments, the zeta series with its Euler-Maclaurin tail,
tail masses) run on the device (csrc/zks_series.cuh).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MAX_FINITE_SUPPORT = 32766   # series.py:20
SERIES_RTOL = 1e-12          # series.py:23

_cache = np.zeros(1)


@dataclass(frozen=True)
class LogTable:
    """Precomputed natural logarithms of 1..limit, indexable by integer value (series.py:47-52)."""

    logs: np.ndarray
    limit: int


def build_log_table(limit: int) -> LogTable:
    """Table of ln k for k = 1..limit; entry 0 is padding (series.py:55-65)."""
    if isinstance(limit, bool) or not isinstance(limit, (int, np.integer)):
        raise ValueError(f"log table limit must be an integer, got {limit!r}")
    if limit < 1 or limit > MAX_FINITE_SUPPORT:
        raise ValueError(f"log table limit must be in [1, {MAX_FINITE_SUPPORT}], got {limit}")
    return LogTable(logs=natural_logs(int(limit)), limit=int(limit))


def _series_rows(gammas, support) -> np.ndarray:
    """(s0, s1, s2, normaliser) per exponent from the device (zks_series_eval)."""
    import torch

    from .engine import get_engine

    eng = get_engine()
    g = torch.as_tensor(np.asarray(gammas, dtype=np.float64).ravel()).to(f"cuda:{eng.device}")
    return eng.series(None if support is None else support.k, g).cpu().numpy()


def finite_log_moments(gamma: float, k: int) -> tuple[float, float, float]:
    """(s0, s1, s2), s_p = sum_{j=1..k} j^-gamma (ln j)^p (series.py:68-73), on the device."""
    from .distribution import Support

    s0, s1, s2, _ = _series_rows([gamma], Support.finite(k))[0]
    return float(s0), float(s1), float(s2)


def zeta_log_moments(gamma: float) -> tuple[float, float, float]:
    """(s0, s1, s2) of the zeta series with its Euler-Maclaurin tail (series.py:102-123)."""
    if gamma <= 1.0:
        raise ValueError(f"series diverges for gamma <= 1, got {gamma}")
    s0, s1, s2, _ = _series_rows([gamma], None)[0]
    return float(s0), float(s1), float(s2)


def zeta_value(gamma: float) -> float:
    """sum_{k>=1} k^-gamma (series.py:126-138)."""
    if gamma <= 1.0:
        raise ValueError(f"series diverges for gamma <= 1, got {gamma}")
    return float(_series_rows([gamma], None)[0][3])


def natural_logs(limit: int) -> np.ndarray:
    """Read-only view ``a`` with ``a[k] = ln k`` for k = 1..limit and ``a[0] = 0``."""
    global _cache
    if _cache.size < limit + 1:
        size = 1024
        while size < limit + 1:
            size *= 2
        table = np.empty(size, dtype=np.float64)
        table[0] = 0.0
        table[1:] = np.log(np.arange(1, size, dtype=np.float64))
        table.flags.writeable = False
        _cache = table
    return _cache[: limit + 1]


_TAIL_MIN_START = 64  # series.py:26


def tail_mass(gamma: float, start):
    """sum_{k >= start} k^-gamma, vectorised over ``start`` (each >= 65), on the device:
    Euler-Maclaurin through the third-derivative term (series.py:141-160)."""
    import torch

    from .engine import get_engine

    a = np.asarray(start, dtype=np.float64)
    if np.any(a < _TAIL_MIN_START + 1):
        raise ValueError("tail_mass requires start > 64; sum small ranges directly")
    eng = get_engine()
    out = eng.tail_mass(gamma, torch.from_numpy(np.ascontiguousarray(a.ravel())).to(f"cuda:{eng.device}"))
    value = out.cpu().numpy().reshape(a.shape)
    return float(value) if np.ndim(start) == 0 else value
