"""Host-side tables shared with the device (reference ``series.py``).

Only the ln-k table lives here: it is built with numpy exactly as the reference's
``natural_logs`` (pkg/src/zipfks/series.py:31-44) and uploaded once per engine, so the
device forms every term ``exp(-gamma * ln k)`` from the same ln k values the reference
uses.  All power sums (finite moments, the zeta series with its Euler-Maclaurin tail,
tail masses) run on the device (csrc/zks_series.cuh).
"""
from __future__ import annotations

import numpy as np

MAX_FINITE_SUPPORT = 32766   # series.py:20
SERIES_RTOL = 1e-12          # series.py:23

_cache = np.zeros(1)


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
