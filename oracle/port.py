"""TEST INFRASTRUCTURE ONLY — CPU restatement (numpy) of the reference hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this module; the
product package never does.  It is the parity checker for the CUDA engine and
the CPU baseline it is timed against.

It restates, function by function, the reference ``zipfks`` 1.0.0 algorithm
(``/root/reference/pkg/src/zipfks``) with the same numpy primitives in the same
order, so that on identical inputs it reproduces the reference bit-for-bit
(checked against golden vectors produced by the reference itself, see
``tests/golden/make_golden.py`` and ``tests/test_oracle_port.py``):

=====================  ==============================================
this module            reference
=====================  ==============================================
``log_table``          ``series.py:31-44`` (natural_logs)
``finite_moments``     ``series.py:68-73`` (finite_log_moments)
``em_tail``            ``series.py:76-99`` (_tail_log_moment)
``zeta_moments``       ``series.py:102-123`` (zeta_log_moments)
``zeta_norm``          ``series.py:126-138`` (zeta_value)
``tail_sum``           ``series.py:141-160`` (tail_mass)
``norm_constant``      ``distribution.py:71-85`` (normalization)
``sampling_cdf``       ``distribution.py:99-105`` (ZipfModel._sampling_cdf)
``draw``               ``distribution.py:190-201`` (sample)
``mean_log``           ``estimate.py:59-73`` (log_mean)
``fit_exponent``       ``estimate.py:76-146`` (mle_gamma, _bisect, ...)
``ks_distance``        ``gof.py:49-105`` (ks_statistic, dense/sparse)
``replicate``          ``montecarlo.py:89-116`` (_attempt, run_replicate)
``repetition``         ``montecarlo.py:151-191`` (run_repetition, pool)
``quantile_ranks``     ``montecarlo.py:119-136`` (order_quantiles)
``simulate``           ``montecarlo.py:194-212`` (run_simulation)
=====================  ==============================================

A support is ``None`` (unbounded, draws from 1..65535) or an int ``K``.
"""
from __future__ import annotations

import math
import multiprocessing
import os
from decimal import ROUND_FLOOR, Decimal

import numpy as np

from . import rng as _rng

LIMIT_UNBOUNDED = 65535          # distribution.py:26
SEAM = 4096                      # distribution.py:30 (_PARTIAL_SEAM) == gof.py:20
RTOL = 1e-12                     # series.py:23
MIN_GAMMA_UNBOUNDED = 1.05       # distribution.py:19
MAX_GAMMA_UNBOUNDED = 20.0       # estimate.py:21
BRACKET = (-20.0, 20.0)          # estimate.py:38
START = 0.5                      # estimate.py:35
TOL = 1e-5                       # estimate.py:36
MAX_ITER = 200                   # estimate.py:37
RETRY_OFFSET = 1 << 32           # montecarlo.py:29
SPAN = 512                       # montecarlo.py:32
LEVELS = (0.9, 0.95, 0.99, 0.999)  # montecarlo.py:26
_LN2 = math.log(2.0)


class NoRoot(ValueError):
    """estimate.py:55 NoRootError."""


class FailedTwice(RuntimeError):
    """montecarlo.py:35 SimulationError (replicate failed twice)."""


# ----------------------------------------------------------------------------
# series (L0)

_LOGS = np.concatenate(([0.0], np.log(np.arange(1, 1 << 16, dtype=np.float64))))


def log_table(limit: int) -> np.ndarray:
    """``a[k] = ln k`` for k = 1..limit, ``a[0] = 0`` (series.py:31-44)."""
    global _LOGS
    if limit + 1 > _LOGS.size:
        size = 1024
        while size < limit + 1:
            size *= 2
        _LOGS = np.concatenate(([0.0], np.log(np.arange(1, size, dtype=np.float64))))
    return _LOGS[: limit + 1]


def finite_moments(gamma: float, k: int) -> tuple[float, float, float]:
    lk = log_table(k)[1:]
    w = np.exp(-gamma * lk)
    wl = w * lk
    return float(w.sum()), float(wl.sum()), float(wl @ lk)


def em_tail(gamma: float, start: int, p: int) -> tuple[float, float]:
    """Euler-Maclaurin tail of sum k^-g (ln k)^p from ``start`` and its bound."""
    a = float(start)
    L = math.log(a)
    g1 = gamma - 1.0
    head = math.exp(-g1 * L)
    if p == 0:
        integral = head / g1
    elif p == 1:
        integral = head * (L / g1 + 1.0 / g1**2)
    else:
        integral = head * (L * L / g1 + 2.0 * L / g1**2 + 2.0 / g1**3)
    lp = L**p
    f = math.exp(-gamma * L) * lp
    df = math.exp(-(gamma + 1.0) * L) * ((p * L ** (p - 1) if p else 0.0) - gamma * lp)
    bound = (gamma + p + 3.0) ** 3 * math.exp(-(gamma + 3.0) * L) * lp
    return integral + 0.5 * f - df / 12.0, bound / 720.0


def zeta_moments(gamma: float) -> tuple[float, float, float]:
    if gamma <= 1.0:
        raise ValueError(f"series diverges for gamma <= 1, got {gamma}")
    m = 256
    while True:
        s = list(finite_moments(gamma, m))
        ok = True
        for p in range(3):
            t, e = em_tail(gamma, m + 1, p)
            s[p] += t
            ok = ok and e <= RTOL * s[p]
        if ok:
            return s[0], s[1], s[2]
        m *= 2
        if m > 1 << 22:
            raise RuntimeError(f"tail bound not converging at gamma={gamma}")


def zeta_norm(gamma: float) -> float:
    if gamma <= 1.0:
        raise ValueError(f"series diverges for gamma <= 1, got {gamma}")
    m = 256
    while True:
        s0 = float(np.exp(-gamma * log_table(m)[1:]).sum())
        t0, e0 = em_tail(gamma, m + 1, 0)
        s0 += t0
        if e0 <= RTOL * s0:
            return s0
        m *= 2


def tail_sum(gamma: float, start):
    a = np.asarray(start, dtype=np.float64)
    if np.any(a < 65):
        raise ValueError("tail_sum requires start > 64")
    L = np.log(a)
    g1 = gamma - 1.0
    v = (
        np.exp(-g1 * L) / g1
        + 0.5 * np.exp(-gamma * L)
        + (gamma / 12.0) * np.exp(-(gamma + 1.0) * L)
        - (gamma * (gamma + 1.0) * (gamma + 2.0) / 720.0) * np.exp(-(gamma + 3.0) * L)
    )
    return float(v) if np.ndim(start) == 0 else v


# ----------------------------------------------------------------------------
# distribution (L1)

def norm_constant(gamma: float, support: int | None) -> float:
    if not math.isfinite(gamma):
        raise ValueError(f"exponent must be finite, got {gamma}")
    if support is not None:
        total = float(np.exp(-gamma * log_table(support)[1:]).sum())
        if not math.isfinite(total):
            raise ValueError(f"normalizer overflows at gamma={gamma} with K={support}")
        return total
    if gamma < MIN_GAMMA_UNBOUNDED:
        raise ValueError(f"unbounded support requires gamma >= {MIN_GAMMA_UNBOUNDED}, got {gamma}")
    return zeta_norm(gamma)


def draw_limit(support: int | None) -> int:
    return LIMIT_UNBOUNDED if support is None else support


def sampling_cdf(gamma: float, support: int | None) -> np.ndarray:
    w = np.exp(-gamma * log_table(draw_limit(support))[1:])
    return np.cumsum(w * (1.0 / w.sum()))


def draw(cdf: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Inverse transform: smallest k with cdf[k-1] >= u, clamped to the table."""
    return np.minimum(np.searchsorted(cdf, u, side="left") + 1, cdf.size).astype(np.int64)


def stream_uniforms(seed: int, repetition: int, index: int, count: int, restated: bool) -> np.ndarray:
    if restated:
        return _rng.uniforms(seed, repetition, index, count)
    return _rng.numpy_uniforms(seed, repetition, index, count)


# ----------------------------------------------------------------------------
# estimate (L2)

def mean_log(obs: np.ndarray) -> float:
    top = int(obs.max())
    if top <= 1 << 20:
        raw = float(log_table(top)[obs].sum())
    else:
        raw = float(np.log(obs.astype(np.float64)).sum())
    if raw <= 0.0:
        raw += _LN2
    return raw / obs.size


def model_mean_var(gamma: float, support: int | None) -> tuple[float, float]:
    s0, s1, s2 = finite_moments(gamma, support) if support is not None else zeta_moments(gamma)
    mu = s1 / s0
    return mu, s2 / s0 - mu * mu


def search_range(support: int | None) -> tuple[float, float]:
    lo, hi = BRACKET
    if support is None:
        lo, hi = max(lo, MIN_GAMMA_UNBOUNDED), min(hi, MAX_GAMMA_UNBOUNDED)
    return lo, hi


def bisect_root(target: float, support: int | None, lo: float, hi: float) -> float:
    f_lo = target - model_mean_var(lo, support)[0]
    f_hi = target - model_mean_var(hi, support)[0]
    if f_lo == 0.0:
        return lo
    if f_hi == 0.0:
        return hi
    if f_lo * f_hi > 0.0:
        raise NoRoot(
            f"estimating equation has no root in [{lo}, {hi}] (mean log of data: {target:.6g})"
        )
    while hi - lo > 1e-8:
        mid = 0.5 * (lo + hi)
        if (target - model_mean_var(mid, support)[0]) * f_lo <= 0.0:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


def fit_target(obs: np.ndarray, support: int | None) -> float:
    target = mean_log(obs)
    if support is not None and int(obs.min()) == support:
        target -= (math.log(support) - math.log(support - 1)) / obs.size
    return target


def fit_exponent(obs: np.ndarray, support: int | None) -> float:
    if int(obs.min()) < 1 or (support is not None and int(obs.max()) > support):
        raise ValueError(f"observations exceed the declared support 1..{support}")
    target = fit_target(obs, support)
    lo, hi = search_range(support)
    x = START if lo < START < hi else lo + 0.01
    for _ in range(MAX_ITER):
        mu, var = model_mean_var(x, support)
        x_next = x + (mu - target) / var
        if not math.isfinite(x_next) or x_next < lo or x_next > hi:
            return bisect_root(target, support, lo, hi)
        if abs(x_next - x) <= TOL:
            return x_next
        x = x_next
    return bisect_root(target, support, lo, hi)


# ----------------------------------------------------------------------------
# goodness of fit (L2)

def _fitted_prefix(gamma: float, norm: float, upto: int) -> np.ndarray:
    return np.cumsum(np.exp(-gamma * log_table(upto)[1:]) * (1.0 / norm))


def ks_distance(obs: np.ndarray, gamma: float, support: int | None, norm: float | None = None) -> float:
    """Largest |fitted cdf - empirical cdf| over 1..max(obs) (gof.py:49-105)."""
    if norm is None:
        norm = norm_constant(gamma, support)
    n = obs.size
    kmax = int(obs.max())
    if support is not None or kmax <= SEAM:
        counts = np.bincount(obs, minlength=kmax + 1)[1:]
        emp = np.cumsum(counts / n)
        return float(np.abs(_fitted_prefix(gamma, norm, kmax) - emp).max())
    values, counts = np.unique(obs, return_counts=True)
    emp = np.cumsum(counts / n)
    left = np.concatenate(([0.0], emp[:-1]))
    table = _fitted_prefix(gamma, norm, SEAM)

    def fitted_at(points: np.ndarray) -> np.ndarray:
        points = np.maximum(points, 1)
        out = np.empty(points.shape)
        small = points <= SEAM
        out[small] = table[points[small] - 1]
        big = points[~small]
        if big.size:
            out[~small] = (norm - tail_sum(gamma, big + 1)) / norm
        return out

    at_values = np.abs(fitted_at(values) - emp)
    before = np.where(values > 1, np.abs(fitted_at(np.maximum(values - 1, 1)) - left), 0.0)
    return float(max(at_values.max(), before.max()))


# ----------------------------------------------------------------------------
# Monte Carlo driver (L3)

_CDF_CACHE: dict[tuple[float, int | None], np.ndarray] = {}


def cdf_for(gamma: float, support: int | None) -> np.ndarray:
    key = (gamma, support)
    if key not in _CDF_CACHE:
        if len(_CDF_CACHE) > 16:
            _CDF_CACHE.clear()
        norm_constant(gamma, support)
        _CDF_CACHE[key] = sampling_cdf(gamma, support)
    return _CDF_CACHE[key]


def attempt(gamma, support, n, seed, repetition, stream_index, restated=False):
    """One sample -> fit -> KS pass; returns (ks, gamma_hat, sample)."""
    u = stream_uniforms(seed, repetition, stream_index, n, restated)
    obs = draw(cdf_for(gamma, support), u)
    g = fit_exponent(obs, support)
    return ks_distance(obs, g, support), g, obs


def replicate(gamma, support, n, seed, index, repetition=0, restated=False):
    """(ks, gamma_hat, status) with status 0 ok / 1 retried (montecarlo.py:98-116)."""
    try:
        ks, g, _ = attempt(gamma, support, n, seed, repetition, index, restated)
        return ks, g, 0
    except NoRoot:
        try:
            ks, g, _ = attempt(gamma, support, n, seed, repetition, index + RETRY_OFFSET, restated)
            return ks, g, 1
        except NoRoot as err:
            raise FailedTwice(
                f"replicate {index} (repetition {repetition}, gamma={gamma}, n={n}, "
                f"support={'inf' if support is None else support}) failed twice: {err}"
            ) from err


def replicate_range(gamma, support, n, seed, repetition, start, stop, restated=False):
    ks = np.empty(stop - start)
    gh = np.empty(stop - start)
    st = np.empty(stop - start, dtype=np.uint8)
    for i in range(start, stop):
        ks[i - start], gh[i - start], st[i - start] = replicate(
            gamma, support, n, seed, i, repetition, restated
        )
    return ks, gh, st


_WORKER_CELL = None


def _worker_init(cell):
    global _WORKER_CELL
    _WORKER_CELL = cell
    cdf_for(cell[0], cell[1])


def _worker_span(task):
    repetition, start, stop = task
    gamma, support, n, seed = _WORKER_CELL
    ks, gh, _ = replicate_range(gamma, support, n, seed, repetition, start, stop)
    return start, ks, gh


def repetition(gamma, support, n, seed, replicates, rep, pool=None):
    """All replicate outcomes of one repetition, index order (montecarlo.py:174-191)."""
    ks = np.empty(replicates)
    gh = np.empty(replicates)
    if pool is None:
        ks[:], gh[:], _ = replicate_range(gamma, support, n, seed, rep, 0, replicates)
        return ks, gh
    tasks = [(rep, s, min(s + SPAN, replicates)) for s in range(0, replicates, SPAN)]
    for start, k, g in pool.imap_unordered(_worker_span, tasks):
        ks[start : start + k.size] = k
        gh[start : start + g.size] = g
    return ks, gh


def quantile_ranks(count: int, levels) -> list[int]:
    """Zero-based ranks floor(Decimal(str(q)) * count) (montecarlo.py:133)."""
    out = []
    for q in levels:
        r = int((Decimal(str(float(q))) * count).to_integral_value(rounding=ROUND_FLOOR))
        if r >= count:
            raise ValueError(f"rank {r} out of range for {count} values")
        out.append(r)
    return out


def order_quantiles(stats, levels) -> list[float]:
    arr = np.sort(np.asarray(stats, dtype=np.float64))
    if arr.size == 0:
        raise ValueError("cannot take quantiles of an empty array")
    return [float(arr[r]) for r in quantile_ranks(arr.size, levels)]


def simulate(gamma, support, n, seed, replicates, repetitions=1, levels=LEVELS, workers=1):
    """(level, cutoff) pairs averaged over repetitions (montecarlo.py:194-212)."""
    acc = np.zeros(len(levels))
    if workers == 1:
        for rep in range(repetitions):
            ks, _ = repetition(gamma, support, n, seed, replicates, rep)
            acc += np.asarray(order_quantiles(ks, levels))
    else:
        ctx = multiprocessing.get_context()
        with ctx.Pool(workers, initializer=_worker_init, initargs=((gamma, support, n, seed),)) as pool:
            for rep in range(repetitions):
                ks, _ = repetition(gamma, support, n, seed, replicates, rep, pool)
                acc += np.asarray(order_quantiles(ks, levels))
    acc /= repetitions
    return list(zip(levels, (float(c) for c in acc)))


def host_workers() -> int:
    return os.cpu_count() or 1
