"""Calibration engine on the GPU: replicates, order-statistic quantiles, cutoff tables.

Drop-in for the reference ``zipfks.montecarlo`` (pkg/src/zipfks/montecarlo.py): same names,
argument meaning, return types and error behaviour.  The per-replicate pipeline
(sample -> re-fit -> KS against the re-fit, one retry on stream ``idx + 2**32``) and the
quantile selection run in ``libzks_b200.so``; this module keeps the host-side contract:
config validation, the Decimal rank rule, repetition averaging in repetition order, the
error messages.  Streams are keyed ``(base_seed, repetition, index)``, so results do not
depend on how replicates are batched or sharded over GPUs.
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from decimal import ROUND_FLOOR, Decimal
from typing import Callable, Iterable, Sequence

import numpy as np

from . import _native
from .distribution import Support, sampling_cdf, validate_pair
from .estimate import MAX_UNBOUNDED_GAMMA

DEFAULT_LEVELS = (0.9, 0.95, 0.99, 0.999)  # montecarlo.py:26
_RETRY_OFFSET = 1 << 32                    # montecarlo.py:29


class SimulationError(RuntimeError):
    """A replicate failed twice, or a table cell could not be computed (montecarlo.py:35)."""


def _validate_levels(levels: Sequence[float]) -> tuple[float, ...]:
    out = tuple(float(q) for q in levels)
    if not out:
        raise ValueError("at least one quantile level is required")
    if any(not 0.0 < q < 1.0 for q in out):
        raise ValueError(f"quantile levels must lie in (0, 1), got {out}")
    if any(b <= a for a, b in zip(out, out[1:])):
        raise ValueError(f"quantile levels must be strictly increasing, got {out}")
    return out


@dataclass(frozen=True)
class SimulationConfig:
    """One calibration experiment: R replicates repeated and averaged (montecarlo.py:50-72)."""

    n: int
    support: Support
    gamma: float
    base_seed: int
    replicates: int = 50000
    repetitions: int = 10
    quantiles: tuple[float, ...] = DEFAULT_LEVELS

    def __post_init__(self) -> None:
        if self.n < 1:
            raise ValueError(f"sample size must be >= 1, got {self.n}")
        if self.replicates < 100:
            raise ValueError(f"need at least 100 replicates, got {self.replicates}")
        if self.repetitions < 1:
            raise ValueError(f"need at least one repetition, got {self.repetitions}")
        if not 0 <= int(self.base_seed) < 1 << 64:
            raise ValueError("base_seed must fit an unsigned 64-bit integer")
        object.__setattr__(self, "quantiles", _validate_levels(self.quantiles))
        validate_pair(self.gamma, self.support)


@dataclass(frozen=True)
class ReplicateOutcome:
    ks: float
    gamma_hat: float
    replicate_index: int


def quantile_ranks(count: int, levels: Sequence[float]) -> list[int]:
    """Zero-based ranks floor(Decimal(str(q)) * count) (montecarlo.py:133-135)."""
    ranks = []
    for level in _validate_levels(levels):
        rank = int((Decimal(str(level)) * count).to_integral_value(rounding=ROUND_FLOOR))
        if rank >= count:
            raise ValueError(f"rank {rank} out of range for {count} values")
        ranks.append(rank)
    return ranks


def resolve_workers(workers: int | None) -> int:
    """Validated worker count (montecarlo.py:162-167).  Accepted for API compatibility: the
    device does the parallel work, so results and speed do not depend on it."""
    if workers is None:
        return os.cpu_count() or 1
    if workers < 1:
        raise ValueError(f"worker count must be >= 1, got {workers}")
    return workers


# ---------------------------------------------------------------------------
# device plumbing

def _torch():
    import torch

    return torch


def _engine():
    from .engine import get_engine

    return get_engine()


_PENDING: dict = {}  # (device, gamma, K) -> future of a host sampling CDF being built (_prefetch_tables)
_POOL = None


def _table(eng, config: SimulationConfig):
    fut = _PENDING.pop((eng.device, float(config.gamma), config.support.k), None)
    if fut is not None:
        cdf = fut.result()
        return eng.table(config.gamma, config.support.k, lambda: cdf)
    return eng.table(config.gamma, config.support.k, lambda: sampling_cdf(config.gamma, config.support))


class _Slab:
    """Reusable device outputs (ks, gamma_hat, status) for up to ``cap`` replicates."""

    def __init__(self, eng, cap: int):
        torch = _torch()
        dev = f"cuda:{eng.device}"
        self.cap = cap
        self.ks = torch.empty(cap, dtype=torch.float64, device=dev)
        self.gh = torch.empty(cap, dtype=torch.float64, device=dev)
        self.st = torch.empty(cap, dtype=torch.uint8, device=dev)


_SLABS: dict[int, _Slab] = {}


def _slab(eng, count: int) -> _Slab:
    s = _SLABS.get(eng.device)
    if s is None or s.cap < count:
        s = _Slab(eng, max(count, 1024))
        _SLABS[eng.device] = s
    return s


def _failure(config: SimulationConfig, repetition: int, index: int, mean_log: float) -> SimulationError:
    low, high = (-20.0, 20.0) if config.support.is_finite else (1.05, MAX_UNBOUNDED_GAMMA)
    reason = f"estimating equation has no root in [{low}, {high}] (mean log of data: {mean_log:.6g})"
    return SimulationError(
        f"replicate {index} (repetition {repetition}, gamma={config.gamma}, "
        f"n={config.n}, support={config.support}) failed twice: {reason}"
    )


def _raise_first_failure(config, repetition, first, status: np.ndarray, gamma_hat: np.ndarray) -> None:
    bad = np.flatnonzero(status == _native.STATUS_FAILED)
    if bad.size:
        i = int(bad[0])
        raise _failure(config, repetition, first + i, float(gamma_hat[i]))


def _enqueue(eng, config: SimulationConfig, repetition: int, first: int, count: int, slab: _Slab, offset: int = 0):
    """Enqueue replicates [first, first+count) into slab[offset : offset+count]."""
    table = _table(eng, config)
    eng.run_replicates(
        table, config.support.k, config.gamma, config.n, config.base_seed, repetition, first, count,
        slab.ks[offset:], slab.gh[offset:], slab.st[offset:],
    )


def set_rng(kind: str = "numpy") -> None:
    """Choose the replicate streams of later simulations on this process's device.

    ``"numpy"`` (the default) draws every replicate from RandomStream.for_replicate
    (distribution.py:173-187) bit for bit, so every statistic matches the reference replicate by
    replicate.  ``"philox4x32"`` is an opt-in faster generator (Philox4x32-10 keyed by the same
    SeedSequence key, about a quarter of the integer work per draw): the samples differ, their
    law does not, so cutoffs agree with the default within Monte Carlo error only (tier 3).
    """
    _engine().set_rng(kind)


# ---------------------------------------------------------------------------
# reference API

def run_replicate(config: SimulationConfig, index: int, repetition: int = 0) -> ReplicateOutcome:
    """Sample, re-fit, and score one replicate (montecarlo.py:98-116), on the device."""
    if not 0 <= index < config.replicates:
        raise ValueError(f"replicate index {index} outside [0, {config.replicates})")
    eng = _engine()
    slab = _slab(eng, 1)
    _enqueue(eng, config, repetition, index, 1, slab)
    ks, gh, st = slab.ks[:1].cpu().numpy(), slab.gh[:1].cpu().numpy(), slab.st[:1].cpu().numpy()
    _raise_first_failure(config, repetition, index, st, gh)
    return ReplicateOutcome(ks=float(ks[0]), gamma_hat=float(gh[0]), replicate_index=index)


def run_repetition(config: SimulationConfig, repetition: int, pool=None) -> tuple[np.ndarray, np.ndarray]:
    """All replicate outcomes of one repetition in replicate-index order (montecarlo.py:174-191).

    ``pool`` is accepted for signature compatibility and ignored: the device is the pool.
    """
    eng = _engine()
    total = config.replicates
    slab = _slab(eng, total)
    _enqueue(eng, config, repetition, 0, total, slab)
    ks = slab.ks[:total].cpu().numpy().copy()
    gh = slab.gh[:total].cpu().numpy().copy()
    st = slab.st[:total].cpu().numpy()
    _raise_first_failure(config, repetition, 0, st, gh)
    return ks, gh


def order_quantiles(stats, levels: Sequence[float]) -> list[float]:
    """Order statistics at zero-based ranks floor(R * level) (montecarlo.py:119-136).

    ``stats`` may be a sequence, a numpy array or a CUDA float64 tensor; the selection runs
    on the device: a radix select over order-preserving 64-bit keys of the values.  For
    non-negative values (KS statistics) the key is the IEEE bit pattern itself; any other input
    is selected on sign-flipped keys (negative values: all bits inverted; others: the sign bit
    set), with NaNs canonicalised to sort last, as ``np.sort`` orders them.
    """
    torch = _torch()
    on_device = isinstance(stats, torch.Tensor) and stats.is_cuda
    arr = None if on_device else np.ascontiguousarray(np.asarray(stats, dtype=np.float64))
    count = stats.numel() if on_device else arr.size
    # argument errors first, as the reference raises them (montecarlo.py:128-135)
    if count == 0:
        raise ValueError("cannot take quantiles of an empty array")
    ranks = quantile_ranks(count, levels)
    eng = _engine()
    if on_device:
        values = stats.to(torch.float64).contiguous().reshape(-1)
    else:
        values = torch.from_numpy(arr.reshape(-1)).to(f"cuda:{eng.device}")
    values = values + 0.0  # canonicalise -0.0 to +0.0 (np.sort treats them as equal)
    nan = torch.isnan(values)
    signed = bool((values < 0).any()) or bool(nan.any())
    if signed:
        bits = torch.where(nan, torch.full_like(values, float("nan")), values).view(torch.int64)
        sign = torch.tensor(-(1 << 63), dtype=torch.int64, device=values.device)
        keys = torch.where(bits < 0, ~bits, bits ^ sign).view(torch.float64)
    else:
        keys = values
    out = []
    for i in range(0, len(ranks), 16):
        chunk = torch.empty(len(ranks[i : i + 16]), dtype=torch.float64, device=values.device)
        eng.select_ranks(keys, ranks[i : i + 16], out=chunk)
        if signed:  # back from keys: a set top bit marks a non-negative value
            kb = chunk.view(torch.int64)
            chunk = torch.where(kb < 0, kb ^ sign, ~kb).view(torch.float64)
        out.extend(float(x) for x in chunk.cpu().tolist())
    return out


@dataclass
class _CellPlan:
    config: SimulationConfig
    quantiles: object = None   # device [reps, levels]
    worst: object = None       # device [reps] max status
    started: object = None
    finished: object = None
    host: object = None        # (quantiles, worst) copied to the host by _fetch_plans


def _keep(keep, cfg, rep, slab, first, stop) -> None:
    """Test hook: a stream-ordered copy of one (cell, repetition)'s per-replicate outputs."""
    if keep is not None:
        keep[(cfg.gamma, cfg.n, rep)] = tuple(t[first:stop].clone() for t in (slab.ks, slab.gh, slab.st))


def _enqueue_cell(eng, plan: _CellPlan, shard: tuple[int, int] | None = None, reduce=None,
                  kernel_events: list | None = None, keep: dict | None = None) -> None:
    """Queue every repetition of one cell: replicates -> selection, all async.

    ``shard`` = (first, stop) restricts this process to replicate indices [first, stop); the
    order statistics are then selected over every process's shard with ``reduce`` summing the
    selection's digit histograms over the processes (NCCL all-reduce, parallel.py).
    """
    torch = _torch()
    cfg = plan.config
    total = cfg.replicates
    first, stop = shard if shard is not None else (0, total)
    dev = f"cuda:{eng.device}"
    ranks = quantile_ranks(total, cfg.quantiles)
    plan.quantiles = torch.empty((cfg.repetitions, len(ranks)), dtype=torch.float64, device=dev)
    plan.worst = torch.zeros(cfg.repetitions, dtype=torch.uint8, device=dev)
    plan.started = torch.cuda.Event(enable_timing=True)
    plan.finished = torch.cuda.Event(enable_timing=True)
    slab = _slab(eng, total)
    stream = eng.bind_stream()
    plan.started.record(stream)
    for rep in range(cfg.repetitions):
        if stop > first:
            if kernel_events is not None:  # bench.py: time the replicate kernel itself
                k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                k0.record(stream)
            _enqueue(eng, cfg, rep, first, stop - first, slab, offset=first)
            if kernel_events is not None:
                k1.record(stream)
                kernel_events.append((k0, k1))
            _keep(keep, cfg, rep, slab, first, stop)
        # the selection launch also reduces the repetition's worst status (first rank chunk)
        jobs = [(slab.ks[first:stop], ranks[i : i + 16], plan.quantiles[rep, i : i + 16])
                + ((slab.st[first:stop], plan.worst[rep : rep + 1]) if i == 0 else ())
                for i in range(0, len(ranks), 16)]
        for job in jobs:  # rank chunks differ in length: one launch each
            if reduce is None:
                eng.select_many([job])
            else:
                eng.select_dist([job], total, reduce)
    plan.finished.record(stream)


def _stage_key(cfg: SimulationConfig):
    return (cfg.support.k, cfg.n, cfg.base_seed, cfg.replicates, cfg.repetitions, cfg.quantiles)


_ROW_CELLS = 32   # cells per zks_run_cells call
_EARLY_CELLS = 6  # cells of a sweep's first row launched ahead of the other tables


def _enqueue_group(eng, plans: list[_CellPlan], shard=None, reduce=None, kernel_events=None, keep=None) -> None:
    """Queue cells that differ only in gamma (one sweep row), sharing one uniform stream per replicate.

    build_table seeds every cell with the same base_seed (montecarlo.py:276-277), so cells with
    equal n draw from identical uniforms: zks_run_cells draws each replicate's stream once for
    all of them (n <= 16384 in table mode; other sizes run cell by cell inside the same call).  The
    cells' order statistics are selected in batched launches.  Results are identical to running
    the cells one by one.
    """
    torch = _torch()
    cfg0 = plans[0].config
    n = cfg0.n
    if len(plans) < 2:
        for plan in plans:
            _enqueue_cell(eng, plan, shard=shard, reduce=reduce, kernel_events=kernel_events, keep=keep)
        return
    total = cfg0.replicates
    first, stop = shard if shard is not None else (0, total)
    dev = f"cuda:{eng.device}"
    ranks = quantile_ranks(total, cfg0.quantiles)
    outs = []
    stream = eng.bind_stream()
    # one allocation (and one fill) for the whole row's quantiles and worst statuses
    quantiles = torch.empty((len(plans), cfg0.repetitions, len(ranks)), dtype=torch.float64, device=dev)
    worst = torch.zeros((len(plans), cfg0.repetitions), dtype=torch.uint8, device=dev)
    for i, plan in enumerate(plans):
        plan.quantiles = quantiles[i]
        plan.worst = worst[i]
        plan.started = torch.cuda.Event(enable_timing=True)
        plan.finished = torch.cuda.Event(enable_timing=True)
        plan.started.record(stream)
        outs.append(_Slab(eng, max(total, 1)))
    # while the host still builds draw tables (the first row of a sweep), the first few cells go
    # ahead in a launch of their own, so the device starts after _EARLY_CELLS tables instead of
    # after all of them (results do not depend on how a row's cells are grouped)
    pending = any((eng.device, float(p.config.gamma), p.config.support.k) in _PENDING for p in plans)
    tables = [None] * len(plans)
    for rep in range(cfg0.repetitions):
        if stop > first:
            if kernel_events is not None:  # bench.py: the row's replicate kernels
                k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                k0.record(stream)
            # (small-n rows only: their extra stream draw is cheap beside the cells' work)
            lead = _EARLY_CELLS if rep == 0 and pending and n < 128 and len(plans) > 2 * _EARLY_CELLS else 0
            bounds = ([0] if lead else []) + list(range(lead, len(plans), _ROW_CELLS)) + [len(plans)]
            for a, b in zip(bounds[:-1], bounds[1:]):
                for j in range(a, b):
                    if tables[j] is None:
                        tables[j] = _table(eng, plans[j].config)
                part = slice(a, b)
                eng.run_cells(tables[part], cfg0.support.k, [p.config.gamma for p in plans[part]], n, cfg0.base_seed,
                              rep, first, stop - first,
                              [(o.ks[first:], o.gh[first:], o.st[first:]) for o in outs[part]])
            if kernel_events is not None:
                k1.record(stream)
                kernel_events.append((k0, k1))
        for plan, out in zip(plans, outs):
            _keep(keep, plan.config, rep, out, first, stop)
        # the row's cells in batched selections; the first rank chunk also takes the worst status
        # (multi-GPU: over this rank's shard, digit histograms summed by `reduce`; the worst
        # status is this rank's, all-reduced by the caller)
        jobs = []
        for plan, out in zip(plans, outs):
            jobs.extend((out.ks[first:stop], ranks[i : i + 16], plan.quantiles[rep, i : i + 16])
                        + ((out.st[first:stop], plan.worst[rep : rep + 1]) if i == 0 else ())
                        for i in range(0, len(ranks), 16))
        for i0 in range(0, len(ranks), 16):  # equal rank counts per launch
            part = [j for j in jobs if j[1] == ranks[i0 : i0 + 16]]
            if reduce is None:
                eng.select_many(part)
            else:
                eng.select_dist(part, total, reduce)
    for plan in plans:
        plan.finished.record(stream)


def _prefetch_tables(eng, configs) -> None:
    """Start building the host sampling CDFs a sweep still lacks on a thread pool (numpy releases
    the GIL); _table() takes each one when its first cell is enqueued, so device work starts
    after the first table instead of after all of them."""
    global _POOL
    missing = {}
    for cfg in configs:
        key = (float(cfg.gamma), cfg.support.k)
        if key not in missing and not eng.has_table(*key) and (eng.device, *key) not in _PENDING:
            missing[key] = cfg
    if len(missing) < 2:
        return
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _POOL = ThreadPoolExecutor(max_workers=min(os.cpu_count() or 1, 16))
    for key, cfg in missing.items():
        _PENDING[(eng.device, *key)] = _POOL.submit(sampling_cdf, cfg.gamma, cfg.support)


def _enqueue_plans(eng, plans: list[_CellPlan], shard=None, reduce=None, kernel_events=None, keep=None) -> None:
    """Queue many cells, grouping those that can share uniform streams (_enqueue_group)."""
    _prefetch_tables(eng, [p.config for p in plans])
    groups: dict = {}
    for plan in plans:
        groups.setdefault(_stage_key(plan.config), []).append(plan)
    for group in groups.values():
        _enqueue_group(eng, group, shard=shard, reduce=reduce, kernel_events=kernel_events, keep=keep)


def _fetch_plans(plans: list[_CellPlan]) -> None:
    """One device-to-host copy of every plan's worst statuses and quantiles (instead of two
    synchronising copies per cell); _finish_cell then reads the host copies."""
    torch = _torch()
    if not plans:
        return
    flat = torch.cat([torch.cat([p.quantiles.reshape(-1), p.worst.to(torch.float64)]) for p in plans]).cpu().numpy()
    at = 0
    for p in plans:
        nq, nw = p.quantiles.numel(), p.worst.numel()
        p.host = (flat[at : at + nq].reshape(p.quantiles.shape), flat[at + nq : at + nq + nw].astype(np.uint8))
        at += nq + nw


def _finish_cell(eng, plan: _CellPlan, shard: tuple[int, int] | None = None) -> list[tuple[float, float]]:
    cfg = plan.config
    host = getattr(plan, "host", None)
    worst = host[1] if host is not None else plan.worst.cpu().numpy()
    if worst.max(initial=0) >= _native.STATUS_FAILED:
        # re-run the first failing repetition to name the first failing replicate
        rep = int(np.flatnonzero(worst >= _native.STATUS_FAILED)[0])
        first, stop = shard if shard is not None else (0, cfg.replicates)
        slab = _slab(eng, cfg.replicates)
        _enqueue(eng, cfg, rep, first, stop - first, slab, offset=first)
        _raise_first_failure(cfg, rep, first, slab.st[first:stop].cpu().numpy(), slab.gh[first:stop].cpu().numpy())
    per_rep = host[0] if host is not None else plan.quantiles.cpu().numpy()
    per_level = np.zeros(per_rep.shape[1])
    for rep in range(cfg.repetitions):  # montecarlo.py:203-211: add in repetition order
        per_level += per_rep[rep]
    per_level /= cfg.repetitions
    return list(zip(cfg.quantiles, (float(c) for c in per_level)))


def run_simulation(config: SimulationConfig, workers: int | None = None) -> list[tuple[float, float]]:
    """(level, cutoff) pairs: per-repetition order quantiles averaged over repetitions
    (montecarlo.py:194-212)."""
    resolve_workers(workers)
    eng = _engine()
    plan = _CellPlan(config)
    _enqueue_cell(eng, plan)
    return _finish_cell(eng, plan)


# ---------------------------------------------------------------------------
# cutoff tables (montecarlo.py:218-314)

class CutoffLookupError(LookupError):
    """No tabulated cell matches the requested (gamma, n, level)."""


GAMMA_LOOKUP_WINDOW = 0.005


@dataclass(frozen=True, eq=True)
class CutoffTable:
    """Grid of cutoffs over (gamma, n) for one support, plus its provenance."""

    support: Support
    levels: tuple[float, ...]
    gammas: tuple[float, ...]
    ns: tuple[int, ...]
    cells: dict[tuple[float, int], tuple[float, ...]] = field(compare=True)
    replicates: int = 50000
    repetitions: int = 10
    base_seed: int = 0

    def cutoffs_for(self, gamma: float, n: int) -> tuple[float, ...]:
        if n not in self.ns:
            raise CutoffLookupError(f"no tabulated sample size n={n}; compute a bespoke cutoff instead")
        delta, nearest = min((abs(g - gamma), g) for g in self.gammas)
        if delta > GAMMA_LOOKUP_WINDOW + 1e-12:
            raise CutoffLookupError(
                f"estimated exponent {gamma:.4f} is not within ±{GAMMA_LOOKUP_WINDOW} of "
                f"any tabulated value; compute a bespoke cutoff instead"
            )
        return self.cells[(nearest, n)]

    def cutoff(self, gamma: float, n: int, level: float) -> float:
        row = self.cutoffs_for(gamma, n)
        try:
            return row[self.levels.index(float(level))]
        except ValueError:
            raise CutoffLookupError(f"level {level} not tabulated (have {self.levels})") from None


def build_table(
    ns: Iterable[int],
    gammas: Iterable[float],
    support: Support,
    base_seed: int,
    replicates: int = 50000,
    repetitions: int = 10,
    quantiles: Sequence[float] = DEFAULT_LEVELS,
    workers: int | None = None,
    progress: Callable[[float, int, float, tuple[float, ...]], None] | None = None,
) -> CutoffTable:
    """Fill the (gamma, n) grid (montecarlo.py:263-314).

    Every cell reuses ``base_seed`` exactly as the reference does.  All cells are queued on
    the device back to back (host table builds overlap device work); ``progress`` receives
    each cell's device time in seconds.
    """
    ns = tuple(int(n) for n in ns)
    gammas = tuple(float(g) for g in gammas)
    if not ns or not gammas:
        raise ValueError("both grids must be nonempty")
    levels = _validate_levels(quantiles)
    resolve_workers(workers)
    plans: list[_CellPlan] = []
    for gamma in gammas:
        for n in ns:
            try:
                cfg = SimulationConfig(n=n, support=support, gamma=gamma, base_seed=base_seed,
                                       replicates=replicates, repetitions=repetitions, quantiles=levels)
            except Exception as err:
                raise SimulationError(f"table cell (gamma={gamma}, n={n}) failed: {err}") from err
            plans.append(_CellPlan(cfg))
    eng = _engine()
    _enqueue_plans(eng, plans)
    _fetch_plans(plans)
    cells: dict[tuple[float, int], tuple[float, ...]] = {}
    for plan in plans:
        cfg = plan.config
        try:
            pairs = _finish_cell(eng, plan)
        except Exception as err:
            raise SimulationError(f"table cell (gamma={cfg.gamma}, n={cfg.n}) failed: {err}") from err
        row = tuple(c for _, c in pairs)
        cells[(cfg.gamma, cfg.n)] = row
        if progress is not None:
            plan.finished.synchronize()
            progress(cfg.gamma, cfg.n, plan.started.elapsed_time(plan.finished) / 1e3, row)
    return CutoffTable(support=support, levels=levels, gammas=gammas, ns=ns, cells=cells,
                       replicates=replicates, repetitions=repetitions, base_seed=base_seed)
