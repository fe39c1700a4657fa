"""Multi-GPU cutoff tables: one process per GPU, replicate ranges sharded, a distributed select.

The reference parallelises one repetition over a process pool of 512-replicate spans
(montecarlo.py:151-191) and is worker-count invariant because streams are keyed
``(base_seed, repetition, index)``.  Here each rank of a ``torch.distributed`` group (NCCL
over NVLink on a B200 box) computes a contiguous shard of replicate indices of every
(cell, repetition) into its slice of a device buffer, and the order statistics are selected
across the shards without moving the KS values: per radix pass every rank histograms the
digits of its own keys, an NCCL all-reduce sums the histograms (4 x 256 counts per cell and
pass), and every rank picks the same digits -- so the table is bit-identical for any number of
GPUs and each rank's selection work stays proportional to its shard.  A cell's worst status is
all-reduced so every rank raises the same SimulationError.  ``ShardGather`` (an all-gather of
the shards in index order) remains for callers that want the full KS arrays.
"""
from __future__ import annotations

from typing import Iterable, Sequence

import numpy as np

from . import _native
from .distribution import Support
from .montecarlo import (
    DEFAULT_LEVELS,
    CutoffTable,
    SimulationConfig,
    SimulationError,
    _CellPlan,
    _engine,
    _enqueue,
    _enqueue_plans,
    _failure,
    _fetch_plans,
    _finish_cell,
    _slab,
    _validate_levels,
)


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous equal-size shards: rank r owns [r*c, min((r+1)*c, total)), c = ceil(total/world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    chunk = -(-total // world)
    start = min(rank * chunk, total)
    return start, min(start + chunk, total)


def padded_size(total: int, world: int) -> int:
    return -(-total // world) * world


class ShardGather:
    """All-gather of equal-size shards of a 1-D tensor into index order."""

    def __init__(self, total: int, world: int, rank: int, group=None):
        self.total, self.world, self.rank, self.group = total, world, rank, group
        self.chunk = -(-total // world)
        self.out = None

    def __call__(self, local_full, fresh: bool = False):
        """All-gathered copy of ``local_full``; into a reused buffer, or a new one (``fresh``) when
        several gathered arrays must stay alive (a sweep row's batched selection)."""
        import torch
        import torch.distributed as dist

        need = self.chunk * self.world
        if fresh:
            self.out = None
        if self.out is None or self.out.numel() < need or self.out.device != local_full.device:
            self.out = torch.empty(need, dtype=local_full.dtype, device=local_full.device)
        start = self.rank * self.chunk
        mine = local_full[start : start + self.chunk]
        if mine.numel() < self.chunk:  # last shard shorter than the padded chunk
            pad = torch.zeros(self.chunk, dtype=local_full.dtype, device=local_full.device)
            pad[: mine.numel()] = mine
            mine = pad
        dist.all_gather_into_tensor(self.out[:need], mine.contiguous(), group=self.group)
        return self.out[: self.total]


def histogram_reducer(group=None):
    """Sum of a device tensor over the ranks of ``group`` in place (NCCL all-reduce): the
    distributed selection's per-pass digit histograms."""
    import torch.distributed as dist

    def reduce(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return reduce


def build_table(
    ns: Iterable[int],
    gammas: Iterable[float],
    support: Support,
    base_seed: int,
    replicates: int = 50000,
    repetitions: int = 10,
    quantiles: Sequence[float] = DEFAULT_LEVELS,
    group=None,
) -> CutoffTable:
    """montecarlo.build_table over every GPU of ``group`` (default: the world group).

    Call collectively from every rank; every rank returns the same table, equal bit for bit
    to the single-GPU result.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ns = tuple(int(n) for n in ns)
    gammas = tuple(float(g) for g in gammas)
    if not ns or not gammas:
        raise ValueError("both grids must be nonempty")
    levels = _validate_levels(quantiles)
    eng = _engine()
    plans = []
    for gamma in gammas:
        for n in ns:
            cfg = SimulationConfig(n=n, support=support, gamma=gamma, base_seed=base_seed, replicates=replicates,
                                   repetitions=repetitions, quantiles=levels)
            plans.append(_CellPlan(cfg))
    shard = shard_bounds(replicates, world, rank)
    _slab(eng, padded_size(replicates, world))
    _enqueue_plans(eng, plans, shard=shard, reduce=histogram_reducer(group))
    # every rank's worst status per (cell, repetition), so every rank raises the same error
    worst = torch.stack([p.worst for p in plans]).to(torch.int32)
    dist.all_reduce(worst, op=dist.ReduceOp.MAX, group=group)
    worst_host = worst.cpu().numpy()
    for plan, w in zip(plans, worst_host):
        plan.worst.copy_(torch.from_numpy(np.where(w < _native.STATUS_FAILED, w, 0).astype(np.uint8)))
    _fetch_plans(plans)
    cells = {}
    for plan, w in zip(plans, worst_host):
        cfg = plan.config
        if w.max() >= _native.STATUS_FAILED:
            err = _first_failure(eng, cfg, int(np.flatnonzero(w >= _native.STATUS_FAILED)[0]), shard, group)
            raise SimulationError(f"table cell (gamma={cfg.gamma}, n={cfg.n}) failed: {err}") from err
        cells[(cfg.gamma, cfg.n)] = tuple(c for _, c in _finish_cell(eng, plan, shard=shard))
    return CutoffTable(support=support, levels=levels, gammas=gammas, ns=ns, cells=cells, replicates=replicates,
                       repetitions=repetitions, base_seed=base_seed)


def _first_failure(eng, cfg: SimulationConfig, repetition: int, shard: tuple[int, int], group) -> SimulationError:
    """The reference's error for the first replicate of ``repetition`` that failed twice
    (montecarlo.py:106-116), agreed by every rank: each re-runs its shard of that repetition,
    an all-reduce MIN finds the first failing index and its owner contributes the mean log."""
    import torch
    import torch.distributed as dist

    first, stop = shard
    slab = _slab(eng, cfg.replicates)
    idx, mean_log = cfg.replicates, 0.0
    if stop > first:
        _enqueue(eng, cfg, repetition, first, stop - first, slab, offset=first)
        st = slab.st[first:stop].cpu().numpy()
        bad = np.flatnonzero(st == _native.STATUS_FAILED)
        if bad.size:
            idx = first + int(bad[0])
            mean_log = float(slab.gh[idx : idx + 1].cpu().numpy()[0])
    dev = f"cuda:{eng.device}"
    at = torch.tensor([idx], dtype=torch.int64, device=dev)
    dist.all_reduce(at, op=dist.ReduceOp.MIN, group=group)
    idx0 = int(at.item())
    ml = torch.tensor([mean_log if idx == idx0 else 0.0], dtype=torch.float64, device=dev)
    dist.all_reduce(ml, op=dist.ReduceOp.SUM, group=group)
    return _failure(cfg, repetition, idx0, float(ml.item()))


def gathered_order(values_by_rank: list[np.ndarray], total: int) -> np.ndarray:
    """Host-side model of the gather (tests): concatenate equal-size padded shards, keep prefix."""
    return np.concatenate(values_by_rank)[:total]
