"""Multi-process host logic of the sharded path (paper_1305_6738_b200/parallel.py) on CPU/gloo.

On a GPU box every rank runs the replicate kernel on its shard and the order statistics are
selected across the shards (per-pass digit histograms summed by an all-reduce, then the same
digit picked on every rank); here the shard values come from the CPU oracle and the collectives
run over gloo: the same sharding, the histogram reduction (parallel.histogram_reducer) with a
host model of the radix passes, and the index-order all-gather (ShardGather).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1305_6738_b200.parallel import ShardGather, gathered_order, histogram_reducer, padded_size, shard_bounds


def test_shard_bounds_cover_in_order():
    for total in (100, 101, 1000, 4097, 1_000_000):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert padded_size(total, world) >= total
            assert max(b - a for a, b in spans) == -(-total // world)
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, cell, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import port as oracle

        gamma, support, n, seed, rep = cell
        start, stop = shard_bounds(total, world, rank)
        local = torch.zeros(padded_size(total, world), dtype=torch.float64)
        ks, _, _ = oracle.replicate_range(gamma, support, n, seed, rep, start, stop)
        local[start:stop] = torch.from_numpy(ks)
        full = ShardGather(total, world, rank)(local)
        worst = torch.tensor([rank], dtype=torch.int32)
        dist.all_reduce(worst, op=dist.ReduceOp.MAX)
        out_q.put((rank, full.numpy().copy(), int(worst.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 203), (2, 100), (3, 128)])
def test_gather_reassembles_index_order_and_quantiles(world, total):
    from oracle import port as oracle

    cell = (1.5, 20, 30, 7, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, cell, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want, _, _ = oracle.replicate_range(1.5, 20, 30, 7, 1, 0, total)
    for rank, full, worst in results:
        np.testing.assert_array_equal(full, want)  # bit-identical to the unsharded run
        assert worst == world - 1
        assert oracle.order_quantiles(full, oracle.LEVELS) == oracle.order_quantiles(want, oracle.LEVELS)


def test_host_model_of_gather():
    parts = [np.arange(0, 4.0), np.arange(4, 8.0), np.array([8.0, 9.0, 0.0, 0.0])]
    np.testing.assert_array_equal(gathered_order(parts, 10), np.arange(10.0))


def _radix_select_model(local_keys: np.ndarray, ranks, reduce) -> list[int]:
    """Host model of the distributed radix select (zks_select.cuh): 8 passes of 8-bit digits
    over uint64 keys; each rank histograms its own keys matching each rank's prefix, ``reduce``
    sums the histograms over the ranks, every rank picks the same digit."""
    pre = [0] * len(ranks)
    want = list(ranks)
    for p in range(8):
        shift = 56 - 8 * p
        mask = 0 if p == 0 else (~0 << (shift + 8)) & 0xFFFFFFFFFFFFFFFF
        hist = torch.zeros((len(ranks), 256), dtype=torch.int32)
        for r in range(len(ranks)):
            sel = local_keys[(local_keys & np.uint64(mask)) == np.uint64(pre[r])]
            digits = ((sel >> np.uint64(shift)) & np.uint64(255)).astype(np.int64)
            hist[r] += torch.from_numpy(np.bincount(digits, minlength=256).astype(np.int32))
        reduce(hist)
        for r in range(len(ranks)):
            cum = np.cumsum(hist[r].numpy().astype(np.int64))
            d = int(np.searchsorted(cum, want[r], side="right"))
            want[r] -= int(cum[d - 1]) if d else 0
            pre[r] |= d << shift
    return pre


def _select_worker(rank, world, port, total, cell, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import port as oracle

        gamma, support, n, seed, rep = cell
        start, stop = shard_bounds(total, world, rank)
        ks, _, _ = oracle.replicate_range(gamma, support, n, seed, rep, start, stop)
        keys = np.ascontiguousarray(ks, dtype=np.float64).view(np.uint64)
        ranks = [0, total // 2, int(0.9 * total), int(0.99 * total), total - 1]
        got = _radix_select_model(keys, ranks, histogram_reducer())
        out_q.put((rank, [float(np.array([k], dtype=np.uint64).view(np.float64)[0]) for k in got], ranks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 301), (3, 200)])
def test_distributed_select_model_matches_order_statistics(world, total):
    from oracle import port as oracle

    cell = (2.0, None, 40, 3, 0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_select_worker, args=(r, world, port, total, cell, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full, _, _ = oracle.replicate_range(2.0, None, 40, 3, 0, 0, total)
    srt = np.sort(full)
    for _, got, ranks in results:
        assert got == [float(srt[r]) for r in ranks]
