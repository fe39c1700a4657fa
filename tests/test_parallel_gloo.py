"""Multi-process host logic of the sharded path (paper_1305_6738_b200/parallel.py) on CPU/gloo.

On a GPU box every rank runs the replicate kernel on its shard and NCCL all-gathers the KS
values; here the shard values come from the CPU oracle and the gather runs over gloo, which
exercises the same sharding, padding and index-order reassembly code.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1305_6738_b200.parallel import ShardGather, gathered_order, padded_size, shard_bounds


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
