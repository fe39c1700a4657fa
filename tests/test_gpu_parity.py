"""GPU parity: the CUDA engine against the reference's golden vectors and the CPU oracle.

Tiers (BASELINE.json north_star):
  1. streams and sampled integers bit-exact;
  2. gamma_hat and KS within 1e-10 relative (absolute floor 1e-12: KS can be exactly 0,
     finite-support gamma_hat can be 0) on identical samples;
  3. cutoff quantiles: bit-exact whenever every replicate KS is (selection is exact), else
     within MC error.
All calls go through the C ABI (libzks_b200.so).
"""
import os
import re

import numpy as np
import pytest



def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

RTOL = 1e-10
ATOL = 1e-12


def close(got, want):
    got, want = np.asarray(got), np.asarray(want)
    return np.abs(got - want) <= RTOL * np.abs(want) + ATOL


@pytest.fixture(scope="module")
def zk():
    import paper_1305_6738_b200 as zk
    from paper_1305_6738_b200 import engine

    eng = engine.get_engine()
    assert eng.lib is not None
    return zk


def run_cell(K, gamma, n, seed, rep, first, count):
    import torch

    from paper_1305_6738_b200 import engine
    from paper_1305_6738_b200.distribution import Support, sampling_cdf

    eng = engine.get_engine()
    support = Support(K)
    table = eng.table(gamma, K, lambda: sampling_cdf(gamma, support))
    dev = f"cuda:{eng.device}"
    ks = torch.empty(count, dtype=torch.float64, device=dev)
    gh = torch.empty(count, dtype=torch.float64, device=dev)
    st = torch.empty(count, dtype=torch.uint8, device=dev)
    eng.run_replicates(table, K, gamma, n, seed, rep, first, count, ks, gh, st)
    return ks.cpu().numpy(), gh.cpu().numpy(), st.cpu().numpy()


def golden_cells(golden):
    for ci, row in enumerate(golden["cells"]):
        k, gamma, n, seed, rep, count = row
        yield ci, (None if k == 0 else int(k)), float(gamma), int(n), int(seed), int(rep), int(count)


def test_streams_bitwise(zk, golden):
    i = 0
    while f"stream{i}_key" in golden:
        key = [int(x) for x in golden[f"stream{i}_key"]]
        u = zk.RandomStream(key).uniforms(37)
        assert u.tobytes() == golden[f"stream{i}_u"].tobytes()
        i += 1


def test_samples_bitwise(zk, golden):
    for ci, K, gamma, n, seed, rep, count in golden_cells(golden):
        if gamma < 0:
            continue
        model = zk.ZipfModel(gamma, zk.Support(K))
        for idx in range(min(count, 4)):
            s = zk.sample(model, n, zk.RandomStream.for_replicate(seed, rep, idx))
            np.testing.assert_array_equal(s.observations, golden[f"cell{ci}_sample{idx}"])


def test_fixed_stream_known_answers(zk):
    class FixedStream:
        def __init__(self, values):
            self.values = list(values)

        def uniforms(self, count):
            out, self.values = self.values[:count], self.values[count:]
            return np.asarray(out, dtype=np.float64)

    two = zk.ZipfModel(1.0, zk.Support.finite(2))
    assert zk.sample(two, 2, FixedStream([0.9, 0.5])).observations.tolist() == [2, 1]
    assert zk.sample(zk.ZipfModel(1.0, zk.Support.finite(5)), 1, FixedStream([1.0])).observations.tolist() == [5]
    assert zk.sample(zk.ZipfModel(1.7, zk.Support.finite(30)), 1, FixedStream([0.3])).observations.tolist() == [1]


@pytest.fixture(params=["table", "direct"])
def mle_mode(request, zk):
    """Run a test with the fit tables (default) and with direct model sums."""
    from paper_1305_6738_b200.engine import get_engine

    eng = get_engine()
    eng.set_mle_mode(direct=request.param == "direct")
    yield request.param
    eng.set_mle_mode(direct=False)


def test_replicates_match_reference_golden(zk, golden, mle_mode):
    for ci, K, gamma, n, seed, rep, count in golden_cells(golden):
        ks, gh, st = run_cell(K, gamma, n, seed, rep, 0, count)
        want_st = golden[f"cell{ci}_status"]
        np.testing.assert_array_equal(st, want_st, err_msg=f"cell {ci}")
        ok = want_st < 2
        assert close(ks[ok], golden[f"cell{ci}_ks"][ok]).all(), (ci, ks[ok], golden[f"cell{ci}_ks"][ok])
        assert close(gh[ok], golden[f"cell{ci}_gamma_hat"][ok]).all(), (ci, gh[ok], golden[f"cell{ci}_gamma_hat"][ok])
        # failed twice: the engine reports the retry sample's mean log for the message
        bad = ~ok
        if bad.any():
            assert close(gh[bad], golden[f"cell{ci}_target"][bad]).all()


@pytest.mark.parametrize(
    "K,gamma,n,seed,rep,count",
    [
        (None, 2.5, 100, 1, 0, 600),
        (None, 1.5, 1000, 3, 1, 200),
        (None, 1.25, 2000, 5, 0, 60),
        (None, 3.5, 10, 2, 0, 600),
        (None, 1.05, 20, 8, 0, 200),
        (1000, 0.5, 500, 4, 0, 300),
        (1000, 2.0, 30, 9, 2, 600),
        (5000, 1.0, 300, 6, 0, 100),
        (20, 0.25, 10, 1, 0, 600),
        (50, 4.0, 40, 12, 0, 600),
        (None, 1.6, 9000, 3, 0, 24),  # two-kernel path with u16 draw bins
        (1000, 1.0, 5000, 2, 0, 24),
        (None, 1.9, 40000, 4, 0, 8),  # two-kernel path near its u16 limit
        (None, 1.25, 30000, 3, 0, 8),  # ~9000 tail values over ~60 pages: page passes compact the tail
        (None, 2.3, 131, 8, 0, 96),  # n not a multiple of 4: the draw kernel's masked last step
        (1000, 0.5, 100, 5, 0, 128),  # n < 128 with tails of ~75 values above the head: warp-scored
        (1000, 0.9, 90, 6, 1, 128),  # tails around kLaneTailMax: lane- and warp-scored in one warp
        (None, 1.05, 120, 3, 0, 96),  # the heaviest unbounded tail at n < 128
        (None, 1.6, 800, 2, 0, 96),  # two-kernel path, tail lists around kFitLaneTailMax (lane + warp)
        (3, 0.7, 200, 6, 0, 64),  # supports shorter than the four counted values (cut table)
        (2, 1.0, 70, 6, 0, 64),  # ... at n < 128 (lane kernel: cuts of 0 from L - 1 on)
        (None, 1.3, 127, 8, 0, 96),  # the largest lane-kernel n (n % 4 = 3 words after the groups)
        (None, 2.0, 1, 3, 0, 64),  # one observation per sample
        (20, 1.0, 1, 3, 0, 64),
        (3, 0.7, 50, 6, 1, 64),
        (5, 2.0, 300, 7, 1, 64),
    ],
)
def test_replicates_match_oracle(zk, mle_mode, K, gamma, n, seed, rep, count):
    from oracle import port

    first = 1000
    ks, gh, st = run_cell(K, gamma, n, seed, rep, first, count)
    for j in range(count):
        want_ks, want_gh, want_st = port.replicate(gamma, K, n, seed, first + j, rep)
        assert st[j] == want_st
        assert close(ks[j], want_ks), (j, ks[j], want_ks)
        assert close(gh[j], want_gh), (j, gh[j], want_gh)


@pytest.mark.parametrize("K,gamma,n", [(6, -20.0, 140), (8, -20.0, 128), (8, -22.0, 60), (8, -22.0, 1000)])
def test_retries_match_oracle(zk, mle_mode, K, gamma, n):
    # cells where first attempts fail often (NoRootError): retried replicates (status 1) take
    # stream idx + 2^32 -- for n >= 128 through retry_kernel -- and double failures report 2
    from oracle import port

    count = 48
    ks, gh, st = run_cell(K, gamma, n, 7, 0, 0, count)
    seen = set()
    for j in range(count):
        try:
            want_ks, want_gh, want_st = port.replicate(gamma, K, n, 7, j, 0)
        except port.FailedTwice:
            assert st[j] == 2, j
            seen.add(2)
            continue
        assert st[j] == want_st, j
        assert close(ks[j], want_ks), (j, ks[j], want_ks)
        assert close(gh[j], want_gh), (j, gh[j], want_gh)
        seen.add(int(want_st))
    assert 1 in seen


def test_run_simulation_matches_reference_golden(zk, golden):
    for si, row in enumerate(golden["sims"]):
        k, gamma, n, seed, reps_r, reps = row
        cfg = zk.SimulationConfig(n=int(n), support=zk.Support(None if k == 0 else int(k)), gamma=float(gamma),
                                  base_seed=int(seed), replicates=int(reps_r), repetitions=int(reps))
        got = [c for _, c in zk.run_simulation(cfg, workers=1)]
        assert close(got, golden[f"sim{si}_cutoffs"]).all(), (si, got, golden[f"sim{si}_cutoffs"])
        ks, gh = zk.run_repetition(cfg, 0)
        assert close(ks, golden[f"sim{si}_rep0_ks"]).all()
        assert close(gh, golden[f"sim{si}_rep0_gamma_hat"]).all()


def test_order_quantiles_exact(zk):
    from oracle import port

    rng = np.random.default_rng(17)
    for count in (101, 1000, 50000, 1 << 20):
        stats = rng.random(count)
        assert zk.order_quantiles(stats, zk.DEFAULT_LEVELS) == port.order_quantiles(stats, zk.DEFAULT_LEVELS)
    stats = np.arange(100) / 100.0
    assert zk.order_quantiles(stats, [0.29]) == [0.29]
    dup = np.repeat(rng.random(50), 40)
    assert zk.order_quantiles(dup, [0.1, 0.5, 0.9]) == port.order_quantiles(dup, [0.1, 0.5, 0.9])
    with pytest.raises(ValueError):
        zk.order_quantiles([], [0.9])


def test_order_quantiles_signed_and_nan(zk):
    # the reference sorts any float64 array (montecarlo.py:119-136): negative values, -0.0,
    # infinities and NaNs (last, as np.sort puts them) select like np.sort
    from oracle import port

    rng = np.random.default_rng(23)
    levels = (0.001, 0.1, 0.25, 0.5, 0.75, 0.9, 0.95, 0.99, 0.999)
    for count in (100, 4097, 300000):
        x = rng.standard_normal(count) * 10.0 ** rng.integers(-300, 300, count)
        x[::7] = -0.0
        x[::11] = 0.0
        x[3::13] = -np.inf
        x[5::17] = np.inf
        want = port.order_quantiles(x, levels)
        np.testing.assert_array_equal(zk.order_quantiles(x, levels), want)
        x[1::5] = np.nan
        x[2::9] = -np.nan
        np.testing.assert_array_equal(zk.order_quantiles(x, levels), port.order_quantiles(x, levels))
    neg = -rng.random(1000)
    np.testing.assert_array_equal(zk.order_quantiles(neg, levels), port.order_quantiles(neg, levels))


def test_double_failure_raises_with_diagnostics(zk):
    cfg = zk.SimulationConfig(n=3, support=zk.Support.finite(20), gamma=-30.0, base_seed=101, replicates=100,
                              repetitions=1)
    with pytest.raises(zk.SimulationError, match=r"gamma=-30.0, n=3"):
        zk.run_simulation(cfg)
    with pytest.raises(zk.SimulationError, match="failed twice: estimating equation has no root"):
        for index in range(20):
            zk.run_replicate(cfg, index)


def test_build_table_matches_run_simulation(zk):
    table = zk.build_table(ns=(20, 50), gammas=(1.0, 1.5), support=zk.Support.finite(20), base_seed=5,
                           replicates=200, repetitions=2)
    for (g, n), row in table.cells.items():
        cfg = zk.SimulationConfig(n=n, support=zk.Support.finite(20), gamma=g, base_seed=5, replicates=200,
                                  repetitions=2)
        assert row == tuple(c for _, c in zk.run_simulation(cfg))
    with pytest.raises(zk.SimulationError, match=r"gamma=-30.0, n=3"):
        zk.build_table(ns=(3,), gammas=(-30.0,), support=zk.Support.finite(20), base_seed=5, replicates=100,
                       repetitions=1)
    # a failing cell inside a batched sweep row (worst status through the batched selection),
    # for the small-n rows and the row kernel (one stream per replicate for every gamma)
    with pytest.raises(zk.SimulationError, match=r"gamma=-30.0, n=3"):
        zk.build_table(ns=(3,), gammas=(1.0, -30.0), support=zk.Support.finite(20), base_seed=5, replicates=100,
                       repetitions=2)
    with pytest.raises(zk.SimulationError, match=r"gamma=-30.0, n=200"):
        zk.build_table(ns=(200,), gammas=(1.0, -30.0), support=zk.Support.finite(20), base_seed=5, replicates=100,
                       repetitions=1)


def test_sweep_with_shared_uniforms_matches_cells(zk):
    # build_table draws each replicate stream once per sweep row for all its gammas (zks_run_cells,
    # 128 <= n <= 16384); every cell must equal its own run_simulation bit for bit
    table = zk.build_table(ns=(131, 200, 701), gammas=(1.6, 2.2, 3.0), support=zk.Support.unbounded(), base_seed=3,
                           replicates=3000, repetitions=2)  # 131, 701: masked last blocks
    for (g, n), row in table.cells.items():
        cfg = zk.SimulationConfig(n=n, support=zk.Support.unbounded(), gamma=g, base_seed=3, replicates=3000,
                                  repetitions=2)
        assert row == tuple(c for _, c in zk.run_simulation(cfg)), (g, n)
    t2 = zk.build_table(ns=(300,), gammas=(0.5, 1.5), support=zk.Support.finite(1000), base_seed=8,
                        replicates=2000, repetitions=1)
    for (g, n), row in t2.cells.items():
        cfg = zk.SimulationConfig(n=n, support=zk.Support.finite(1000), gamma=g, base_seed=8, replicates=2000,
                                  repetitions=1)
        assert row == tuple(c for _, c in zk.run_simulation(cfg)), (g, n)


def test_large_n_config4_sample_properties(zk):
    # BASELINE config 4 shape at n = 10^6: size-independent checks (range, determinism)
    ks1, gh1, st1 = run_cell(None, 2.0, 1_000_000, 1, 0, 0, 8)
    ks2, gh2, st2 = run_cell(None, 2.0, 1_000_000, 1, 0, 0, 8)
    assert (st1 == 0).all()
    np.testing.assert_array_equal(ks1, ks2)
    np.testing.assert_array_equal(gh1, gh2)
    assert ((gh1 > 1.95) & (gh1 < 2.05)).all()
    assert ((ks1 > 0) & (ks1 < 0.01)).all()


def test_sharded_ranges_are_bitwise_identical(zk):
    ks, gh, st = run_cell(None, 2.0, 100, 3, 0, 0, 4096)
    parts = [run_cell(None, 2.0, 100, 3, 0, a, b - a) for a, b in ((0, 1000), (1000, 3001), (3001, 4096))]
    np.testing.assert_array_equal(ks, np.concatenate([p[0] for p in parts]))
    np.testing.assert_array_equal(gh, np.concatenate([p[1] for p in parts]))


def test_cells_on_two_streams_match_sequential(zk):
    # the engine keeps its scratch (work counters, pre-drawn rows) per CUDA stream: cells enqueued
    # on two streams at once give the same results as one after the other
    import torch

    from paper_1305_6738_b200 import engine
    from paper_1305_6738_b200.distribution import Support, sampling_cdf

    eng = engine.get_engine()
    cells = [(None, 2.2, 300), (None, 1.8, 600), (1000, 1.0, 50), (None, 2.6, 400)]
    R = 3000

    def run(streams):
        outs = []
        for i, (K, g, n) in enumerate(cells):
            table = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))
            with torch.cuda.stream(streams[i % len(streams)]):
                ks = torch.empty(R, dtype=torch.float64, device="cuda")
                gh = torch.empty_like(ks)
                st = torch.empty(R, dtype=torch.uint8, device="cuda")
                eng.run_replicates(table, K, g, n, 5, 0, 0, R, ks, gh, st)
                outs.append((ks, gh, st))
        torch.cuda.synchronize()
        eng.bind_stream()
        return [tuple(x.cpu().numpy() for x in o) for o in outs]

    seq = run([torch.cuda.current_stream()])
    par = run([torch.cuda.Stream(), torch.cuda.Stream()])
    for a, b in zip(seq, par):
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


def test_parallel_build_table_single_rank_matches(zk):
    # the multi-GPU path (shards, the distributed radix select with its histogram all-reduces,
    # all-reduced worst status) on a one-rank NCCL group equals the single-GPU table bit for bit
    import socket

    import torch
    import torch.distributed as dist

    from paper_1305_6738_b200 import parallel

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        kw = dict(ns=(20, 300), gammas=(1.7, 2.4), support=zk.Support.unbounded(), base_seed=9, replicates=2000,
                  repetitions=2)
        assert parallel.build_table(**kw).cells == zk.build_table(**kw).cells
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("split", [(500, 7500), (0, 8000), (2999, 5001), (4000, 4000)])
def test_distributed_select_over_shards_matches_whole_array(zk, split):
    # the distributed selection's arithmetic without NCCL: two engines on one GPU each hold a
    # shard; their per-pass digit counts land in ONE histogram (the all-reduce's sum), both pick
    # from it -- every order statistic equals the single-array selection, on both engines
    import ctypes

    import torch

    from paper_1305_6738_b200 import _native, engine

    rng = np.random.default_rng(split[0] + 7)
    n = sum(split)
    vals = torch.tensor(np.concatenate([rng.random(n // 2) * 0.08, rng.random(n - n // 2) * 0.3]) ** 1.5,
                        dtype=torch.float64, device="cuda")
    vals[::97] = vals[3]  # ties
    ranks = [0, 1, n // 3, int(0.9 * n), int(0.99 * n), n - 1]
    want = torch.empty(len(ranks), dtype=torch.float64, device="cuda")
    main = engine.get_engine()
    main.select_ranks(vals, ranks, out=want)
    engines = [main, engine.Engine(0)]
    shards = [vals[: split[0]], vals[split[0] :]]
    outs = [torch.empty(len(ranks), dtype=torch.float64, device="cuda") for _ in engines]
    lib = main.lib
    r = np.ascontiguousarray([ranks], dtype=np.int64)
    for eng, sh, out in zip(engines, shards, outs):
        eng.bind_stream()
        ptr = (ctypes.c_void_p * 1)(sh.data_ptr() if sh.numel() else None)
        optr = (ctypes.c_void_p * 1)(out.data_ptr())
        nil = (ctypes.c_void_p * 1)(None)
        cnt = np.array([sh.numel()], dtype=np.int64)
        tot = np.array([n], dtype=np.int64)
        _native.check(lib.zks_select_dist_begin(eng.handle, ptr, cnt.ctypes.data, tot.ctypes.data, 1, r.ctypes.data,
                                                len(ranks), optr, nil, nil))
    hist = torch.empty(len(ranks) * 256, dtype=torch.int32, device="cuda")
    for p in range(8):
        hist.zero_()
        for eng in engines:
            _native.check(lib.zks_select_dist_count(eng.handle, p, hist.data_ptr()))
        for eng in engines:
            _native.check(lib.zks_select_dist_pick(eng.handle, p, hist.data_ptr()))
    for eng in engines:
        _native.check(lib.zks_select_dist_end(eng.handle))
    torch.cuda.synchronize()
    for out in outs:
        assert out.cpu().tolist() == want.cpu().tolist()
    engines[1].close()


@pytest.mark.parametrize("direct", [False, True])
def test_slab_and_selection_on_two_streams_match_sequential(zk, direct):
    # every scratch buffer a launch writes (overflow slab of replicate_kernel at n > 65535 and in
    # direct-MLE mode, selection state and candidates) is per stream; tables built on one stream
    # are waited for by the first use on another
    import torch

    from paper_1305_6738_b200 import engine
    from paper_1305_6738_b200.distribution import Support, sampling_cdf

    eng = engine.get_engine()
    cells = [(None, 1.5, 70000, 24), (None, 1.3, 66000, 24), (None, 1.7, 700, 600), (1000, 0.9, 3000, 600)]
    ranks = [3, 10, 20]

    def run(streams, fresh):
        outs = []
        if fresh:
            eng.clear_tables()
        for i, (K, g, n, R) in enumerate(cells):
            with torch.cuda.stream(streams[i % len(streams)]):
                table = eng.table(g, K, lambda: sampling_cdf(g, Support(K)))  # built on this stream
                ks = torch.empty(R, dtype=torch.float64, device="cuda")
                gh = torch.empty_like(ks)
                st = torch.empty(R, dtype=torch.uint8, device="cuda")
                q = torch.empty(len(ranks), dtype=torch.float64, device="cuda")
                eng.run_replicates(table, K, g, n, 5, 0, 0, R, ks, gh, st)
                eng.select_ranks(ks, ranks, out=q)
                outs.append((ks, gh, st, q))
        torch.cuda.synchronize()
        eng.bind_stream()
        return [tuple(x.cpu().numpy() for x in o) for o in outs]

    eng.set_mle_mode(direct)
    try:
        seq = run([torch.cuda.current_stream()], True)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        par = run([s1, s2], True)
        par2 = run([s2, s1], False)  # tables now used on the other stream
    finally:
        eng.set_mle_mode(False)
    for a, b, c in zip(seq, par, par2):
        for x, y, z in zip(a, b, c):
            np.testing.assert_array_equal(x, y)
            np.testing.assert_array_equal(x, z)


def test_parallel_build_table_failure_names_the_replicate(zk):
    # multi-GPU build_table raises the single-GPU (reference) message: first failing replicate,
    # its repetition and mean log (montecarlo.py:106-116), agreed over the ranks
    import socket

    import torch
    import torch.distributed as dist

    from paper_1305_6738_b200 import parallel

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        kw = dict(ns=(3,), gammas=(1.0, -30.0), support=zk.Support.finite(20), base_seed=5, replicates=100,
                  repetitions=2)
        with pytest.raises(zk.SimulationError) as single:
            zk.build_table(**kw)
        with pytest.raises(zk.SimulationError) as multi:
            parallel.build_table(**kw)
        assert str(multi.value) == str(single.value)
        assert re.search(r"failed: replicate \d+ \(repetition 0, gamma=-30.0, n=3, support=20\) failed twice: "
                         r"estimating equation has no root .*\(mean log of data: ", str(multi.value))
    finally:
        dist.destroy_process_group()


def _row_outputs(zk, K, n, gammas, R, seed=3):
    """Per-replicate (ks, gamma_hat, status) of a sweep row through build_table's scheduler."""
    import torch

    from paper_1305_6738_b200 import montecarlo as mc

    eng = mc._engine()
    plans = [mc._CellPlan(zk.SimulationConfig(n=n, support=zk.Support(K), gamma=g, base_seed=seed, replicates=R,
                                              repetitions=1)) for g in gammas]
    keep = {}
    mc._enqueue_plans(eng, plans, keep=keep)
    torch.cuda.synchronize()
    return {g: tuple(t.cpu().numpy() for t in keep[(g, n, 0)]) for g in gammas}


@pytest.mark.parametrize("K,n", [(None, 300), (None, 5000), (None, 12000), (1000, 300), (1000, 5000), (1000, 12000)])
def test_chunked_rows_match_single_chunk(zk, K, n):
    # the pre-drawn rows of a sweep row run in >= 3 chunks (budget shrunk): every replicate's
    # (ks, gamma_hat, status) equals the single-chunk run's and the cell's run on its own
    from paper_1305_6738_b200 import montecarlo as mc

    R = 20000 if n <= 5000 else 6000
    gammas = (0.8, 1.6) if K else (1.6, 2.5)
    eng = mc._engine()
    whole = _row_outputs(zk, K, n, gammas, R)
    eng.set_chunk_bytes(max(1, (R // 4) * (200 + 4 * n) * len(gammas)))  # >= 4 chunks of pre-drawn rows
    try:
        chunked = _row_outputs(zk, K, n, gammas, R)
    finally:
        eng.set_chunk_bytes(0)
    for g in gammas:
        for a, b in zip(whole[g], chunked[g]):
            np.testing.assert_array_equal(a, b)
        cell = run_cell(K, g, n, 3, 0, 0, R)
        for a, b in zip(whole[g], cell):
            np.testing.assert_array_equal(a, b)
        assert (whole[g][2] == 0).mean() > 0.99


@pytest.mark.parametrize("direct", [False, True])
@pytest.mark.parametrize("gamma,n,idxs", [(2.0, 1_000_000, (0, 1, 2)), (1.5, 100_000, (0, 7)), (1.3, 70_000, (3,))])
def test_large_n_per_replicate_oracle_parity(zk, direct, gamma, n, idxs):
    # n > 65535 (BASELINE config 4 at n = 10^6; heavy tails through the overflow slab and its
    # in-place page compaction): per replicate against the oracle at 1e-10
    from oracle import port
    from paper_1305_6738_b200 import engine

    eng = engine.get_engine()
    eng.set_mle_mode(direct)
    try:
        for i in idxs:
            ks, gh, st = run_cell(None, gamma, n, 1, 0, i, 1)
            want_ks, want_gh, want_st = port.replicate(gamma, None, n, 1, i, 0)
            assert st[0] == want_st
            assert close(ks[0], want_ks), (i, ks[0], want_ks)
            assert close(gh[0], want_gh), (i, gh[0], want_gh)
    finally:
        eng.set_mle_mode(False)


@pytest.mark.parametrize("K", [100, 500, 1000])
def test_truncated_corner_negative_gamma_hat(zk, K):
    # K in {100, 500, 1000}, gamma = 0.25, n = 10: gamma_hat is often negative (the finite
    # bracket [-20, 20]) and values above 64 are scored past the lane-walk head
    from oracle import port

    R = 400
    ks, gh, st = run_cell(K, 0.25, 10, 1, 0, 0, R)
    neg = 0
    for i in range(R):
        want_ks, want_gh, want_st = port.replicate(0.25, K, 10, 1, i, 0)
        assert st[i] == want_st, i
        assert close(ks[i], want_ks), (i, ks[i], want_ks)
        assert close(gh[i], want_gh), (i, gh[i], want_gh)
        neg += want_gh < 0
    assert neg > R // 10


@pytest.mark.parametrize("K,n", [(None, 128), (None, 16384), (None, 16385), (1000, 128), (1000, 16384), (20, 777)])
def test_row_kernel_bounds_and_many_cells(zk, K, n):
    # the row kernel's size bounds (n = 128 and 16384; 16385 runs cell by cell) and rows of more
    # cells than one call takes (33 gammas: two calls): every cell equals its own run
    gammas = tuple(np.round(np.linspace(1.2 if K is None else 0.3, 3.5, 33), 6))
    R = 512
    rows = _row_outputs(zk, K, n, gammas, R)
    for g in gammas[::4] + gammas[-1:]:
        cell = run_cell(K, g, n, 3, 0, 0, R)
        for a, b in zip(rows[g], cell):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("K,n,gammas", [
    (None, 5, (1.1, 2.0, 3.5)),
    (None, 37, tuple(np.round(np.linspace(1.1, 3.5, 21), 6))),
    (None, 127, (1.06, 1.1, 1.3, 2.2, 4.0)),
    (20, 10, tuple(np.round(np.linspace(0.25, 4.0, 33), 6))),
    (1000, 100, (0.25, 0.5, 1.0, 2.0)),
    (20, 3, (1.0, -30.0)),
])
def test_small_row_kernel_matches_cells(zk, K, n, gammas):
    # n < 128 rows: (replicate, cell) pairs lane by lane, streams drawn once per tile; every cell
    # equals its own run (the lane kernel above n = 16) bit for bit -- long tails (gamma ~ 1.1 at
    # n = 127), double failures (gamma = -30), rows of more than 32 cells
    R = 1000
    rows = _row_outputs(zk, K, n, gammas, R)
    for g in gammas:
        cell = run_cell(K, g, n, 3, 0, 0, R)
        for a, b in zip(rows[g], cell):
            np.testing.assert_array_equal(a, b)
    if -30.0 in gammas:
        assert (rows[-30.0][2] == 2).any()


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_build_table_matches_single_process(zk, world):
    # real ranks (torchrun, one process each) sharing the one GPU, gloo collectives: shards, the
    # distributed selection's histogram all-reduces, the all-reduced statuses and the agreed
    # failure message -- equal to the single-process results bit for bit
    import json
    import socket
    import subprocess
    import sys

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", f"--nproc-per-node={world}",
                          "--master-addr=127.0.0.1", f"--master-port={port}",
                          os.path.join(root, "tools", "multirank_check.py")],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["world"] == world
    assert all(line["tables_bit_identical"]), line
    assert line["error_equal"] and "failed twice" in line["error"], line


def _run_table(table, K, n, seed, rep, first, count):
    import torch

    from paper_1305_6738_b200 import engine

    eng = engine.get_engine()
    dev = f"cuda:{eng.device}"
    ks = torch.empty(count, dtype=torch.float64, device=dev)
    gh = torch.empty(count, dtype=torch.float64, device=dev)
    st = torch.empty(count, dtype=torch.uint8, device=dev)
    eng.run_replicates(table, K, 1.3, n, seed, rep, first, count, ks, gh, st)
    return ks.cpu().numpy(), gh.cpu().numpy(), st.cpu().numpy()


@pytest.mark.parametrize("n", [100, 300])
def test_words_on_cuts_resolve_exactly(zk, n):
    # The small-n kernel classifies each stored word by its top 32 bits against top-32-bit cuts
    # and resolves the undecided words (a cut inside the word's 2^21-wide key range) from their
    # Philox block.  A sampling table with entries placed exactly on, and just beside, chosen
    # words' uniforms -- in the head (value <= 64) and in the tail -- makes those words
    # undecided; every replicate must still equal the oracle on the same table (the row kernel,
    # n = 300, compares full 53-bit keys: the same table checks its cut positions at equality).
    from oracle import port

    from paper_1305_6738_b200 import engine

    seed, rep, count = 11, 0, 64
    cdf = port.sampling_cdf(1.3, None).copy()
    us = [port.stream_uniforms(seed, rep, i, n, False) for i in range(count)]
    ulp = 2.0 ** -53
    edits = {}
    for i, u in enumerate(us):
        v = port.draw(cdf, u)
        mode = i % 4
        head = np.flatnonzero((v >= 2) & (v <= 64))
        tail = np.flatnonzero(v > 70)
        if mode in (0, 1) and head.size:
            j = head[0]
            k = int(v[j]) - 1 if mode == 0 else int(v[j]) - 2  # on the value's own cut / the one below
            edits.setdefault(k, u[j])
        elif mode in (2, 3) and tail.size:
            j = tail[0]
            k = int(v[j]) - 2  # the cut just below the word: inside its 2^-32 range, or on it
            edits.setdefault(k, u[j] - (3 * ulp if mode == 2 else 0.0))
    for k, x in edits.items():
        cdf[k] = x
    cdf = np.maximum.accumulate(cdf)
    assert len(edits) >= count // 2
    eng = engine.get_engine()
    table = engine.DrawTable(eng, cdf)
    try:
        ks, gh, st = _run_table(table, None, n, seed, rep, 0, count)
    finally:
        table.close()
    for i, u in enumerate(us):
        obs = port.draw(cdf, u)
        want_gh = port.fit_exponent(obs, None)
        want_ks = port.ks_distance(obs, want_gh, None)
        assert st[i] == 0
        assert close(gh[i], want_gh), (i, gh[i], want_gh)
        assert close(ks[i], want_ks), (i, ks[i], want_ks)


@pytest.mark.parametrize("K", [None, 20, 1000])
def test_small_n_rows_match_cells(zk, K):
    # n < 128 sweep rows draw each stream once for all cells (lane_row_kernel); with enough
    # replicates a work item covers every cell of the row, with few the cells split into groups
    # -- both must equal each cell run alone, bit for bit
    import torch

    from paper_1305_6738_b200 import engine
    from paper_1305_6738_b200.distribution import Support, sampling_cdf

    eng = engine.get_engine()
    gammas = (0.25, 1.2, 2.0, 3.1) if K else (1.1, 1.6, 2.4, 3.5)
    dev = f"cuda:{eng.device}"
    for n, count in ((10, 300_000), (57, 2_000), (100, 240_000)):
        tables = [eng.table(g, K, lambda g=g: sampling_cdf(g, Support(K))) for g in gammas]
        outs = [(torch.empty(count, dtype=torch.float64, device=dev), torch.empty(count, dtype=torch.float64, device=dev),
                 torch.empty(count, dtype=torch.uint8, device=dev)) for _ in gammas]
        eng.run_cells(tables, K, gammas, n, 4, 1, 17, count, outs)
        for g, o in zip(gammas, outs):
            ks, gh, st = run_cell(K, g, n, 4, 1, 17, count)
            np.testing.assert_array_equal(o[0].cpu().numpy(), ks)
            np.testing.assert_array_equal(o[1].cpu().numpy(), gh)
            np.testing.assert_array_equal(o[2].cpu().numpy(), st)


def test_small_n_warp_tails_match_oracle(zk):
    # n < 128 with a 48-value lane tail buffer (the row's expected tail n P(X > 64) = 39 <= 40):
    # the replicates whose tails are longer are scored by the warp from an exact redraw -- the
    # one lane-kernel path the heavier rows (whole-sample lane buffers) no longer take
    from oracle import port

    gamma, n, seed, count = 1.15, 102, 4, 320
    ks, gh, st = run_cell(None, gamma, n, seed, 0, 0, count)
    cdf = port.sampling_cdf(gamma, None)
    long_tails = 0
    for j in range(count):
        obs = port.draw(cdf, port.stream_uniforms(seed, 0, j, n, False))
        long_tails += int((obs > 64).sum() > 48)
        want_ks, want_gh, want_st = port.replicate(gamma, None, n, seed, j, 0)
        assert st[j] == want_st
        assert close(ks[j], want_ks), (j, ks[j], want_ks)
        assert close(gh[j], want_gh), (j, gh[j], want_gh)
    assert long_tails >= 2
