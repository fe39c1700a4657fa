"""Pin the CPU oracle (oracle/port.py) against golden vectors produced by the reference itself.

The port restates the reference with the same numpy primitives in the same order, so it
must reproduce the reference BIT-FOR-BIT on identical inputs (tests/golden/make_golden.py).
"""
import hashlib
import math

import numpy as np
import pytest

from oracle import port


def cells(golden):
    for ci, row in enumerate(golden["cells"]):
        k, gamma, n, seed, rep, count = row
        yield ci, (None if k == 0 else int(k)), float(gamma), int(n), int(seed), int(rep), int(count)


def test_log_table_matches_reference(golden):
    logs = port.log_table(65536)
    assert hashlib.sha256(logs.tobytes()).digest() == golden["logs_65536_sha256"].tobytes()


def test_sampling_cdf_bitwise(golden):
    for ci, K, gamma, *_ in cells(golden):
        if gamma < 0:
            continue
        cdf = port.sampling_cdf(gamma, K)
        assert cdf[:64].tobytes() == golden[f"cell{ci}_cdf_head"][: cdf[:64].size].tobytes()
        assert cdf[-8:].tobytes() == golden[f"cell{ci}_cdf_tail"].tobytes()


def test_samples_bitwise(golden):
    for ci, K, gamma, n, seed, rep, count in cells(golden):
        if n > 20000:
            continue
        cdf = port.sampling_cdf(gamma, K)
        for idx in range(min(count, 4)):
            obs = port.draw(cdf, port.stream_uniforms(seed, rep, idx, n, restated=True))
            np.testing.assert_array_equal(obs, golden[f"cell{ci}_sample{idx}"])


def test_replicates_bitwise(golden):
    for ci, K, gamma, n, seed, rep, count in cells(golden):
        if n > 20000:
            count = min(count, 2)
        want_ks = golden[f"cell{ci}_ks"]
        want_gh = golden[f"cell{ci}_gamma_hat"]
        want_st = golden[f"cell{ci}_status"]
        for idx in range(count):
            try:
                ks, gh, st = port.replicate(gamma, K, n, seed, idx, rep)
            except port.FailedTwice:
                assert want_st[idx] == 2
                continue
            assert st == want_st[idx]
            assert ks == want_ks[idx], (ci, idx)
            assert gh == want_gh[idx], (ci, idx)


def test_failure_message_format():
    with pytest.raises(port.FailedTwice, match=r"gamma=-30.0, n=3, support=20\) failed twice"):
        for idx in range(16):
            port.replicate(-30.0, 20, 3, 101, idx, 0)


def test_simulations_bitwise(golden):
    for si, row in enumerate(golden["sims"]):
        k, gamma, n, seed, reps_r, reps = row
        K = None if k == 0 else int(k)
        got = port.simulate(float(gamma), K, int(n), int(seed), int(reps_r), int(reps))
        assert [c for _, c in got] == list(golden[f"sim{si}_cutoffs"])


def test_series_tables(golden):
    for g, want in zip(golden["zeta_grid"], golden["zeta_moments"]):
        assert port.zeta_moments(float(g)) == tuple(want)
    for g, want in zip(golden["zeta_grid"], golden["zeta_value"]):
        assert port.zeta_norm(float(g)) == want
    for g, want in zip(golden["finite_grid"], golden["finite_moments_1000"]):
        assert port.finite_moments(float(g), 1000) == tuple(want)


def test_known_answers(known):
    assert port.norm_constant(1.0, 2) == known["normalization_1_K2"]
    assert port.fit_exponent(np.array([1, 1, 2]), 2) == known["mle_112_K2"]
    assert port.fit_exponent(np.array([2, 2, 2]), 2) == known["mle_222_K2"]
    assert port.fit_exponent(np.array([2, 2]), 10) == port.fit_exponent(np.array([4, 1]), 10)
    assert port.fit_exponent(np.array([17, 19, 20, 20, 16]), 20) == known["mle_short_tail_K20"]
    assert port.fit_exponent(np.ones(50, dtype=np.int64), None) == known["mle_ones50_inf"]
    assert port.ks_distance(np.array([1, 1, 2]), 1.0, 2) == known["ks_112_K2"] == 0.0
    assert port.ks_distance(np.array([2, 2, 2]), 1.0, 2) == known["ks_222_K2"] == 2.0 / 3.0
    assert port.ks_distance(np.array([5000, 6000]), 1.5, None) == known["ks_sparse_5000_6000"]
    assert port.mean_log(np.array([1, 2, 4])) == known["log_mean_124"]
    assert port.mean_log(np.ones(10, dtype=np.int64)) == known["log_mean_ones10"]
    assert port.order_quantiles(np.arange(100) / 100.0, [0.29]) == known["quantiles_r100_q029"]
    with pytest.raises(port.NoRoot):
        port.fit_exponent(np.array([20, 20, 20]), 20)


def test_quantile_ranks_decimal_rule():
    assert port.quantile_ranks(100, [0.29]) == [29]
    assert port.quantile_ranks(50000, port.LEVELS) == [45000, 47500, 49500, 49950]
    assert math.floor(100 * 0.29) == 28  # the binary product would be wrong
