"""The reference's scalar API on the device: log_mean, mle_gamma, ks_statistic, the series
helpers, fit_samples and fit_bespoke.

Checks restate the reference's own unit tests (pkg/tests/test_estimate.py, test_gof.py,
test_series.py, test_distribution.py; cited per test) against this package, plus batched
parity with the CPU oracle.
"""
import math

import numpy as np
import pytest


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def zk():
    import paper_1305_6738_b200 as zk

    return zk


def draw(zk, gamma, k, n, seed):
    """The reference test helper: sample(model, n, RandomStream.for_replicate(seed, 0, 0))."""
    return zk.sample(zk.ZipfModel(gamma, zk.Support(k)), n, zk.RandomStream.for_replicate(seed, 0, 0))


# ---- log_mean (test_estimate.py:24-47)

def test_log_mean_known_answers(zk, known):
    assert zk.log_mean(zk.Sample([1, 2, 4])) == pytest.approx(math.log(2.0), abs=1e-15)
    assert zk.log_mean(zk.Sample([1] * 10)) == pytest.approx(math.log(2.0) / 10, abs=1e-15)
    assert zk.log_mean(zk.Sample([1])) == pytest.approx(math.log(2.0), abs=1e-15)
    assert zk.log_mean(zk.Sample([2])) == pytest.approx(math.log(2.0), abs=1e-15)
    assert zk.log_mean(zk.Sample([1, 2, 4])) == pytest.approx(known["log_mean_124"], rel=1e-15)
    big = [3, 10**7, 10**9]
    assert zk.log_mean(zk.Sample(big)) == pytest.approx(math.fsum(math.log(v) for v in big) / 3, rel=1e-12)
    obs = draw(zk, 2.0, 1000, 1000, 3).observations
    assert zk.log_mean(zk.Sample(obs)) == pytest.approx(math.fsum(math.log(int(v)) for v in obs) / obs.size,
                                                         rel=1e-12)


# ---- mle_gamma (test_estimate.py:51-172)

def test_mle_known_answers(zk, known):
    K2, K10, K20 = zk.Support.finite(2), zk.Support.finite(10), zk.Support.finite(20)
    assert zk.mle_gamma(zk.Sample([1, 1, 2]), K2) == pytest.approx(1.0, abs=1e-5)
    assert zk.mle_gamma(zk.Sample([2, 2, 2]), K2) == pytest.approx(-1.0, abs=1e-5)
    # equal size and equal log-sum give bitwise-equal estimates
    assert zk.mle_gamma(zk.Sample([2, 2]), K10) == zk.mle_gamma(zk.Sample([4, 1]), K10)
    for key, obs, sup in (("mle_112_K2", [1, 1, 2], K2), ("mle_222_K2", [2, 2, 2], K2),
                          ("mle_short_tail_K20", [17, 19, 20, 20, 16], K20),
                          ("mle_ones10_K20", [1] * 10, K20), ("mle_ones50_inf", [1] * 50, zk.Support.unbounded())):
        assert zk.mle_gamma(zk.Sample(obs), sup) == pytest.approx(known[key], rel=1e-10, abs=1e-12), key
    assert zk.mle_gamma(zk.Sample([17, 19, 20, 20, 16]), K20) < 0.0
    got = zk.mle_gamma(zk.Sample([1] * 50), zk.Support.unbounded())
    assert 1.05 <= got <= 20.0


def test_mle_errors(zk):
    with pytest.raises(zk.NoRootError):
        zk.mle_gamma(zk.Sample([20, 20, 20]), zk.Support.finite(20))
    with pytest.raises(zk.NoRootError):
        zk.mle_gamma(zk.Sample([10**9, 10**9]), zk.Support.unbounded())
    with pytest.raises(ValueError):
        zk.mle_gamma(zk.Sample([1, 25]), zk.Support.finite(20))
    with pytest.raises(ValueError):
        zk.MleSettings(absolute_tolerance=0.0)
    with pytest.raises(ValueError):
        zk.MleSettings(bracket=(1.0, 0.2))


def test_mle_matches_oracle_on_random_samples(zk):
    from oracle import port

    rng = np.random.default_rng(42)
    for _ in range(60):
        k = int(rng.choice([2, 5, 20, 100, 1000]))
        gamma = float(rng.uniform(0.3, 3.5))
        obs = draw(zk, gamma, k, int(rng.integers(5, 200)), int(rng.integers(1 << 30))).observations
        got = zk.mle_gamma(zk.Sample(obs), zk.Support.finite(k))
        want = port.fit_exponent(obs, k)
        assert got == pytest.approx(want, rel=1e-10, abs=1e-12)
    for _ in range(10):
        obs = draw(zk, float(rng.uniform(1.3, 3.5)), None, int(rng.integers(20, 200)),
                   int(rng.integers(1 << 30))).observations
        assert zk.mle_gamma(zk.Sample(obs), zk.Support.unbounded()) == pytest.approx(port.fit_exponent(obs, None),
                                                                                      rel=1e-10)


def test_bisection_and_root_condition(zk):
    from paper_1305_6738_b200.estimate import _bisect, _mean_log_and_slope

    for seed, gamma, k in [(5, 0.8, 20), (6, 2.2, 200)]:
        obs = draw(zk, gamma, k, 100, seed)
        sup = zk.Support.finite(k)
        assert abs(zk.mle_gamma(obs, sup) - _bisect(zk.log_mean(obs), sup, -20.0, 20.0)) < 1e-4
    rng = np.random.default_rng(9)
    for _ in range(10):
        k = int(rng.choice([20, 100, 1000]))
        obs = draw(zk, float(rng.uniform(0.3, 3.5)), k, int(rng.integers(10, 500)), int(rng.integers(1 << 30)))
        got = zk.mle_gamma(obs, zk.Support.finite(k))
        mean, _ = _mean_log_and_slope(got, zk.Support.finite(k))
        assert abs(mean - zk.log_mean(obs)) < 1e-6


def test_custom_settings(zk):
    from oracle import port

    obs = zk.Sample([1, 1, 2, 3, 1, 7])
    s = zk.MleSettings(initial_guess=1.5, absolute_tolerance=1e-9, max_iterations=50, bracket=(-5.0, 9.0))
    got = zk.mle_gamma(obs, zk.Support.finite(50), s)
    assert got == pytest.approx(port.fit_exponent(obs.observations, 50), abs=1e-8)


# ---- ks_statistic (test_gof.py:10-107)

def test_ks_exact_cases(zk, known):
    r = zk.ks_statistic(zk.Sample([1, 1, 2]), zk.ZipfModel(1.0, zk.Support.finite(2)))
    assert r.statistic == 0.0
    r = zk.ks_statistic(zk.Sample([2, 2, 2]), zk.ZipfModel(1.0, zk.Support.finite(2)))
    assert r.statistic == 2.0 / 3.0 and r.argmax_k == 1
    with pytest.raises(ValueError):
        zk.ks_statistic(zk.Sample([1, 30]), zk.ZipfModel(1.0, zk.Support.finite(20)))
    r = zk.ks_statistic(zk.Sample([5000, 6000]), zk.ZipfModel(1.5, zk.Support.unbounded()))
    assert r.statistic == pytest.approx(known["ks_sparse_5000_6000"], rel=1e-10)
    assert r.statistic > 0.9 and r.argmax_k == 4999


def test_ks_matches_oracle_and_brute_force(zk):
    from oracle import port

    rng = np.random.default_rng(123)
    for trial in range(200):
        k = int(rng.choice([2, 5, 10, 20, 50, 1000]))
        obs = draw(zk, float(rng.uniform(0.3, 3.0)), k, int(rng.integers(3, 80)), 1000 + trial).observations
        g = float(rng.uniform(0.3, 3.0))
        got = zk.ks_statistic(zk.Sample(obs), zk.ZipfModel(g, zk.Support.finite(k)))
        want = port.ks_distance(obs, g, k)
        assert got.statistic == pytest.approx(want, rel=1e-10, abs=1e-12)
        # argmax: the smallest k attaining the supremum (brute-force scan, oracles.py:69-91)
        norm = port.norm_constant(g, k)
        F = np.cumsum(np.exp(-g * port.log_table(int(obs.max()))[1:]) * (1.0 / norm))
        E = np.cumsum(np.bincount(obs, minlength=int(obs.max()) + 1)[1:] / obs.size)
        gaps = np.abs(F - E)
        assert abs(gaps[got.argmax_k - 1] - gaps.max()) <= 1e-12


def test_ks_unbounded_heavy_tail_sparse_path(zk):
    from oracle import port

    model = zk.ZipfModel(1.25, zk.Support.unbounded())
    obs = zk.sample(model, 400, zk.RandomStream.for_replicate(77, 0, 0)).observations
    assert int(obs.max()) > 4096
    got = zk.ks_statistic(zk.Sample(obs), model).statistic
    assert got == pytest.approx(port.ks_distance(obs, 1.25, None), rel=1e-10)


# ---- series (test_series.py) and normalization (test_distribution.py:57-81)

def test_series_against_golden(zk, golden):
    for g, want in zip(golden["zeta_grid"][::8], golden["zeta_moments"][::8]):
        np.testing.assert_allclose(zk.zeta_log_moments(float(g)), want, rtol=1e-13)
    for g, want in zip(golden["zeta_grid"][::8], golden["zeta_value"][::8]):
        assert zk.zeta_value(float(g)) == pytest.approx(want, rel=1e-13)
    for g, want in zip(golden["finite_grid"][::8], golden["finite_moments_1000"][::8]):
        np.testing.assert_allclose(zk.finite_log_moments(float(g), 1000), want, rtol=1e-13)
    assert zk.normalization(1.0, zk.Support.finite(2)) == pytest.approx(1.5, abs=1e-12)
    assert zk.normalization(2.0, zk.Support.unbounded()) == pytest.approx(math.pi**2 / 6, abs=1e-9)
    with pytest.raises(ValueError):
        zk.zeta_value(1.0)
    with pytest.raises(ValueError):
        zk.normalization(1.0, zk.Support.unbounded())


# ---- batched fitting and fit --bespoke (row 1)

def test_fit_samples_batched_matches_oracle(zk):
    from oracle import port

    rng = np.random.default_rng(3)
    samples = [draw(zk, 1.8, None, int(rng.integers(5, 400)), s).observations for s in range(300)]
    samples.append(np.array([20, 20, 20]))  # NoRoot on K=inf? no: inf support -> fits; use K below
    fits = zk.fit_samples(samples, zk.Support.unbounded())
    for obs, f in zip(samples, fits):
        assert f.status == 0
        g = port.fit_exponent(obs, None)
        assert f.gamma_hat == pytest.approx(g, rel=1e-10)
        assert f.ks == pytest.approx(port.ks_distance(obs, g, None), rel=1e-10, abs=1e-12)
    bad = zk.fit_samples([np.array([20, 20, 20]), np.array([1, 30]), np.array([1, 2, 3])], zk.Support.finite(20))
    assert [f.status for f in bad] == [2, 3, 0]


def test_fit_bespoke(zk):
    obs = draw(zk, 2.0, None, 500, 11)
    report = zk.fit_bespoke(obs, zk.Support.unbounded(), base_seed=5, replicates=20000, repetitions=2)
    assert report.n == 500 and 1.8 < report.gamma_hat < 2.2
    levels = [v.level for v in report.verdicts]
    assert levels == list(zk.DEFAULT_LEVELS)
    cut = [v.cutoff for v in report.verdicts]
    assert all(0 < c < 1 for c in cut) and cut == sorted(cut)
    cfg = zk.SimulationConfig(n=500, support=zk.Support.unbounded(), gamma=report.gamma_hat, base_seed=5,
                              replicates=20000, repetitions=2)
    assert [c for _, c in zk.run_simulation(cfg)] == cut


@pytest.mark.parametrize("key", [5, 0, [1, 2, 3, 4, 5], [7], [], 2**100, [2**64 - 1, 3, 2**32 + 7], [1, 2, 2**64]])
def test_random_stream_any_seedsequence_key(zk, key):
    # RandomStream takes whatever SeedSequence takes (distribution.py:173-180); continuing calls
    # continue the stream
    want = 1.0 - np.random.Generator(np.random.Philox(np.random.SeedSequence(key))).random(23)
    s = zk.RandomStream(key)
    got = np.concatenate([s.uniforms(5), s.uniforms(18)])
    assert got.tobytes() == want.tobytes()


def test_random_stream_rejects_what_seedsequence_rejects(zk):
    with pytest.raises(ValueError):
        zk.RandomStream([-1, 2, 3])
