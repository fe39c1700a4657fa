"""Host-side argument handling of the drop-in API, on CPU (no device call is reached).

Mirrors the reference's validation tests — pkg/tests/test_montecarlo.py:36-57, 92-93, 126-127,
240-268 and pkg/tests/test_distribution.py:36-41, 74-81, 143-151 — against this package's
names: every error must be raised before the engine is touched, with the reference's
exception type.
"""
import os
from decimal import ROUND_FLOOR, Decimal

import numpy as np
import pytest

import paper_1305_6738_b200 as zk
from paper_1305_6738_b200.montecarlo import quantile_ranks, resolve_workers


def config(**overrides):
    base = dict(n=50, support=zk.Support.finite(20), gamma=1.5, base_seed=101, replicates=400, repetitions=2)
    base.update(overrides)
    return zk.SimulationConfig(**base)


def test_support_bounds():
    assert zk.Support.finite(2).k == 2
    assert zk.Support.finite(32766).k == 32766
    assert zk.Support.unbounded().k is None
    for bad in (1, 0, -5, 32767, 2.5, True):
        with pytest.raises(ValueError):
            zk.Support.finite(bad)


def test_config_validation():
    with pytest.raises(ValueError):
        config(replicates=99)
    with pytest.raises(ValueError):
        config(n=0)
    with pytest.raises(ValueError):
        config(repetitions=0)
    for levels in ((0.9, 0.9), (0.9, 0.5), (0.0, 0.9), (0.9, 1.0), ()):
        with pytest.raises(ValueError):
            config(quantiles=levels)
    with pytest.raises(ValueError):
        config(support=zk.Support.unbounded(), gamma=1.0)
    with pytest.raises(ValueError):
        config(gamma=float("nan"))
    with pytest.raises(ValueError):
        config(support=zk.Support.finite(32766), gamma=-100.0)  # normaliser overflows
    with pytest.raises(ValueError):
        config(base_seed=-1)
    with pytest.raises(ValueError):
        config(base_seed=1 << 64)
    cfg = config(base_seed=(1 << 64) - 1, quantiles=[0.5, 0.9])
    assert cfg.quantiles == (0.5, 0.9)
    assert config(support=zk.Support.unbounded(), gamma=zk.MIN_UNBOUNDED_GAMMA).gamma == zk.MIN_UNBOUNDED_GAMMA


def test_normalization_rejects_before_device():
    with pytest.raises(ValueError):
        zk.normalization(1.0, zk.Support.unbounded())
    with pytest.raises(ValueError):
        zk.normalization(zk.MIN_UNBOUNDED_GAMMA - 0.01, zk.Support.unbounded())
    with pytest.raises(ValueError):
        zk.normalization(float("nan"), zk.Support.finite(10))
    with pytest.raises(ValueError):
        zk.ZipfModel(1.0, zk.Support.unbounded())


def test_sample_validation():
    with pytest.raises(ValueError):
        zk.Sample(np.array([], dtype=np.int64))
    with pytest.raises(ValueError):
        zk.Sample(np.array([1, 0]))
    with pytest.raises(ValueError):
        zk.Sample(np.array([1.5]))
    with pytest.raises(ValueError):
        zk.Sample(np.ones((2, 2), dtype=np.int64))
    s = zk.Sample(np.array([3.0, 1.0]))
    assert s.n == 2 and s.observations.dtype == np.int64


@pytest.mark.parametrize("count", [1, 7, 100, 400, 50000, 123457])
def test_quantile_ranks_follow_the_decimal_rule(count):
    levels = zk.DEFAULT_LEVELS + (0.1, 0.333, 0.999)
    levels = tuple(sorted(set(levels)))
    want = [int((Decimal(str(q)) * count).to_integral_value(rounding=ROUND_FLOOR)) for q in levels]
    assert quantile_ranks(count, levels) == want


def test_order_quantiles_argument_errors_precede_the_device():
    with pytest.raises(ValueError):
        zk.order_quantiles([], [0.9])
    with pytest.raises(ValueError):
        zk.order_quantiles([0.1, 0.2], [0.9, 0.5])
    with pytest.raises(ValueError):
        zk.order_quantiles([0.1, 0.2], [])


def test_replicate_index_range():
    with pytest.raises(ValueError):
        zk.run_replicate(config(), 400)
    with pytest.raises(ValueError):
        zk.run_replicate(config(), -1)


def test_workers_and_grid_validation():
    assert resolve_workers(3) == 3
    assert resolve_workers(None) >= 1
    with pytest.raises(ValueError):
        resolve_workers(0)
    with pytest.raises(ValueError):
        zk.build_table(ns=(), gammas=(1.0,), support=zk.Support.finite(20), base_seed=1)
    with pytest.raises(ValueError):
        zk.build_table(ns=(10,), gammas=(), support=zk.Support.finite(20), base_seed=1)
    with pytest.raises(ValueError):
        zk.build_table(ns=(10,), gammas=(1.0,), support=zk.Support.finite(20), base_seed=1, workers=0)


def test_cutoff_table_lookup_window():
    row = (0.05, 0.06, 0.07, 0.08)
    table = zk.CutoffTable(support=zk.Support.finite(20), levels=zk.DEFAULT_LEVELS, gammas=(1.0, 1.5),
                           ns=(20, 50), cells={(g, n): row for g in (1.0, 1.5) for n in (20, 50)},
                           replicates=400, repetitions=2, base_seed=101)
    assert table.cutoffs_for(1.5004, 50) == row
    assert table.cutoff(1.4996, 50, 0.9) == row[0]
    with pytest.raises(zk.CutoffLookupError):
        table.cutoffs_for(1.4, 50)  # between grid points
    with pytest.raises(zk.CutoffLookupError):
        table.cutoffs_for(1.5, 30)  # sample size not tabulated
    with pytest.raises(zk.CutoffLookupError):
        table.cutoff(1.5, 50, 0.8)  # level not tabulated
    assert issubclass(zk.CutoffLookupError, LookupError)
    assert issubclass(zk.SimulationError, RuntimeError)


def _golden_fit():
    import json

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fit")
    with open(os.path.join(here, "fit.json")) as fh:
        return here, json.load(fh)


def test_fit_reports_format_like_the_reference():
    # the reference's machine block carries full-precision values: rebuilt into a FitReport, both
    # formats reproduce the reference's own stdout of that run (reporting.py:27-62)
    from paper_1305_6738_b200.bespoke import FitReport, format_human, format_machine
    from paper_1305_6738_b200.gof import Verdict

    _, cases = _golden_fit()
    block = dict(line.split("=", 1) for line in cases["inf_bespoke_machine"]["stdout"].strip().splitlines())
    levels = (0.9, 0.95, 0.99, 0.999)
    tags = ("90", "95", "99", "999")
    report = FitReport(n=int(block["n"]), support=zk.Support.unbounded(), gamma_hat=float(block["gamma_hat"]),
                       ks=float(block["ks"]), ks_argmax=int(block["ks_argmax"]), cutoff_source=block["cutoff_source"],
                       verdicts=tuple(Verdict(q, float(block[f"cutoff_q{t}"]), block[f"rejected_q{t}"] == "true")
                                      for q, t in zip(levels, tags)))
    assert format_machine(report) + "\n" == cases["inf_bespoke_machine"]["stdout"]
    assert format_human(report) + "\n" == cases["inf_bespoke_human"]["stdout"]


def test_observation_files_parse_like_the_reference(tmp_path):
    from paper_1305_6738_b200.bespoke import ObservationParseError, parse_observations, write_observations

    here, cases = _golden_fit()
    with pytest.raises(ObservationParseError) as err:
        parse_observations("bad_token.txt" if os.getcwd() == here else os.path.join(here, "bad_token.txt"))
    assert str(err.value).endswith(cases["bad_token"]["stderr"].strip().split("bad_token.txt")[1])
    s = parse_observations(os.path.join(here, "inf_g22_n300.txt"))
    assert s.n == 300
    write_observations(s, tmp_path / "o.txt")
    assert (tmp_path / "o.txt").read_text() == open(os.path.join(here, "inf_g22_n300.txt")).read()
    (tmp_path / "empty.txt").write_text("  \n")
    with pytest.raises(ObservationParseError, match="no observations found"):
        parse_observations(tmp_path / "empty.txt")
