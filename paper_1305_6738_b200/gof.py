"""Discrete Kolmogorov-Smirnov statistic and cutoff verdicts (reference ``gof.py``), on the device.

``ks_statistic`` and the batched ``fit_samples`` run ``zks_fit_samples`` (one warp per sample):
the dense head / endpoint scan of csrc/zks_ks.cuh in its reference-exact form (E = C/n, F as
the running sum of k^-g/norm), which also returns the smallest k attaining the supremum.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .distribution import Sample, Support, ZipfModel


@dataclass(frozen=True)
class KsResult:
    """Supremum gap and the (smallest) support point where it is attained (gof.py:23-28)."""

    statistic: float
    argmax_k: int


@dataclass(frozen=True)
class Verdict:
    """Comparison of a statistic against one tabulated cutoff level (gof.py:31-37)."""

    level: float
    cutoff: float
    rejected: bool


def judge(statistic: float, cutoff: float, level: float) -> Verdict:
    """Reject only when the statistic strictly exceeds the cutoff (gof.py:40-46)."""
    if not 0.0 <= statistic <= 1.0:
        raise ValueError(f"statistic must lie in [0, 1], got {statistic}")
    if not 0.0 <= cutoff <= 1.0:
        raise ValueError(f"cutoff must lie in [0, 1], got {cutoff}")
    return Verdict(level=level, cutoff=cutoff, rejected=statistic > cutoff)


def fit_samples_device(samples, support: Support | None, mode: int, settings=None, gamma=None, norm=None,
                       single: bool = False) -> dict:
    """Run zks_fit_samples over a list of integer arrays; returns numpy arrays."""
    import torch

    from .engine import get_engine

    eng = get_engine()
    arrays = [np.asarray(s, dtype=np.int64).ravel() for s in samples]
    offsets = np.zeros(len(arrays) + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([a.size for a in arrays])
    flat = np.concatenate(arrays) if arrays else np.zeros(0, dtype=np.int64)
    dev = f"cuda:{eng.device}"
    values = torch.from_numpy(flat).to(dev) if flat.size else torch.zeros(1, dtype=torch.int64, device=dev)
    offs = torch.from_numpy(offsets).to(dev)
    g_in = None if gamma is None else torch.as_tensor(np.broadcast_to(np.asarray(gamma, dtype=np.float64),
                                                                      (len(arrays),)).copy()).to(dev)
    n_in = None if norm is None else torch.as_tensor(np.broadcast_to(np.asarray(norm, dtype=np.float64),
                                                                     (len(arrays),)).copy()).to(dev)
    k = None if support is None else support.k
    out = eng.fit_samples(k, values, offs, mode, settings, g_in, n_in)
    return {key: v.cpu().numpy() for key, v in out.items()}


def ks_statistic(sample: Sample, model: ZipfModel) -> KsResult:
    """Largest |fitted cdf - empirical cdf| over 1..max(observations) (gof.py:49-57)."""
    if not model.support.contains(sample.observations):
        raise ValueError(f"observations exceed the support 1..{model.support}")
    r = fit_samples_device([sample.observations], model.support, _native.FIT_KS, None, model.gamma, model.norm,
                           single=True)
    if int(r["status"][0]) != _native.SAMPLE_OK:
        raise ValueError(f"observations exceed the support 1..{model.support}")
    return KsResult(statistic=float(r["ks"][0]), argmax_k=int(r["argmax"][0]))


def _ks_sparse(obs, model: ZipfModel, kmax: int) -> KsResult:
    """Endpoint evaluation (gof.py:71-92); the device scan uses endpoints above k = 64 always."""
    return ks_statistic(Sample(np.asarray(obs)), model)


def _ks_dense(obs, model: ZipfModel, kmax: int) -> KsResult:
    return ks_statistic(Sample(np.asarray(obs)), model)


@dataclass(frozen=True)
class SampleFit:
    """Batched fit of one user sample: exponent, KS against the refit, argmax, mean log."""

    gamma_hat: float
    ks: float
    argmax_k: int
    log_mean: float
    status: int


def fit_samples(samples, support: Support, settings=None) -> list[SampleFit]:
    """mle_gamma then ks_statistic against the refitted model for many samples in one launch
    (SURVEY §8f row 3).  NoRootError / out-of-support samples come back with status 2 / 3."""
    from .estimate import DEFAULT_SETTINGS

    s = None if settings is None or settings == DEFAULT_SETTINGS else settings
    r = fit_samples_device(samples, support, _native.FIT_EXPONENT | _native.FIT_KS, s)
    return [SampleFit(float(g), float(k), int(a), float(m), int(st))
            for g, k, a, m, st in zip(r["gamma"], r["ks"], r["argmax"], r["log_mean"], r["status"])]
