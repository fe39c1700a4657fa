"""Zipf model types and the device-backed sampler (reference ``distribution.py``).

Host side keeps only what must be bit-exact with the reference and is built once per
model: the sampling CDF (``ZipfModel._sampling_cdf``, distribution.py:99-105), formed with
the same numpy calls so that device draws reproduce the reference's integers exactly.
Streams and draws run on the GPU (``zks_stream_uniforms``, ``zks_draw``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .series import MAX_FINITE_SUPPORT, natural_logs

MIN_UNBOUNDED_GAMMA = 1.05        # distribution.py:19
UNBOUNDED_SAMPLE_LIMIT = 65535    # distribution.py:26
_PARTIAL_SEAM = 4096              # distribution.py:30


@dataclass(frozen=True)
class Support:
    """1..k when ``k`` is an int, all positive integers when ``k`` is None (distribution.py:33-68)."""

    k: int | None

    def __post_init__(self) -> None:
        if self.k is None:
            return
        if isinstance(self.k, bool) or not isinstance(self.k, (int, np.integer)):
            raise ValueError(f"finite support bound must be an integer, got {self.k!r}")
        if not 2 <= self.k <= MAX_FINITE_SUPPORT:
            raise ValueError(f"finite support bound must be in [2, {MAX_FINITE_SUPPORT}], got {self.k}")
        object.__setattr__(self, "k", int(self.k))

    @classmethod
    def finite(cls, k: int) -> "Support":
        return cls(k=k)

    @classmethod
    def unbounded(cls) -> "Support":
        return cls(k=None)

    @property
    def is_finite(self) -> bool:
        return self.k is not None

    @property
    def draw_limit(self) -> int:
        """Length L of the sampling table: K, or 65535 for the unbounded model."""
        return self.k if self.k is not None else UNBOUNDED_SAMPLE_LIMIT

    def contains(self, values: np.ndarray) -> bool:
        values = np.asarray(values)
        if values.size == 0:
            return True
        return int(values.min()) >= 1 and (self.k is None or int(values.max()) <= self.k)

    def __str__(self) -> str:
        return "inf" if self.k is None else str(self.k)


def validate_pair(gamma: float, support: Support) -> None:
    """Host-side check of an (exponent, support) pair, as normalization() validates it
    (distribution.py:71-85); used by SimulationConfig (montecarlo.py:72) without a device."""
    if not math.isfinite(gamma):
        raise ValueError(f"exponent must be finite, got {gamma}")
    if support.is_finite:
        # the finite normaliser overflows iff its largest term K^-gamma (gamma < 0) is huge
        with np.errstate(over="ignore"):
            total = float(np.exp(-gamma * natural_logs(support.k)[1:]).sum())
        if not math.isfinite(total):
            raise ValueError(f"normalizer overflows at gamma={gamma} with K={support.k}")
    elif gamma < MIN_UNBOUNDED_GAMMA:
        raise ValueError(f"unbounded support requires gamma >= {MIN_UNBOUNDED_GAMMA}, got {gamma}")


def normalization(gamma: float, support: Support) -> float:
    """Sum of k^-gamma over the support (distribution.py:71-85), formed on the device:
    the finite power sum, or the zeta series with its Euler-Maclaurin tail (series.py:126-138)."""
    validate_pair(gamma, support)
    from .engine import get_engine

    return get_engine().normaliser(gamma, support.k)


def sampling_cdf(gamma: float, support: Support) -> np.ndarray:
    """cumsum(w * (1 / sum(w))), w_k = exp(-gamma ln k), k = 1..L — bit-exact with the reference."""
    w = np.exp(-gamma * natural_logs(support.draw_limit)[1:])
    return np.cumsum(w * (1.0 / w.sum()))


@dataclass(frozen=True)
class ZipfModel:
    """p(k) = k^-gamma / norm over the declared support (distribution.py:88-121)."""

    gamma: float
    support: Support
    _norm: list = field(default_factory=list, init=False, compare=False, repr=False)

    def __post_init__(self) -> None:
        validate_pair(self.gamma, self.support)

    @property
    def norm(self) -> float:
        """Normaliser, computed on the device on first use."""
        if not self._norm:
            self._norm.append(normalization(self.gamma, self.support))
        return self._norm[0]

    @property
    def _sampling_cdf(self) -> np.ndarray:
        return sampling_cdf(self.gamma, self.support)

    def _sample_limit(self) -> int:
        return self.support.draw_limit

    def device_table(self):
        """The engine's cached device copy of this model's sampling table."""
        from .engine import get_engine

        return get_engine().table(self.gamma, self.support.k, lambda: sampling_cdf(self.gamma, self.support))


@dataclass(frozen=True)
class Sample:
    """Ordered collection of positive integer observations (distribution.py:124-146)."""

    observations: np.ndarray

    def __post_init__(self) -> None:
        values = np.asarray(self.observations)
        if values.ndim != 1 or values.size == 0:
            raise ValueError("a sample must be a nonempty one-dimensional collection")
        if np.issubdtype(values.dtype, np.integer):
            values = values.astype(np.int64, copy=False)
        else:
            if not np.all(values == np.floor(values)):
                raise ValueError("observations must be integers")
            values = values.astype(np.int64)
        if values.min() < 1:
            raise ValueError("observations must be positive integers")
        object.__setattr__(self, "observations", values)

    @property
    def n(self) -> int:
        return int(self.observations.size)


def _check_in_support(model: "ZipfModel", k) -> int:
    if not isinstance(k, (int, np.integer)) or isinstance(k, bool):
        raise ValueError(f"support point must be an integer, got {k!r}")
    k = int(k)
    if k < 1 or (model.support.is_finite and k > model.support.k):
        raise ValueError(f"value {k} lies outside the support 1..{model.support}")
    return k


def pmf(model: "ZipfModel", k) -> float:
    """P(X = k) = k^-gamma / norm (distribution.py:158-161); the normaliser from the device."""
    k = _check_in_support(model, k)
    return math.exp(-model.gamma * math.log(k)) * (1.0 / model.norm)


def cdf(model: "ZipfModel", k) -> float:
    """P(X <= k) (distribution.py:164-170), on the device: the power sum over 1..k (the finite
    normaliser at support k) over the model's normaliser; beyond the partial-table seam of the
    unbounded model, (norm - tail_mass(gamma, k + 1)) / norm as the reference forms it."""
    k = _check_in_support(model, k)
    from .engine import get_engine

    if model.support.is_finite or k <= _PARTIAL_SEAM:
        head = 1.0 if k == 1 else get_engine().normaliser(model.gamma, k)
        return float(head / model.norm)
    from .series import tail_mass

    return float((model.norm - tail_mass(model.gamma, k + 1)) / model.norm)


class RandomStream:
    """Deterministic uniform(0, 1] stream keyed ``[seed, repetition, index]``, drawn on the GPU.

    Bit-exact with ``numpy.random.Generator(Philox(SeedSequence(key))).random`` as the
    reference uses it (distribution.py:173-187).  Successive ``uniforms`` calls continue
    the stream.  Replicate keys ``[base_seed, repetition, index]`` are hashed on the device
    (the hot path's derivation); any other SeedSequence entropy the reference accepts (an int,
    a sequence of any length) gets its Philox key from numpy's SeedSequence on the host -- the
    reference's own dependency -- and its uniforms from the device.
    """

    __slots__ = ("_key", "_philox", "_offset")

    def __init__(self, key) -> None:
        words = [int(key)] if isinstance(key, (int, np.integer)) else [int(x) for x in key]
        self._philox = None
        if len(words) == 3 and all(0 <= x < 1 << 64 for x in words):
            self._key = tuple(words)
        else:
            k = np.random.SeedSequence(key).generate_state(2, np.uint64)  # raises as the reference does
            self._key = None
            self._philox = (int(k[0]), int(k[1]))
        self._offset = 0

    @classmethod
    def for_replicate(cls, base_seed: int, repetition: int, index: int) -> "RandomStream":
        return cls([int(base_seed), int(repetition), int(index)])

    def uniforms(self, count: int) -> np.ndarray:
        import torch

        from .engine import get_engine

        eng = get_engine()
        total = self._offset + int(count)
        buf = torch.empty(max(total, 1), dtype=torch.float64, device=f"cuda:{eng.device}")
        if self._philox is not None:
            eng.uniforms_key(*self._philox, total, buf)
        else:
            eng.uniforms(*self._key, total, buf)
        out = buf[self._offset : total].cpu().numpy()
        self._offset = total
        return out


def sample(model: ZipfModel, n: int, stream) -> Sample:
    """n inverse-transform draws: the smallest k with cdf(k) >= u (distribution.py:190-201).

    ``stream`` is anything with ``uniforms(count)`` (the reference's duck type, e.g. its
    tests' FixedStream); the lookup runs on the device.
    """
    import torch

    if n < 1:
        raise ValueError(f"sample size must be >= 1, got {n}")
    from .engine import get_engine

    eng = get_engine()
    u = np.ascontiguousarray(stream.uniforms(n), dtype=np.float64)
    dev = f"cuda:{eng.device}"
    u_dev = torch.from_numpy(u).to(dev)
    out = torch.empty(u.size, dtype=torch.int64, device=dev)
    eng.draw(model.device_table(), u_dev, out)
    return Sample(out.cpu().numpy())
