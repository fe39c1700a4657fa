"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's random streams.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this module.  The product (``paper_1305_6738_b200``) never does.

The reference keys one stream per replicate as

    np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, rep, idx])))

(``pkg/src/zipfks/distribution.py:178-184``) and draws ``1 - Generator.random(n)``
(``distribution.py:186-187``).  The arithmetic lives in the third-party
dependency numpy (``pkg/pyproject.toml:10`` pins ``numpy>=1.24``; this image
ships 2.3.5), which is not vendored under ``/root/reference``.  Its published
algorithms are restated here:

* ``SeedSequence``: uint32 hash-mix of the entropy words into a 4-word pool,
  then ``generate_state(2, uint64)`` for the Philox key (numpy
  ``random/bit_generator.pyx``: ``_coerce_to_uint32_array``, ``mix_entropy``,
  ``generate_state``).
* ``Philox4x64-10`` (Salmon et al., SC'11 / Random123), counter incremented
  *before* each 4-word block, so draw ``j`` is word ``j % 4`` of the block at
  counter ``[1 + j // 4, 0, 0, 0]`` (numpy ``random/src/philox/philox.h``).
* ``Generator.random``: ``(x >> 11) * 2**-53``.

Parity pinning: ``tests/test_oracle_rng.py`` checks every function here against
numpy's own implementation and against golden vectors in ``tests/golden``.
"""
from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF

# SeedSequence constants (numpy bit_generator.pyx)
_INIT_A = 0x43B0D7E5
_MULT_A = 0x931E8875
_INIT_B = 0x8B51F9DD
_MULT_B = 0x58F38DED
_MIX_L = 0xCA01F9DD
_MIX_R = 0x4973F715
_POOL = 4

# Philox4x64 constants (Random123)
PHILOX_M0 = 0xD2E7470EE14C6C93
PHILOX_M1 = 0xCA5A826395121157
PHILOX_W0 = 0x9E3779B97F4A7C15
PHILOX_W1 = 0xBB67AE8584CAA73B
PHILOX_ROUNDS = 10


def int_words(value: int) -> list[int]:
    """Little-endian uint32 words of a non-negative int; 0 -> [0]."""
    if value < 0:
        raise ValueError("entropy must be non-negative")
    if value == 0:
        return [0]
    words = []
    while value:
        words.append(value & M32)
        value >>= 32
    return words


def entropy_words(key: list[int]) -> list[int]:
    out: list[int] = []
    for item in key:
        out.extend(int_words(int(item)))
    return out


def seedseq_pool(words: list[int]) -> list[int]:
    """The 4-word entropy pool SeedSequence builds from its entropy words."""
    h = _INIT_A

    def hashmix(v: int) -> int:
        nonlocal h
        v = (v ^ h) & M32
        h = (h * _MULT_A) & M32
        v = (v * h) & M32
        return v ^ (v >> 16)

    def mix(x: int, y: int) -> int:
        r = (_MIX_L * x - _MIX_R * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(words[i] if i < len(words) else 0) for i in range(_POOL)]
    for src in range(_POOL):
        for dst in range(_POOL):
            if src != dst:
                pool[dst] = mix(pool[dst], hashmix(pool[src]))
    for src in range(_POOL, len(words)):
        for dst in range(_POOL):
            pool[dst] = mix(pool[dst], hashmix(words[src]))
    return pool


def seedseq_state32(pool: list[int], n_words: int) -> list[int]:
    h = _INIT_B
    out = []
    for i in range(n_words):
        v = (pool[i % _POOL] ^ h) & M32
        h = (h * _MULT_B) & M32
        v = (v * h) & M32
        out.append(v ^ (v >> 16))
    return out


def philox_key(seed: int, repetition: int, index: int) -> tuple[int, int]:
    """The 128-bit Philox key numpy derives for stream ``(seed, rep, idx)``."""
    s = seedseq_state32(seedseq_pool(entropy_words([seed, repetition, index])), 4)
    return s[0] | (s[1] << 32), s[2] | (s[3] << 32)


def _mulhilo(a: int, b: int) -> tuple[int, int]:
    p = a * b
    return p >> 64, p & M64


def philox_block(counter: tuple[int, int, int, int], key: tuple[int, int]) -> list[int]:
    """One Philox4x64-10 block (scalar, exact Python ints)."""
    c0, c1, c2, c3 = counter
    k0, k1 = key
    for r in range(PHILOX_ROUNDS):
        if r:
            k0 = (k0 + PHILOX_W0) & M64
            k1 = (k1 + PHILOX_W1) & M64
        hi0, lo0 = _mulhilo(PHILOX_M0, c0)
        hi1, lo1 = _mulhilo(PHILOX_M1, c2)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return [c0, c1, c2, c3]


def _mulhilo_vec(a: int, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Vectorised 64x64->128 multiply of a constant by a uint64 array."""
    a_lo, a_hi = np.uint64(a & M32), np.uint64(a >> 32)
    b_lo = b & np.uint64(M32)
    b_hi = b >> np.uint64(32)
    s32 = np.uint64(32)
    t = a_lo * b_lo
    u = a_hi * b_lo + (t >> s32)
    w = a_lo * b_hi + (u & np.uint64(M32))
    hi = a_hi * b_hi + (u >> s32) + (w >> s32)
    return hi, np.uint64(a) * b


def philox_blocks(first_counter: int, count: int, key: tuple[int, int]) -> np.ndarray:
    """``count`` consecutive blocks with counter word 0 = first..first+count-1.

    Returns uint64[count, 4].  Counters here never carry into word 1 (the
    reference draws at most a few million values per stream).
    """
    with np.errstate(over="ignore"):
        c0 = np.arange(first_counter, first_counter + count, dtype=np.uint64)
        c1 = np.zeros(count, dtype=np.uint64)
        c2 = np.zeros(count, dtype=np.uint64)
        c3 = np.zeros(count, dtype=np.uint64)
        k0, k1 = key
        for r in range(PHILOX_ROUNDS):
            if r:
                k0 = (k0 + PHILOX_W0) & M64
                k1 = (k1 + PHILOX_W1) & M64
            hi0, lo0 = _mulhilo_vec(PHILOX_M0, c0)
            hi1, lo1 = _mulhilo_vec(PHILOX_M1, c2)
            c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
    return np.stack([c0, c1, c2, c3], axis=1)


def raw_words(seed: int, repetition: int, index: int, count: int) -> np.ndarray:
    """First ``count`` uint64 outputs of the stream (block 0 at counter 1)."""
    key = philox_key(seed, repetition, index)
    blocks = philox_blocks(1, (count + 3) // 4, key)
    return blocks.reshape(-1)[:count]


def uniforms(seed: int, repetition: int, index: int, count: int) -> np.ndarray:
    """``RandomStream.for_replicate(seed, rep, idx).uniforms(count)``: values in (0, 1]."""
    x = raw_words(seed, repetition, index, count)
    return 1.0 - (x >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def numpy_uniforms(seed: int, repetition: int, index: int, count: int) -> np.ndarray:
    """The same stream drawn through numpy itself (the reference's dependency)."""
    gen = np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, repetition, index])))
    return 1.0 - gen.random(count)
