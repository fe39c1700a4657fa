"""Pin the oracle's stream restatement (oracle/rng.py) against numpy and the golden vectors."""
import numpy as np
import pytest

from oracle import rng


def stream_keys(golden):
    i = 0
    while f"stream{i}_key" in golden:
        yield i, tuple(int(x) for x in golden[f"stream{i}_key"])
        i += 1


def test_entropy_words():
    assert rng.int_words(0) == [0]
    assert rng.int_words(5) == [5]
    assert rng.int_words(1 << 32) == [0, 1]
    assert rng.int_words((1 << 64) - 1) == [0xFFFFFFFF, 0xFFFFFFFF]


def test_philox_key_matches_golden(golden):
    for i, key in stream_keys(golden):
        assert rng.philox_key(*key) == tuple(int(x) for x in golden[f"stream{i}_philox_key"])


def test_raw_words_match_golden(golden):
    for i, key in stream_keys(golden):
        np.testing.assert_array_equal(rng.raw_words(*key, 9), golden[f"stream{i}_raw"])


def test_uniforms_match_golden_bitwise(golden):
    for i, key in stream_keys(golden):
        got = rng.uniforms(*key, 37)
        assert got.tobytes() == golden[f"stream{i}_u"].tobytes()


@pytest.mark.parametrize("key", [(1, 0, 0), (3, 2, 2**33 + 5), (2**63, 0, 7), (0, 2**40, 0)])
def test_uniforms_match_numpy(key):
    assert rng.uniforms(*key, 1001).tobytes() == rng.numpy_uniforms(*key, 1001).tobytes()


def test_scalar_and_vector_philox_agree():
    key = rng.philox_key(9, 8, 7)
    blocks = rng.philox_blocks(1, 5, key)
    for j in range(5):
        assert [int(x) for x in blocks[j]] == rng.philox_block((j + 1, 0, 0, 0), key)


def test_uniform_range():
    u = rng.uniforms(1, 0, 0, 100000)
    assert u.min() > 0.0 and u.max() <= 1.0
