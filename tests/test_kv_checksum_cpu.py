"""K6 migration checksum: the C oracle's XXH64
pinned against the published algorithm (the `xxhash` package) and the
checksum's defining properties, on the CPU."""
import numpy as np
import pytest

from oracle import hashes

xxhash = pytest.importorskip("xxhash")


@pytest.mark.parametrize("n", [0, 1, 3, 4, 7, 8, 15, 31, 32, 33, 63, 64, 100, 1024, 8192])
def test_oracle_xxh64_matches_published(n):
    rng = np.random.default_rng(n)
    data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
    for seed in (0, 1, 2 ** 32 + 17, 2 ** 64 - 1):
        assert hashes.xxh64(data, seed) == xxhash.xxh64_intdigest(data, seed=seed)


def test_known_answers():
    assert hashes.xxh64(b"", 0) == 0xEF46DB3751D8E999
    assert hashes.xxh64(b"abc", 0) == xxhash.xxh64_intdigest(b"abc")


def test_checksum_is_position_and_content_sensitive():
    rng = np.random.default_rng(3)
    planes = rng.integers(0, 2 ** 16, (3, 2, 40, 512), dtype=np.uint16)
    rows = rng.permutation(40)[:25].astype(np.int32)
    c = hashes.kv_checksum(planes, rows, 25)
    # the same rows gathered densely (what an exact copy produces)
    dense = np.ascontiguousarray(planes[:, :, rows])
    assert hashes.kv_checksum(dense, None, 25) == c
    # one flipped bit, two swapped rows, a row on the wrong plane: all change it
    bad = dense.copy()
    bad[1, 0, 7, 100] ^= 1
    assert hashes.kv_checksum(bad, None, 25) != c
    sw = dense.copy()
    sw[:, :, [3, 4]] = sw[:, :, [4, 3]]
    assert hashes.kv_checksum(sw, None, 25) != c
    kv = dense.copy()
    kv[2, [0, 1], 5] = kv[2, [1, 0], 5]
    assert hashes.kv_checksum(kv, None, 25) != c
