"""Oracle pinning (CPU): the C hash oracle reproduces the committed
known-answer vectors, and the product's host restatement agrees with it."""
import ctypes as C
import json
import os

import numpy as np

from oracle import hashes

KATS = os.path.join(os.path.dirname(__file__), "golden", "hash_kats.json")


def _kats():
    with open(KATS) as fh:
        return json.load(fh)


def test_oracle_prefix_kats():
    for c in _kats()["prefix"]:
        k = np.array([int(x) for x in c["keys"]], np.uint64)
        h0, h1 = hashes.prefix_hashes(k, np.array(c["weights"], np.int64))
        assert [str(x) for x in h0] == c["h0"]
        assert [str(x) for x in h1] == c["h1"]


def test_oracle_pixel_kats():
    for c in _kats()["pixel"]:
        data = np.random.default_rng(c["seed"]).integers(0, 256, c["n"], dtype=np.uint8)
        d = hashes.pixel_digest(data)
        assert [str(d[0]), str(d[1])] == c["digest"]


def test_host_control_plane_hash_matches_oracle():
    from paper_2507_10069_b200._lib import lib
    rng = np.random.default_rng(11)
    for n in (0, 1, 17, 999):
        k = rng.integers(0, 2**64 - 1, n, dtype=np.uint64)
        w = rng.integers(1, 8000, n).astype(np.int64)
        a = np.empty(max(n, 1), np.uint64)
        b = np.empty(max(n, 1), np.uint64)
        assert lib.emm_prefix_hashes_host(k.ctypes.data, w.ctypes.data, n, a.ctypes.data,
                                          b.ctypes.data) == 0
        o0, o1 = hashes.prefix_hashes(k, w)
        assert np.array_equal(a[:n], o0) and np.array_equal(b[:n], o1)
