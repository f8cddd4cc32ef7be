"""K1 on the GPU vs the C oracle: block (prefix) hashes and pixel digests,
bit-exact, including the edge cases (empty / length-1 / chunk-boundary
sequences, byte lengths that are not multiples of 8, segment boundaries)."""
import numpy as np
import pytest
import torch

from oracle import hashes

pytestmark = pytest.mark.gpu


def _rand_seq(rng, n):
    keys = rng.integers(0, 2**63, n, dtype=np.uint64) | np.uint64(1 << 62)
    w = rng.choice([1, 1, 1, 576, 6516, 7410], n).astype(np.int64)
    return keys, w


def test_block_hash_matches_oracle():
    from paper_2507_10069_b200 import dataplane
    rng = np.random.default_rng(3)
    # run (8), warp (256), chunk (2048) boundaries of block_hash_kernel
    lens = [0, 1, 2, 7, 8, 9, 31, 32, 33, 255, 256, 257, 511, 512, 1000, 2047, 2048, 2049,
            4097, 6145]
    seqs = [_rand_seq(rng, n) for n in lens]
    b = dataplane.block_hash([s[0] for s in seqs], [s[1] for s in seqs])
    torch.cuda.synchronize()
    h0 = b.h0.cpu().numpy().view(np.uint64)
    h1 = b.h1.cpu().numpy().view(np.uint64)
    cw = b.cumw.cpu().numpy()
    for i, (k, w) in enumerate(seqs):
        o0, o1 = hashes.prefix_hashes(k, w)
        s, e = b.off_host[i], b.off_host[i + 1]
        assert np.array_equal(h0[s:e], o0), lens[i]
        assert np.array_equal(h1[s:e], o1), lens[i]
        assert np.array_equal(cw[s:e], np.cumsum(w)), lens[i]


def test_block_hash_golden_kats():
    import json
    import os
    from paper_2507_10069_b200 import dataplane
    with open(os.path.join(os.path.dirname(__file__), "golden", "hash_kats.json")) as fh:
        kats = json.load(fh)
    seqs = [(np.array([int(x) for x in c["keys"]], np.uint64), np.array(c["weights"], np.int64))
            for c in kats["prefix"]]
    b = dataplane.block_hash([s[0] for s in seqs], [s[1] for s in seqs])
    h0 = b.h0.cpu().numpy().view(np.uint64)
    h1 = b.h1.cpu().numpy().view(np.uint64)
    for i, c in enumerate(kats["prefix"]):
        s, e = b.off_host[i], b.off_host[i + 1]
        assert [str(x) for x in h0[s:e]] == c["h0"]
        assert [str(x) for x in h1[s:e]] == c["h1"]


@pytest.mark.parametrize("sizes", [[0, 1, 7, 8, 9, 100], [8191, 8192, 8193, 65536 + 3],
                                   [336 * 336 * 3], [904 * 904 * 3, 17]])
def test_pixel_digest_matches_oracle(sizes):
    from paper_2507_10069_b200 import dataplane
    rng = np.random.default_rng(sum(sizes))
    imgs = [rng.integers(0, 256, n, dtype=np.uint8) for n in sizes]
    out = dataplane.pixel_digests([torch.from_numpy(x).cuda() for x in imgs]).cpu().numpy()
    for i, x in enumerate(imgs):
        o = hashes.pixel_digest(x)
        assert (int(out[i, 0]) & (2**64 - 1), int(out[i, 1]) & (2**64 - 1)) == o, sizes[i]


def test_pixel_identity_pass_matches_content_hash_pass():
    """The serving path keyed by the K1 digest of the uploaded pixels
    (driver.identify_images) makes exactly the cache decisions of the
    content_hash-keyed pass and produces the same first tokens: on the C1
    trace (images shared across requests) the digests are a bijection of the
    trace's content hashes."""
    from goldens import trace_path
    from paper_2507_10069_b200 import shapes
    from paper_2507_10069_b200.driver import TraceDriver
    from paper_2507_10069_b200.pipeline import HotPath, synthetic_pixels
    from paper_2507_10069_b200.workload import read_trace
    reqs = read_trace(trace_path("c1"))
    hp = HotPath(shapes.TINY, budget_tokens=600_000, image_fraction=0.25)
    drv = TraceDriver(hp, max_batch_tokens=16384)
    P = shapes.TINY.vision.patch
    host = {}
    for r in reqs:
        for img in r.images:
            if img.content_hash not in host:
                gh, gw = hp.image_grid(img.token_count)
                host[img.content_hash] = torch.from_numpy(
                    synthetic_pixels(img.content_hash, gh * P, gw * P)).pin_memory()
    a = drv.run_backlog(reqs, host_pixels=host, fetch_results=True)
    b = drv.run_backlog(reqs, host_pixels=host, fetch_results=True, identity="pixels")
    assert sum(len(r.images) for r in reqs) > len(host)          # shared images exist
    for f in ("requests", "batches", "input_tokens", "computed_tokens", "cached_tokens",
              "images_encoded", "encode_tokens"):
        assert getattr(a, f) == getattr(b, f), f
    assert a.first_tokens == b.first_tokens
    assert b.h2d_bytes > a.h2d_bytes          # every payload is uploaded and hashed
    assert hp.slabs and not (set(hp.slabs) & set(host))   # slabs keyed by digests
