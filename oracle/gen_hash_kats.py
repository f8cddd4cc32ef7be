"""Known-answer vectors pinning the block-hash / pixel-digest definitions
(TEST INFRASTRUCTURE).  Written by the C oracle; re-run only if the hash
definition in csrc/emm_hash.h is deliberately changed."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import hashes  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                   "hash_kats.json")


def main():
    rng = np.random.default_rng(20250710)
    prefix = []
    # engine-shaped symbols: image, shared prefix, request text (keys.py tags)
    img = (3 << 62) | 0x0123456789ABCDE
    seqs = [
        ([img] + [(1 << 62) | (2 << 32) | i for i in range(5)] + [(2 << 62) | (7 << 32) | i
                                                                     for i in range(4)],
         [576] + [1] * 9),
        ([0, 1, 2, 3], [1, 1, 1, 1]),
        ([2**64 - 1], [7410]),
    ]
    for n in (0, 1, 300):
        k = rng.integers(0, 2**63, n, dtype=np.uint64)
        w = rng.choice([1, 6516], n)
        seqs.append((list(map(int, k)), list(map(int, w))))
    for keys, w in seqs:
        h0, h1 = hashes.prefix_hashes(np.array(keys, np.uint64), np.array(w, np.int64))
        prefix.append({"keys": [str(k) for k in keys], "weights": [int(x) for x in w],
                       "h0": [str(x) for x in h0], "h1": [str(x) for x in h1]})
    pix = []
    for n in (0, 1, 8, 9, 8193, 336 * 336 * 3):
        data = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
        d = hashes.pixel_digest(data)
        pix.append({"n": n, "seed": n, "digest": [str(d[0]), str(d[1])]})
    with open(OUT, "w") as fh:
        json.dump({"prefix": prefix, "pixel": pix}, fh, indent=0)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
