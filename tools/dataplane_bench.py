"""K1 throughput at scale: block hashes of a large CSR batch of unified
sequences and pixel digests of C3-sized images, in GB/s of algorithmic bytes
(keys + weights in, h0 + h1 + cumw out; pixel bytes in)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_10069_b200 import dataplane  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


rng = np.random.default_rng(0)
for n_seq, n_sym in [(212, 4400), (8192, 256), (2048, 4096)]:
    keys = [rng.integers(0, 2**62, n_sym, dtype=np.uint64) for _ in range(n_seq)]
    ws = [np.ones(n_sym, np.int64) for _ in range(n_seq)]
    b = dataplane.SeqBatch(keys, ws)
    ms = timeit(b.hash)
    nbytes = n_seq * n_sym * (8 + 8 + 8 + 8 + 8)
    print(f"K1 block hash {n_seq} x {n_sym} symbols: {ms * 1e3:.1f} us, "
          f"{nbytes / ms / 1e6:.0f} GB/s ({n_seq * n_sym / ms / 1e6:.2f} G symbols/s)", flush=True)
for n_img, (h, w) in [(65, (2184, 2660)), (68, (336, 336))]:
    imgs = [torch.randint(0, 256, (h * w * 3,), dtype=torch.uint8, device="cuda")
            for _ in range(n_img)]
    sizes = np.array([h * w * 3] * n_img, np.int64)
    starts = np.zeros(n_img, np.int64)
    starts[1:] = np.cumsum((sizes[:-1] + 15) // 16 * 16)
    buf = torch.empty(int(starts[-1] + sizes[-1]), dtype=torch.uint8, device="cuda")
    for i, t in enumerate(imgs):
        buf[starts[i]:starts[i] + sizes[i]].copy_(t)
    ms = timeit(lambda: dataplane.pixel_digest_ranges(buf, starts, sizes))
    print(f"K1 pixel digest {n_img} x {h}x{w}x3: {ms * 1e3:.1f} us, "
          f"{sizes.sum() / ms / 1e6:.0f} GB/s", flush=True)

# K2: batched GPU prefix match + token-granular block tables over a populated
# index (host tree inserts mirrored to the device by the journal flush)
from paper_2507_10069_b200.cache import GpuUnifiedCache  # noqa: E402
from paper_2507_10069_b200.keys import KeySeq  # noqa: E402
for n_seq, n_sym, w_img in [(212, 400, 64), (1024, 256, 16)]:
    cache = GpuUnifiedCache(4_000_000, 0.1)
    idx = dataplane.DeviceIndex(cache, n_layers=1, kv_dim=8, alloc_pool=False)
    keys, ws = [], []
    for i in range(n_seq):
        k = rng.integers(0, 2**62, n_sym, dtype=np.uint64)
        k[: n_sym // 2] = np.arange(n_sym // 2, dtype=np.uint64) + np.uint64(1 << 40)  # shared half
        w = np.ones(n_sym, np.int64)
        w[:4] = w_img                                    # a few image-weight symbols
        keys.append(k)
        ws.append(w)
        s = KeySeq(k, w, cache.codec)
        cache.insert_prefix(s, s.weights, float(i))
    idx.flush()
    torch.cuda.synchronize()
    b = dataplane.SeqBatch(keys, ws)
    b.hash()
    want = np.array([int(w.sum()) for w in ws], np.int64)
    ms = timeit(lambda: idx.match(b, want))
    probes = n_seq * n_sym
    nbytes = probes * (32 + 16) + int(want.sum()) * 8
    print(f"K2 match {n_seq} x {n_sym} symbols ({int(want.sum())} tokens): {ms * 1e3:.1f} us, "
          f"{nbytes / ms / 1e6:.0f} GB/s of probe + block-table bytes", flush=True)
