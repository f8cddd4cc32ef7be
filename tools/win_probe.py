"""Per-item cost of the packed-window ViT attention (attn_fwd_tc1_kernel):
time vs number of heads on one 29 640-patch image (232 packed 128-row tiles
per head), so time = fixed + ceil(items / 148) * t_item."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402


def bench(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


N, hd = 29640, 80
for H in [1, 2, 4, 8, 16, 32, 64]:
    q = torch.randn(N, H * hd, device="cuda").bfloat16()
    k = torch.randn(N, H * hd, device="cuda").bfloat16()
    v = torch.randn(N, H * hd, device="cuda").bfloat16()
    meta = ops.AttnMeta.window_packed([0], [[64] * 463 + [8]], H)
    t = bench(lambda: ops.attention(q, k, v, meta, H, hd))
    items = meta.n_tiles
    waves = (items + 147) // 148
    mb = 4 * N * H * hd * 2 / 1e6
    print(f"H={H:3d} items={items:6d} waves={waves:4d}: {t * 1e3:8.1f} us  "
          f"{t * 1e3 / waves:6.2f} us/item-wave  {mb / t / 1e3:6.2f} TB/s of q/k/v/o", flush=True)
