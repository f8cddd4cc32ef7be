"""One packed-window attention launch (single-tile kernel) for ncu:
    ncu --nvtx --nvtx-include win/ ... python tools/win_one.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402

N, H, hd = 29640, 16, 80
q = torch.randn(N, H * hd, device="cuda").bfloat16()
k = torch.randn(N, H * hd, device="cuda").bfloat16()
v = torch.randn(N, H * hd, device="cuda").bfloat16()
meta = ops.AttnMeta.window_packed([0], [[64] * 463 + [8]], H)
for _ in range(3):
    ops.attention(q, k, v, meta, H, hd)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("win")
ops.attention(q, k, v, meta, H, hd)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
