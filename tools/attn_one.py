"""One attention launch pattern for ncu: python tools/attn_one.py <case>."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402

from attn_one_cases import CASES  # noqa: E402
ql, kl, hq, hkv, hd, causal = CASES[sys.argv[1] if len(sys.argv) > 1 else "qwen"]
qs = [sum(ql[:i]) for i in range(len(ql))]
ks = [sum(kl[:i]) for i in range(len(kl))]
q = torch.randn(sum(ql), hq * hd, device="cuda").bfloat16()
k = torch.randn(sum(kl), hkv * hd, device="cuda").bfloat16()
v = torch.randn(sum(kl), hkv * hd, device="cuda").bfloat16()
if causal == "win":
    meta = ops.AttnMeta(qs, ql, ks, kl, hq, False, windows=[[64] * 463 + [8]])
else:
    meta = ops.AttnMeta(qs, ql, ks, kl, hq, causal)
for _ in range(3):
    ops.attention(q, k, v, meta, hkv, hd)
torch.cuda.synchronize()
