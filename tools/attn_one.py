import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10069_b200 import ops
ql, kl, hq, hkv, hd = [400] * 35, [700] * 35, 32, 32, 128
qs = [sum(ql[:i]) for i in range(len(ql))]; ks = [sum(kl[:i]) for i in range(len(kl))]
q = torch.randn(sum(ql), hq * hd, device="cuda").bfloat16()
k = torch.randn(sum(kl), hkv * hd, device="cuda").bfloat16()
v = torch.randn(sum(kl), hkv * hd, device="cuda").bfloat16()
meta = ops.AttnMeta(qs, ql, ks, kl, hq, True)
for _ in range(3):
    ops.attention(q, k, v, meta, hkv, hd)
torch.cuda.synchronize()
