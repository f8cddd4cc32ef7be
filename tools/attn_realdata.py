"""Attention kernel on real activations vs random data: capture q/k/v of the
first ViT layer of a C4-shaped (CLIP-style, hd 80) encode and time the
kernel on them in isolation, next to the same shapes filled with randn."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402
from paper_2507_10069_b200.pipeline import HotPath  # noqa: E402
from paper_2507_10069_b200.shapes import SHAPES  # noqa: E402
from paper_2507_10069_b200.workload import ImageInput  # noqa: E402

shape = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "llama-11b-v"]
hp = HotPath(shape, budget_tokens=10000, own_cache=True)
cap = {}
orig = ops.attention


def spy(q, k, v, meta, hkv, hd, **kw):
    if "q" not in cap:
        cap.update(q=q.clone(), k=k.clone(), v=v.clone(), meta=meta, hkv=hkv, hd=hd)
    return orig(q, k, v, meta, hkv, hd, **kw)


ops.attention = spy
import paper_2507_10069_b200.encoder as enc  # noqa: E402
enc.ops.attention = spy
hp.encode([ImageInput("7" * 32, 6516, (0, 0))])
torch.cuda.synchronize()
ops.attention = orig


def bench(q, k, v):
    f = lambda: orig(q, k, v, cap["meta"], cap["hkv"], cap["hd"])
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    return ms, cap["meta"].flops(cap["hd"]) / ms / 1e9


q, k, v = cap["q"], cap["k"], cap["v"]
print("real q/k/v: %.3f ms %.0f TF/s" % bench(q, k, v))
sc = (q.float() @ k.float().t()[:, :1]).abs().max().item()
print("real |q|=%.3g |k|=%.3g" % (q.float().abs().mean().item(), k.float().abs().mean().item()))
print("randn    : %.3f ms %.0f TF/s" % bench(torch.randn_like(q), torch.randn_like(k),
                                          torch.randn_like(v)))
for s_ in (0.05, 3.0):
    print(f"randn*{s_}: %.3f ms %.0f TF/s" % bench(torch.randn_like(q) * s_,
                                                 torch.randn_like(k) * s_, torch.randn_like(v)))
