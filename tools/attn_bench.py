"""Attention kernel throughput on representative shapes (decoder causal with
cached prefix, ViT bidirectional)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10069_b200 import ops

def bench(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

for name, ql, kl, hq, hkv, hd, causal in [
        ("c2-batch", [400] * 35, [700] * 35, 32, 32, 128, True),
        ("long", [2048] * 8, [4096] * 8, 32, 32, 128, True),
        ("qwen-gqa", [1024] * 8, [8192] * 8, 28, 4, 128, True),
        ("vit-clip", [577] * 16, [577] * 16, 16, 16, 64, False),
        ("vit-qwen-full", [29640], [29640], 16, 16, 80, False),
        ("vit-qwen-win", [29640], [29640], 16, 16, 80, "win"),
        ("vit-qwen-win-packed", [29640], [29640], 16, 16, 80, "pack"),
        ("vit-c4-1img", [6517], [6517], 16, 16, 80, False),
        ("vit-c4-3img", [6517] * 3, [6517] * 3, 16, 16, 80, False),
        ("vit-c4-hd128", [6517] * 3, [6517] * 3, 10, 10, 128, False)]:
    qs = [sum(ql[:i]) for i in range(len(ql))]
    ks = [sum(kl[:i]) for i in range(len(kl))]
    q = torch.randn(sum(ql), hq * hd, device="cuda").bfloat16()
    k = torch.randn(sum(kl), hkv * hd, device="cuda").bfloat16()
    v = torch.randn(sum(kl), hkv * hd, device="cuda").bfloat16()
    if causal == "pack":
        meta = ops.AttnMeta.window_packed(qs, [[64] * 463 + [8]], hq)
    elif causal == "win":  # 463 windows of 64 patches (+ a ragged tail), row bounds
        meta = ops.AttnMeta(qs, ql, ks, kl, hq, False, windows=[[64] * 463 + [8]])
    else:
        meta = ops.AttnMeta(qs, ql, ks, kl, hq, causal)
    t = bench(lambda: ops.attention(q, k, v, meta, hkv, hd))
    print(f"{name}: {t:.3f} ms  {meta.flops(hd)/t/1e9:.0f} TF/s", flush=True)
