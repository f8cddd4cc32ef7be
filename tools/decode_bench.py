"""Decode attention throughput (paged GQA, one query per request): bytes of
K/V rows read per launch / CUDA-event time, against HBM peak.  Shapes: the
C3 decode batch at Qwen2-7B (28/4 heads, hd 128), LLaVA-7B (MHA 32/32) and
Qwen-72B (64/8)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def run(name, n_req, ctx, hq, hkv, hd, iters=50, lens=None):
    g = torch.Generator(device="cuda").manual_seed(0)
    lens = lens or [ctx] * n_req
    n_req, ctx = len(lens), max(lens)
    n = sum(lens)
    K = torch.randn(n, hkv * hd, device="cuda", generator=g).bfloat16()
    V = torch.randn(n, hkv * hd, device="cuda", generator=g).bfloat16()
    bt = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
    off = [0]
    for x in lens:
        off.append(off[-1] + x)
    bt_off = torch.tensor(off, dtype=torch.int64, device="cuda")
    kv_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    q = torch.randn(n_req, hq * hd, device="cuda", generator=g).bfloat16()
    out = torch.empty_like(q)
    f = lambda: ops.decode_attention(q, K, V, bt, bt_off, kv_len, hkv, hd, ctx, out=out)
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    # flush L2 between launches: K/V of one launch (>= 126 MB) mostly exceed it anyway
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        f()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    byts = 2.0 * n * hkv * hd * 2 + n * 4
    print(f"{name}: {n_req} req x {n // n_req} ctx (max {ctx}): {ms * 1e3:.1f} us  {byts / ms / 1e6:.0f} GB/s "
          f"({byts / ms / 1e6 / peak:.2f} of {peak:.0f})", flush=True)


run("qwen7b", 64, 4400, 28, 4, 128)
# mixed lengths as in the bench's decode leg (C3: mean ~4.3k, longest ~15.5k)
rng = __import__("random").Random(1)
mixed = [int(min(15500, rng.lognormvariate(8.0, 0.8))) + 16 for _ in range(63)] + [15464]
run("qwen7b-mixed", 0, 0, 28, 4, 128, lens=mixed)
run("qwen7b-1long", 0, 0, 28, 4, 128, lens=[15000] + [3000] * 63)
run("qwen7b-mixed40", 0, 0, 28, 4, 128, lens=mixed[:39] + [15464])
run("qwen7b", 16, 4400, 28, 4, 128)
run("qwen7b", 128, 2048, 28, 4, 128)
run("qwen7b", 8, 16384, 28, 4, 128)
run("llava7b", 32, 1200, 32, 32, 128)
run("qwen72b", 32, 4400, 64, 8, 128)
run("tiny", 64, 1000, 4, 2, 64)
