"""Decode step breakdown at a true decoder shape: B requests with `ctx`
tokens of (random) KV already in the arena, one decode step timed per kernel
class (ops.TIMER) and end to end; HBM bytes per step = decoder weights read +
KV rows attended."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402
from paper_2507_10069_b200.decode import DecodeArena  # noqa: E402
from paper_2507_10069_b200.pipeline import HotPath  # noqa: E402
from paper_2507_10069_b200.shapes import SHAPES  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen-7b"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
# ctx: one length for every request, or "mixed": lengths like the bench's decode
# leg at C3 (lognormal, mean ~3.8k, one 15.5k row)
mixed = len(sys.argv) > 3 and sys.argv[3] in ("mixed",) or sys.argv[3:4] and sys.argv[3].endswith(".json")
ctx = 4400 if mixed or len(sys.argv) <= 3 else int(sys.argv[3])
if sys.argv[3:4] and sys.argv[3].endswith(".json"):   # kv lengths of a recorded step
    import json
    lens = [x - 1 for x in json.load(open(sys.argv[3]))][:B]
    B = len(lens)
elif mixed:
    import random
    rng = random.Random(1)
    lens = [int(min(15500, rng.lognormvariate(8.0, 0.8))) + 16 for _ in range(B - 1)] + [15464]
else:
    lens = [ctx] * B
shape = SHAPES[name]
hp = HotPath(shape, budget_tokens=1000, own_cache=False)
d = shape.decoder
arena = DecodeArena(shape, sum(lens) + 8 * B, device=hp.device)
arena.kv.normal_(0, 1)
slots = arena.alloc(sum(lens) + 8 * B)
off = np.zeros(B + 1, np.int64)
np.cumsum([x + 1 for x in lens], out=off[1:])      # each request: ctx rows + the new token
bt = ops.h2d(slots[:off[-1]], hp.device, np.int32)
bt_off = ops.h2d(off, hp.device, np.int64)
kv_len = ops.h2d(np.array(lens) + 1, hp.device, np.int32)
new = ops.h2d(slots[off[1:] - 1], hp.device, np.int32)
pos = ops.h2d(np.array(lens), hp.device, np.int32)
tok = ops.h2d(np.arange(B) * 7 % d.vocab, hp.device, np.int32)
ctx = max(lens)
f = lambda: hp.decoder.decode_step(tok, arena.kv, new, pos, bt, bt_off, kv_len, ctx + 1)
for _ in range(3):
    f()
torch.cuda.synchronize()
if "--ncu" in sys.argv:  # one step inside an NVTX range for ncu --nvtx-include prof/
    torch.cuda.nvtx.range_push("prof")
    f()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    sys.exit(0)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
s.record()
for _ in range(n):
    f()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / n
wbytes = sum(t.numel() * t.element_size() for L in hp.Wd["layers"] for t in L.values()
             if t is not None) + hp.Wd["lm_head"].numel() * 2
kvbytes = (sum(lens) + B) * d.layers * 2 * d.kv_dim * 2
peak = 6533.0
print(f"{name} B={B} ctx={'mixed' if mixed else ctx} (mean {sum(lens) // B}): step {ms:.3f} ms  ({B / ms * 1e3:.0f} tok/s)  weights "
      f"{wbytes / 1e9:.2f} GB + KV {kvbytes / 1e9:.2f} GB -> {(wbytes + kvbytes) / ms / 1e6:.0f} "
      f"GB/s ({(wbytes + kvbytes) / ms / 1e6 / peak:.2f} of HBM)")
# CUDA graph of the same step (what DecodeSession replays)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    f()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
s.record()
for _ in range(n):
    g.replay()
e.record()
torch.cuda.synchronize()
gms = s.elapsed_time(e) / n
print(f"  graph replay: {gms:.3f} ms  ({B / gms * 1e3:.0f} tok/s)  "
      f"{(wbytes + kvbytes) / gms / 1e6:.0f} GB/s ({(wbytes + kvbytes) / gms / 1e6 / peak:.2f} of HBM)")
ops.TIMER.start()
f()
torch.cuda.synchronize()
ops.TIMER.stop()
for k, v in ops.TIMER.summary().items():
    print(f"  {k:18s} {v['launches']:4d} launches {v['ms']:8.3f} ms")
# per-launch GEMM detail for layer 0 and the lm_head: bytes of B (weights) / time
recs = ops.TIMER.records.get("gemm", [])
for i in list(range(4)) + [len(recs) - 1]:
    s_, e_, w_ = recs[i][:3]
    ms_ = s_.elapsed_time(e_)
    nk = w_ / (2.0 * B)
    print(f"  gemm #{i}: N*K={nk / 1e6:.1f}M  {ms_ * 1e3:.1f} us  {nk * 2 / ms_ / 1e6:.0f} GB/s")
