"""Per-phase cycle breakdown of the attention kernel (needs the ATT_PROF build:
tools/build_variant.sh prof -DATT_PROF=1; run with
EMM_LIB_PATH=build/libemm_prof.so python tools/attn_prof.py [case])."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import _lib, ops  # noqa: E402
from attn_one_cases import CASES  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "qwen"
ql, kl, hq, hkv, hd, causal = CASES[case]
qs = [sum(ql[:i]) for i in range(len(ql))]
ks = [sum(kl[:i]) for i in range(len(kl))]
q = torch.randn(sum(ql), hq * hd, device="cuda").bfloat16()
k = torch.randn(sum(kl), hkv * hd, device="cuda").bfloat16()
v = torch.randn(sum(kl), hkv * hd, device="cuda").bfloat16()
if causal == "win":
    meta = ops.AttnMeta(qs, ql, ks, kl, hq, False, windows=[[64] * 463 + [8]])
else:
    meta = ops.AttnMeta(qs, ql, ks, kl, hq, causal)
f = _lib.lib.emm_attn_prof
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 16)()
ops.attention(q, k, v, meta, hkv, hd)
f(buf, 1)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
ops.attention(q, k, v, meta, hkv, hd)
e.record()
torch.cuda.synchronize()
f(buf, 1)
n_tb = sum(1 for _ in range(1))  # placeholder
warp_blocks = buf[6]  # softmax warp-blocks counted
names = ["wait S", "tmem ld S", "mask+max+rescale", "exp+pack+st P", "wait st+arrive P"]
names_x = {7: "  (of which mask+max)"}
print(f"{case}: {s.elapsed_time(e):.3f} ms; softmax warp-blocks {warp_blocks}")
for i, nm in enumerate(names):
    print(f"  {nm:18s} {buf[i] / max(1, warp_blocks):8.1f} cyc / warp-block")
for i, nm in names_x.items():
    print(f"  {nm:18s} {buf[i] / max(1, warp_blocks):8.1f} cyc / warp-block")
print(f"  epilogue total     {buf[5] / max(1, warp_blocks):8.1f} cyc / warp-block (amortised)")
mb = max(1, warp_blocks // 8)  # MMA-warp blocks (8 softmax warps per CTA)
print(f"  MMA wait V         {buf[8] / mb:8.1f} cyc / block")
print(f"  MMA wait next K    {buf[10] / mb:8.1f} cyc / block")
print(f"  MMA wait P (x2)    {buf[9] / mb:8.1f} cyc / block")
