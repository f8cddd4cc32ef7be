"""Per-phase cycles of the single-tile attention kernel on the packed ViT
windows (needs tools/build_variant.sh p1 -DATT1_PROF=1 and
EMM_LIB_PATH=build/libemm_p1.so)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import _lib, ops  # noqa: E402

N, H, hd = 29640, 16, 80
q = torch.randn(N, H * hd, device="cuda").bfloat16()
k = torch.randn(N, H * hd, device="cuda").bfloat16()
v = torch.randn(N, H * hd, device="cuda").bfloat16()
meta = ops.AttnMeta.window_packed([0], [[64] * 463 + [8]], H)
f = _lib.lib.emm_attn_prof
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 16)()
ops.attention(q, k, v, meta, H, hd)
f(buf, 1)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
ops.attention(q, k, v, meta, H, hd)
e.record()
torch.cuda.synchronize()
f(buf, 0)
warps = buf[4]  # items x 4 softmax warps (each warp adds 1 per item)
print(f"kernel {s.elapsed_time(e) * 1e3:.1f} us, {meta.n_tiles} items, softmax warp-items {warps}")
names = ["wait S (per block)", "softmax of the last block", "epilogue: wait last PV",
         "epilogue: TMEM -> global"]
for i, n in enumerate(names):
    print(f"  {n:28s} {buf[i] / max(warps, 1):8.1f} cycles / warp-item")
