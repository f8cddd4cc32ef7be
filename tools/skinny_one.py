"""One decode-size GEMM shape, a few launches (for ncu):
    python tools/skinny_one.py M N K [glu]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
glu = len(sys.argv) > 4 and sys.argv[4] == "glu"
a = torch.randn(M, K, device="cuda").bfloat16()
w = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
ss = ops.row_sumsq(a)
for _ in range(3):
    if glu:
        ops.gemm_ex(a, w, epi=ops.EPI_GLU_SILU, row_ss_in=ss, rms_dim=K, rms_eps=1e-6)
    else:
        ops.gemm(a, w)
torch.cuda.synchronize()
print("ok")
