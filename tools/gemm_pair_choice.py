"""Single-CTA (BN=256) vs CTA-pair tcgen05 GEMM at decoder shapes whose M is
an odd number of 128-row blocks (where the wave model picks the single-CTA
kernel): EMM_GEMM_PAIR=0 / default / 2 (force pair)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402


def bench(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for M in (6528, 6656, 8064, 8192, 12928, 16256):
    for name, N, K, epi in (("gate-up", 37888, 3584, ops.EPI_GLU_SILU), ("down", 3584, 18944, 0),
                            ("o", 3584, 3584, 0)):
        a = torch.randn(M, K, device="cuda").bfloat16()
        b = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        t = bench(lambda: ops.gemm(a, b, epi=epi))
        print(f"M={M} {name}: {t:.3f} ms {2 * M * N * K / t / 1e9:.0f} TF/s", flush=True)
