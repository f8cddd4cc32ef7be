"""CTA-pair GEMMs whose tile count leaves a partial last round (decoder o /
down projections at prefill-batch M, the ViT at one image): time with and
without the tail K split (EMM_GEMM_TAIL_SPLIT), checked against torch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402


def timeit(fn, iters=10):
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


for M, N, K in [(16384, 3584, 3584), (16384, 3584, 18944), (16384, 4608, 3584),
                (12000, 3584, 18944), (8000, 3584, 3584), (29640, 1280, 3456),
                (16384, 37888, 3584)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    a = (torch.randn(M, K, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    res = (torch.randn(M, N, device="cuda", generator=g) * 0.05).bfloat16()
    out = ops.gemm(a, b, residual=res)
    ref = a.float() @ b.float().t() + res.float()
    err = ((out.float() - ref).norm() / ref.norm()).item()
    t = timeit(lambda: ops.gemm(a, b, residual=res))
    print(f"M={M} N={N} K={K}: {t * 1e3:8.1f} us {2 * M * N * K / t / 1e9:6.0f} TF/s "
          f"rel err {err:.1e}", flush=True)
