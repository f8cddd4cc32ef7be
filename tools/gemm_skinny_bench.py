"""Decode-size (small M) GEMMs: weight-stream GB/s of the tcgen05 GEMM with
and without split-K, vs cuBLAS, each timed as a CUDA-graph replay of 20
back-to-back launches (no host launch cost in the number)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402


def graph_time(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (5 * reps)


for M, N, K in [(64, 4608, 3584), (64, 3584, 3584), (64, 3584, 18944), (64, 37888, 3584),
                (16, 4608, 3584), (128, 4608, 3584), (64, 152064, 3584), (40, 4608, 3584),
                (40, 3584, 3584), (40, 3584, 18944)]:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t = graph_time(lambda: ops.gemm(a, b, out=c))
    tr = graph_time(lambda: torch.matmul(a, b.t(), out=c))
    byts = N * K * 2
    print(f"M={M} N={N} K={K}: emm {t * 1e3:.1f} us {byts / t / 1e6:.0f} GB/s | cublas "
          f"{tr * 1e3:.1f} us {byts / tr / 1e6:.0f} GB/s", flush=True)
