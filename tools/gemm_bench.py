"""Quick tcgen05 GEMM throughput check vs cuBLAS (torch.matmul) on the box."""
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

for (M, N, K) in [(8192, 8192, 8192), (16384, 22016, 4096), (16384, 4096, 11008),
                  (16384, 12288, 4096), (16384, 4096, 4096), (4096, 4096, 4096), (577*8, 3072, 1024)]:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t = bench(lambda: ops.gemm(a, b, out=c))
    tr = bench(lambda: torch.matmul(a, b.t(), out=c))
    fl = 2 * M * N * K
    print(f"M={M} N={N} K={K}: emm {t:.3f} ms {fl/t/1e9:.0f} TF/s | cublas {tr:.3f} ms {fl/tr/1e9:.0f} TF/s", flush=True)
