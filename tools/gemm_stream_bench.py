"""Decode GEMMs as the decode step sees them: small M, every weight matrix
streamed from HBM once (rotating over enough copies that nothing stays in
the 126 MB L2), CUDA-graph replay.  Ours (tcgen05, split-K) vs cuBLAS on the
same inputs, in GB/s of weight bytes and as a fraction of measured HBM.

    python tools/gemm_stream_bench.py [M ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p)).get("hbm_gbs", 6538.0)
    return 6650.0


def graph_time(fns, reps=3):
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (reps * len(fns))


def main():
    Ms = [int(x) for x in sys.argv[1:]] or [40, 64]
    peak = hbm_peak()
    # Qwen2-7B decoder layer: QKV, o-proj, gate/up (interleaved), down
    shapes = [("qkv", 4608, 3584), ("o", 3584, 3584), ("gate_up", 37888, 3584),
              ("down", 3584, 18944)]
    for M in Ms:
        for name, N, K in shapes:
            wbytes = N * K * 2
            copies = max(2, int(512e6 // wbytes) + 1)   # > 4x L2 in rotation
            ws = [(torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16() for _ in range(copies)]
            a = torch.randn(M, K, device="cuda").bfloat16()
            c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            t = graph_time([lambda w=w: ops.gemm(a, w, out=c) for w in ws])
            tr = graph_time([lambda w=w: torch.matmul(a, w.t(), out=c) for w in ws])
            print(f"M={M:3d} {name:8s} N={N:6d} K={K:6d}: emm {t * 1e3:6.1f} us "
                  f"{wbytes / t / 1e6:5.0f} GB/s ({wbytes / t / 1e6 / peak:.2f}) | cublas "
                  f"{tr * 1e3:6.1f} us {wbytes / tr / 1e6:5.0f} GB/s ({wbytes / tr / 1e6 / peak:.2f})"
                  f" | ideal {wbytes / peak / 1e3:5.1f} us", flush=True)
            del ws
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
