"""The four decoder-layer GEMMs of a decode step with their real epilogues
(QKV + RoPE + KV-cache scatter, o-proj + residual + row sum of squares,
gate/up SwiGLU with the folded RMSNorm scale, down + residual + sum of
squares) at Qwen2-7B shapes, weights rotated over > 4x L2, CUDA-graph
replay; us per GEMM.
    python tools/gemm_decode_layer_bench.py [M ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402


def graph_time(fns, reps=5):
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
    return s.elapsed_time(e) * 1e3 / (reps * len(fns))


def main():
    Ms = [int(x) for x in sys.argv[1:]] or [40, 64]
    d, hq, hkv, hd, ff = 3584, 28, 4, 128, 18944
    nq = (hq + 2 * hkv) * hd
    copies = 6
    r = lambda *s: (torch.randn(*s, device="cuda") * 0.02).bfloat16()
    W = [dict(qkv=r(nq, d), qkv_b=r(nq), o=r(d, d), gu=r(2 * ff, d), dn=r(d, ff))
         for _ in range(copies)]
    cs = ops.rope_table(8192, hd, 1e6)
    for M in Ms:
        x = r(M, d)
        ss = ops.row_sumsq(x)
        ss2 = torch.zeros(M, device="cuda")
        pos = torch.randint(0, 5000, (M,), device="cuda", dtype=torch.int32)
        kv_row = torch.arange(M, device="cuda", dtype=torch.int32)
        q = torch.empty(M, hq * hd, device="cuda", dtype=torch.bfloat16)
        k = torch.empty(M, hkv * hd, device="cuda", dtype=torch.bfloat16)
        v = torch.empty_like(k)
        a = r(M, d)
        x2 = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
        h = torch.empty(M, ff, device="cuda", dtype=torch.bfloat16)
        y = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
        qkv = dict(q_out=q, k_out=k, v_out=v, kv_row=kv_row, pos=pos, rope_cs=cs, hq=hq, hkv=hkv,
                   hd=hd)
        cases = {
            "qkv+rope": [lambda w=w: ops.gemm_ex(x, w["qkv"], epi=ops.EPI_QKV_ROPE, bias=w["qkv_b"],
                                                 row_ss_in=ss, rms_dim=d, rms_eps=1e-6, qkv=qkv,
                                                 row_ss_zero=ss2) for w in W],
            "o+res+ss": [lambda w=w: ops.gemm_ex(a, w["o"], out=x2, residual=x, row_ss_out=ss2)
                         for w in W],
            "gate_up glu": [lambda w=w: ops.gemm_ex(x2, w["gu"], out=h, epi=ops.EPI_GLU_SILU,
                                                    row_ss_in=ss2, rms_dim=d, rms_eps=1e-6)
                            for w in W],
            "down+res+ss": [lambda w=w: ops.gemm_ex(h, w["dn"], out=y, residual=x2, row_ss_out=ss)
                            for w in W],
        }
        tot = 0.0
        for name, fns in cases.items():
            t = graph_time(fns)
            tot += t
            print(f"M={M:3d} {name:12s} {t:7.1f} us", flush=True)
        layer = [f for fns in cases.values() for f in fns[:1]]
        seq = []
        for i in range(copies):
            seq += [fns[i] for fns in cases.values()]
        t = graph_time(seq) * 4
        print(f"M={M:3d} sum {tot:7.1f} us; back-to-back layer {t:7.1f} us", flush=True)


if __name__ == "__main__":
    main()
