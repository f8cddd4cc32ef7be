"""Context for the attention roofline: our tcgen05 attention kernel next to
FlashAttention-4 (the CuTe-DSL sm100 forward kernel vLLM ships,
vllm.vllm_flash_attn.cute — LIBRARY code, used here only as a yardstick, never
on the product path) on the shapes the bench runs.  Same inputs, CUDA-event
timing after warm-up, outputs cross-checked.

    python tools/fa4_compare.py > gpurun_out/fa4_compare.txt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402

SHAPES = [  # name, q lens, kv lens, hq, hkv, hd, causal
    ("vit-qwen-full hd80", [29640], [29640], 16, 16, 80, False),
    ("vit-c4-3img hd80", [6517] * 3, [6517] * 3, 16, 16, 80, False),
    ("vit-c4-3img hd128", [6517] * 3, [6517] * 3, 10, 10, 128, False),
    ("qwen-gqa hd128 causal", [1024] * 8, [8192] * 8, 28, 4, 128, True),
    ("long hd128 causal", [2048] * 8, [4096] * 8, 32, 32, 128, True),
    ("c3-batch hd128 causal", [2048, 300, 5000, 900], [16384, 5000, 5000, 7410 + 900], 28, 4, 128,
     True),
]


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


def main():
    try:
        from vllm.vllm_flash_attn.cute.interface import flash_attn_varlen_func
    except Exception as exc:  # pragma: no cover
        print("FA4 not importable:", exc)
        flash_attn_varlen_func = None
    print(f"# {torch.cuda.get_device_name()}  ours = attn_fwd_tc_kernel, fa4 = "
          "vllm_flash_attn.cute flash_attn_varlen_func (FA4 sm100 forward)")
    for name, ql, kl, hq, hkv, hd, causal in SHAPES:
        qs = [sum(ql[:i]) for i in range(len(ql))]
        ks = [sum(kl[:i]) for i in range(len(kl))]
        g = torch.Generator(device="cuda").manual_seed(0)
        q = torch.randn(sum(ql), hq * hd, device="cuda", generator=g).bfloat16()
        k = torch.randn(sum(kl), hkv * hd, device="cuda", generator=g).bfloat16()
        v = torch.randn(sum(kl), hkv * hd, device="cuda", generator=g).bfloat16()
        meta = ops.AttnMeta(qs, ql, ks, kl, hq, causal)
        flops = meta.flops(hd)
        t_ours = timeit(lambda: ops.attention(q, k, v, meta, hkv, hd))
        out = ops.attention(q, k, v, meta, hkv, hd)
        line = f"{name:26s} ours {t_ours:7.3f} ms {flops / t_ours / 1e9:6.0f} TF/s"
        if flash_attn_varlen_func is not None:
            try:
                cu_q = torch.tensor([0] + [sum(ql[:i + 1]) for i in range(len(ql))],
                                    device="cuda", dtype=torch.int32)
                cu_k = torch.tensor([0] + [sum(kl[:i + 1]) for i in range(len(kl))],
                                    device="cuda", dtype=torch.int32)
                q3, k3, v3 = (q.view(-1, hq, hd), k.view(-1, hkv, hd), v.view(-1, hkv, hd))

                def fa():
                    return flash_attn_varlen_func(q3, k3, v3, cu_seqlens_q=cu_q, cu_seqlens_k=cu_k,
                                                  max_seqlen_q=max(ql), max_seqlen_k=max(kl),
                                                  causal=causal)
                r = fa()
                o4 = (r[0] if isinstance(r, tuple) else r).reshape(out.shape)
                t_fa = timeit(fa)
                err = ((o4.float() - out.float()).norm() / o4.float().norm()).item()
                line += (f" | fa4 {t_fa:7.3f} ms {flops / t_fa / 1e9:6.0f} TF/s"
                         f" | ours/fa4 {t_fa / t_ours:5.2f} | rel diff {err:.1e}")
            except Exception as exc:
                line += f" | fa4 failed: {type(exc).__name__}: {str(exc)[:120]}"
        print(line, flush=True)
    mhz = os.popen("nvidia-smi --query-gpu=clocks.sm --format=csv,noheader").read().strip()
    print("# sm clock after the runs:", mhz)


if __name__ == "__main__":
    main()
