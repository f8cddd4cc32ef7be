"""The Qwen2.5-VL vision tower's four GEMMs on one image (26 064 or 29 640
patches) with the epilogues the encoder uses (folded RMSNorm row scale, bias,
2-D RoPE, SwiGLU, residual, row sum-of-squares), timed back to back;
cuBLAS on the bare matmuls as a yardstick.  EMM_GEMM_PAIR / build variants
select the kernel.

    python tools/gemm_vit_bench.py
"""
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


def main():
    d, ff = 1280, 3456
    for M in (26064, 29640):
        g = torch.Generator(device="cuda").manual_seed(0)
        r = lambda *s: (torch.randn(*s, device="cuda", generator=g) * 0.05).bfloat16()
        x, a, h = r(M, d), r(M, d), r(M, ff)
        o_w, o_b, gu_w, gu_b, dn_w, dn_b = r(d, d), r(d), r(2 * ff, d), r(2 * ff), r(d, ff), r(d)
        ss = torch.ones(M, device="cuda")
        ss2 = torch.empty_like(ss)
        cases = [
            ("o-proj   N=1280 K=1280 +res+ss", 2 * M * d * d,
             lambda: ops.gemm_ex(a, o_w, bias=o_b, residual=x, row_ss_out=ss2),
             lambda: torch.matmul(a, o_w.t())),
            ("gate-up  N=6912 K=1280 glu  ", 2 * M * 2 * ff * d,
             lambda: ops.gemm_ex(x, gu_w, epi=ops.EPI_GLU_SILU, bias=gu_b, row_ss_in=ss,
                                 rms_dim=d, rms_eps=1e-6),
             lambda: torch.matmul(x, gu_w.t())),
            ("down     N=1280 K=3456 +res+ss", 2 * M * d * ff,
             lambda: ops.gemm_ex(h, dn_w, bias=dn_b, residual=x, row_ss_out=ss2),
             lambda: torch.matmul(h, dn_w.t())),
        ]
        for name, fl, f, fr in cases:
            t, tr = timeit(f), timeit(fr)
            print(f"M={M} {name}: emm {t * 1e3:7.1f} us {fl / t / 1e9:6.0f} TF/s | cublas (bare) "
                  f"{tr * 1e3:7.1f} us {fl / tr / 1e9:6.0f} TF/s", flush=True)


if __name__ == "__main__":
    main()
