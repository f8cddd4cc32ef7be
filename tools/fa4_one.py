"""One attention launch on a bench shape, ours or FA4 (yardstick), for ncu:
    ncu --nvtx --nvtx-include cmp/ ... python tools/fa4_one.py {ours|fa4} {c3-batch|vit-qwen-full}"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402

CASES = {"c3-batch": ([2048, 300, 5000, 900], [16384, 5000, 5000, 8310], 28, 4, 128, True),
         "vit-qwen-full": ([29640], [29640], 16, 16, 80, False)}
which, case = sys.argv[1], sys.argv[2]
ql, kl, hq, hkv, hd, causal = CASES[case]
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(sum(ql), hq * hd, device="cuda", generator=g).bfloat16()
k = torch.randn(sum(kl), hkv * hd, device="cuda", generator=g).bfloat16()
v = torch.randn(sum(kl), hkv * hd, device="cuda", generator=g).bfloat16()
if which == "ours":
    meta = ops.AttnMeta([sum(ql[:i]) for i in range(len(ql))], ql,
                        [sum(kl[:i]) for i in range(len(kl))], kl, hq, causal)
    fn = lambda: ops.attention(q, k, v, meta, hkv, hd)
else:
    from vllm.vllm_flash_attn.cute.interface import flash_attn_varlen_func
    cu_q = torch.tensor([0] + [sum(ql[:i + 1]) for i in range(len(ql))], device="cuda",
                        dtype=torch.int32)
    cu_k = torch.tensor([0] + [sum(kl[:i + 1]) for i in range(len(kl))], device="cuda",
                        dtype=torch.int32)
    fn = lambda: flash_attn_varlen_func(q.view(-1, hq, hd), k.view(-1, hkv, hd),
                                        v.view(-1, hkv, hd), cu_seqlens_q=cu_q,
                                        cu_seqlens_k=cu_k, max_seqlen_q=max(ql),
                                        max_seqlen_k=max(kl), causal=causal)
for _ in range(3):
    fn()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("cmp")   # ncu --nvtx --nvtx-include cmp/
fn()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
