"""tcgen05 GEMM vs a plain torch fp32 reference (bf16 output tolerance)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [
    (128, 128, 64), (1, 256, 64), (77, 96, 40), (300, 512, 640), (577, 3072, 1024),
    (1000, 4096, 4096), (4096, 11008, 4096), (256, 32000, 4096), (8192, 4096, 11008),
    # decode-size M: split-K over the SMs (fp32 partials, last-arriver epilogue)
    (64, 4608, 3584), (16, 3584, 18944), (1, 512, 4096), (200, 1024, 2048),
]


def _ref(a, b, bias=None, residual=None, act=None):
    y = a.float() @ b.float().t()
    if bias is not None:
        y = y + bias.float()
    if act is not None:
        y = act(y)
    if residual is not None:
        y = y + residual.float()
    return y


def _close(out, ref, tol=2e-2):
    err = (out.float() - ref).abs()
    scale = ref.abs().mean().item() + 1e-6
    assert err.max().item() <= tol * max(ref.abs().max().item(), 1.0) + 4e-2 * scale, (
        err.max().item(), ref.abs().max().item())
    rel = (err.norm() / ref.norm()).item()
    assert rel < 8e-3, rel


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_plain(M, N, K):
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    out = ops.gemm(a, b)
    torch.cuda.synchronize()
    _close(out, _ref(a, b))


@pytest.mark.parametrize("epi", [1, 2, 3])
def test_gemm_bias_act_residual(epi):
    from paper_2507_10069_b200 import ops
    M, N, K = 333, 1024, 512
    g = torch.Generator(device="cuda").manual_seed(epi)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g).bfloat16()
    res = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    acts = {1: lambda x: torch.nn.functional.gelu(x, approximate="tanh"),
            2: lambda x: x * torch.sigmoid(1.702 * x),
            3: lambda x: torch.nn.functional.gelu(x)}
    out = ops.gemm(a, b, bias=bias, residual=res, epi=epi)
    torch.cuda.synchronize()
    _close(out, _ref(a, b, bias, res, acts[epi]))


def test_gemm_glu():
    from paper_2507_10069_b200 import ops
    M, I, K = 700, 1024, 768
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    wg = (torch.randn(I, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    wu = (torch.randn(I, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    out = ops.gemm(a, ops.interleave_glu(wg, wu), epi=ops.EPI_GLU_SILU)
    torch.cuda.synchronize()
    ref = torch.nn.functional.silu(a.float() @ wg.float().t()) * (a.float() @ wu.float().t())
    _close(out, ref)


def test_gemm_strided_views():
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(9)
    big = torch.randn(512, 1024, device="cuda", generator=g).bfloat16()
    a = big[:, 256:768]  # row pitch 1024, K = 512
    b = (torch.randn(384, 512, device="cuda", generator=g) / 20).bfloat16()
    out = torch.zeros(512, 640, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, out=out[:, 128:512])
    torch.cuda.synchronize()
    _close(out[:, 128:512], _ref(a, b))
    assert out[:, :128].abs().max().item() == 0


@pytest.mark.parametrize("M,D", [(300, 512), (64, 3584)])   # the second one splits K
@pytest.mark.parametrize("hq,hkv,hd", [(32, 32, 128), (28, 4, 128), (4, 2, 64)])
def test_gemm_qkv_rope_epilogue(hq, hkv, hd, M, D):
    """Fused folded-RMSNorm row scale + QKV split + RoPE + KV-cache write."""
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(hq)
    N = (hq + 2 * hkv) * hd
    x = torch.randn(M, D, device="cuda", generator=g).bfloat16()
    w = (torch.randn(N, D, device="cuda", generator=g) / D ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g).bfloat16()
    ss = ops.row_sumsq(x)
    pos = torch.randint(0, 5000, (M,), device="cuda", generator=g, dtype=torch.int32)
    kv_row = torch.randperm(400, device="cuda", generator=g)[:M].int()
    cs = ops.rope_table(8192, hd, 10000.0)
    q = torch.zeros(M, hq * hd, device="cuda", dtype=torch.bfloat16)
    k = torch.zeros(400, hkv * hd, device="cuda", dtype=torch.bfloat16)
    v = torch.zeros_like(k)
    ops.gemm_ex(x, w, epi=ops.EPI_QKV_ROPE, bias=bias, row_ss_in=ss, rms_dim=D, rms_eps=1e-5,
                qkv=dict(q_out=q, k_out=k, v_out=v, kv_row=kv_row, pos=pos, rope_cs=cs,
                         hq=hq, hkv=hkv, hd=hd))
    torch.cuda.synchronize()
    xf = x.float()
    h = xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + 1e-5)
    y = h @ w.float().t() + bias.float()
    half = hd // 2
    c = cs[pos.long()]  # [M, half, 2]

    def rot(t, nh):
        t = t.view(M, nh, hd)
        a, b = t[..., :half], t[..., half:]
        cc, sn = c[:, None, :, 0], c[:, None, :, 1]
        return torch.cat([a * cc - b * sn, b * cc + a * sn], -1).view(M, nh * hd)
    qr = rot(y[:, : hq * hd], hq)
    kr = rot(y[:, hq * hd:(hq + hkv) * hd], hkv)
    vr = y[:, (hq + hkv) * hd:]
    _close(q, qr)
    _close(k[kv_row.long()], kr)
    _close(v[kv_row.long()], vr)


@pytest.mark.parametrize("M,K,N", [(333, 768, 1024), (48, 4096, 1024)])  # second: split-K
def test_gemm_row_sumsq_out_and_scaled_glu(M, K, N):
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    res = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    ss = torch.zeros(M, device="cuda")
    out = ops.gemm_ex(a, b, residual=res, row_ss_out=ss)
    torch.cuda.synchronize()
    _close(out, _ref(a, b, residual=res))
    assert torch.allclose(ss, (out.float() ** 2).sum(-1), rtol=1e-3, atol=1e-2)
    wg = (torch.randn(512, N, device="cuda", generator=g) / N ** 0.5).bfloat16()
    wu = (torch.randn(512, N, device="cuda", generator=g) / N ** 0.5).bfloat16()
    m = ops.gemm_ex(out, ops.interleave_glu(wg, wu), epi=ops.EPI_GLU_SILU, row_ss_in=ss,
                    rms_dim=N, rms_eps=1e-5)
    torch.cuda.synchronize()
    of = out.float()
    h = of * torch.rsqrt((of * of).mean(-1, keepdim=True) + 1e-5)
    ref = torch.nn.functional.silu(h @ wg.float().t()) * (h @ wu.float().t())
    _close(m, ref)


@pytest.mark.parametrize("M", [300, 29640 // 8])
def test_gemm_rope2_epilogue_equals_rope2d_pass(M):
    """Qwen ViT: the 2-D RoPE applied in the QKV GEMM epilogue on
    pair-interleaved q / k weight rows equals the plain GEMM followed by the
    rope2d pass (rotate-half layout), after undoing the row permutation."""
    from paper_2507_10069_b200 import ops
    from paper_2507_10069_b200.weights import rope_pair_perm
    g = torch.Generator(device="cuda").manual_seed(M)
    d, hd, heads, theta = 1280, 80, 16, 10000.0
    x = torch.randn(M, d, device="cuda", generator=g).bfloat16()
    w = (torch.randn(3 * d, d, device="cuda", generator=g) / d ** 0.5).bfloat16()
    b = torch.randn(3 * d, device="cuda", generator=g).bfloat16()
    ph = torch.randint(0, 200, (M,), device="cuda", generator=g, dtype=torch.int32)
    pw = torch.randint(0, 200, (M,), device="cuda", generator=g, dtype=torch.int32)
    ref = ops.gemm(x, w, bias=b)
    ops.rope2d_(ref, 2 * heads, hd, ph, pw, theta)
    perm = rope_pair_perm(d, hd)
    cs = ops.rope_table(4096, hd // 2, theta)
    out = ops.gemm_ex(x, w[perm].contiguous(), bias=b[perm].contiguous(),
                      rope2=dict(cs=cs, cols=2 * d, hd=hd, pos_h=ph, pos_w=pw))
    torch.cuda.synchronize()
    got = torch.empty_like(out)
    got[:, perm] = out
    _close(got, ref.float())
