"""Decode-size GEMMs (M <= 64) on the transposed weight-stream kernel
(csrc/gemm_skinny.cu) vs a plain torch fp32 reference: every epilogue the
decode step uses, split and unsplit K, partial weight tiles, persistent CTAs,
repeated launches and CUDA-graph replay (the split counters re-arm
themselves), and run-to-run determinism of the split reduction."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _close(out, ref, tol=2e-2):
    err = (out.float() - ref).abs()
    scale = ref.abs().mean().item() + 1e-6
    assert err.max().item() <= tol * max(ref.abs().max().item(), 1.0) + 4e-2 * scale, (
        err.max().item(), ref.abs().max().item())
    rel = (err.norm() / ref.norm()).item()
    assert rel < 8e-3, rel


def _rand(g, *shape, scale=1.0):
    return (torch.randn(*shape, device="cuda", generator=g) * scale).bfloat16()


@pytest.mark.parametrize("M", [1, 7, 16, 33, 40, 64])
@pytest.mark.parametrize("N,K", [(3584, 3584), (4608, 3584), (3584, 18944), (96, 640),
                                 (37984, 256)])
def test_skinny_plain(M, N, K):
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M * 131 + N + K)
    a = _rand(g, M, K)
    b = _rand(g, N, K, scale=K ** -0.5)
    out = ops.gemm(a, b)
    torch.cuda.synchronize()
    _close(out, a.float() @ b.float().t())


@pytest.mark.parametrize("epi", [1, 2, 3])
@pytest.mark.parametrize("M", [5, 40])
def test_skinny_bias_act_residual(epi, M):
    from paper_2507_10069_b200 import ops
    N, K = 1024, 2048
    g = torch.Generator(device="cuda").manual_seed(epi * 10 + M)
    a = _rand(g, M, K)
    b = _rand(g, N, K, scale=K ** -0.5)
    bias = _rand(g, N)
    res = _rand(g, M, N)
    acts = {1: lambda x: torch.nn.functional.gelu(x, approximate="tanh"),
            2: lambda x: x * torch.sigmoid(1.702 * x),
            3: lambda x: torch.nn.functional.gelu(x)}
    out = ops.gemm(a, b, bias=bias, residual=res, epi=epi)
    torch.cuda.synchronize()
    ref = acts[epi](a.float() @ b.float().t() + bias.float()) + res.float()
    _close(out, ref)


@pytest.mark.parametrize("M", [1, 40, 64])
@pytest.mark.parametrize("N,K", [(3584, 3584), (3584, 18944), (1000, 512)])
def test_skinny_residual_row_sumsq_and_zero(M, N, K):
    """o-proj / down shape: residual + row sum of squares of the stored bf16
    output; row_ss_zero clears the next layer's buffer."""
    from paper_2507_10069_b200 import ops
    if N % 32:
        N = (N // 32) * 32
    g = torch.Generator(device="cuda").manual_seed(M + N)
    a = _rand(g, M, K)
    b = _rand(g, N, K, scale=K ** -0.5)
    res = _rand(g, M, N)
    ss = torch.zeros(M, device="cuda")
    z = torch.full((M,), 7.0, device="cuda")
    out = ops.gemm_ex(a, b, residual=res, row_ss_out=ss, row_ss_zero=z)
    torch.cuda.synchronize()
    _close(out, a.float() @ b.float().t() + res.float())
    assert torch.allclose(ss, (out.float() ** 2).sum(-1), rtol=1e-3, atol=1e-2)
    assert z.abs().max().item() == 0


@pytest.mark.parametrize("M", [1, 40, 64])
@pytest.mark.parametrize("I,K", [(18944, 3584), (512, 2048), (1280, 640)])
def test_skinny_glu_rms(M, I, K):
    """gate/up with the folded RMSNorm row scale: 148 units (no split), 4
    units (split K) and 10 units."""
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M * 3 + I)
    x = _rand(g, M, K)
    wg = _rand(g, I, K, scale=K ** -0.5)
    wu = _rand(g, I, K, scale=K ** -0.5)
    bias = _rand(g, 2 * I)
    ss = ops.row_sumsq(x)
    m = ops.gemm_ex(x, ops.interleave_glu(wg, wu), epi=ops.EPI_GLU_SILU,
                    bias=ops.interleave_glu_bias(bias[:I], bias[I:]).contiguous(),
                    row_ss_in=ss, rms_dim=K, rms_eps=1e-6)
    torch.cuda.synchronize()
    xf = x.float()
    h = xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + 1e-6)
    ref = (torch.nn.functional.silu(h @ wg.float().t() + bias[:I].float())
           * (h @ wu.float().t() + bias[I:].float()))
    _close(m, ref)


@pytest.mark.parametrize("M", [1, 17, 64])
@pytest.mark.parametrize("hq,hkv,hd,mrope", [(28, 4, 128, False), (28, 4, 128, True),
                                             (14, 2, 64, False), (7, 1, 64, False)])
def test_skinny_qkv_rope(M, hq, hkv, hd, mrope):
    """Decode QKV: folded RMSNorm, bias, rotate-half RoPE (1-D or Qwen2-VL
    M-RoPE sections) and the KV-cache row scatter; (7, 1, 64) leaves a
    64-row head alone in the last weight tile."""
    from paper_2507_10069_b200 import ops
    D = 3584 if hd == 128 else 896
    g = torch.Generator(device="cuda").manual_seed(M * 5 + hq + mrope)
    N = (hq + 2 * hkv) * hd
    x = _rand(g, M, D)
    w = _rand(g, N, D, scale=D ** -0.5)
    bias = _rand(g, N)
    ss = ops.row_sumsq(x)
    pos = torch.randint(0, 5000, (M,), device="cuda", generator=g, dtype=torch.int32)
    ph = torch.randint(0, 5000, (M,), device="cuda", generator=g, dtype=torch.int32)
    pw = torch.randint(0, 5000, (M,), device="cuda", generator=g, dtype=torch.int32)
    kv_row = torch.randperm(400, device="cuda", generator=g)[:M].int()
    cs = ops.rope_table(8192, hd, 1e6)
    q = torch.zeros(M, hq * hd, device="cuda", dtype=torch.bfloat16)
    k = torch.zeros(400, hkv * hd, device="cuda", dtype=torch.bfloat16)
    v = torch.zeros_like(k)
    sec = (16, 24, 24) if hd == 128 else (8, 12, 12)
    qkv = dict(q_out=q, k_out=k, v_out=v, kv_row=kv_row, pos=pos, rope_cs=cs, hq=hq, hkv=hkv,
               hd=hd)
    if mrope:
        qkv.update(pos_h=ph, pos_w=pw, mrope=sec)
    ops.gemm_ex(x, w, epi=ops.EPI_QKV_ROPE, bias=bias, row_ss_in=ss, rms_dim=D, rms_eps=1e-6,
                qkv=qkv)
    torch.cuda.synchronize()
    xf = x.float()
    h = xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + 1e-6)
    y = h @ w.float().t() + bias.float()
    half = hd // 2
    i = torch.arange(half, device="cuda")
    if mrope:
        pp = torch.where(i[None] < sec[0], pos[:, None],
                         torch.where(i[None] < sec[0] + sec[1], ph[:, None], pw[:, None]))
    else:
        pp = pos[:, None].expand(M, half)
    c = cs[pp.long(), i[None].expand(M, half)]  # [M, half, 2]

    def rot(t, nh):
        t = t.view(M, nh, hd)
        a, b = t[..., :half], t[..., half:]
        cc, sn = c[:, None, :, 0], c[:, None, :, 1]
        return torch.cat([a * cc - b * sn, b * cc + a * sn], -1).view(M, nh * hd)
    _close(q, rot(y[:, : hq * hd], hq))
    _close(k[kv_row.long()], rot(y[:, hq * hd:(hq + hkv) * hd], hkv))
    _close(v[kv_row.long()], y[:, (hq + hkv) * hd:])


def test_skinny_split_deterministic_repeated_and_graphed():
    """The split reduction adds partials in split order: repeated launches and
    CUDA-graph replays give bit-identical outputs (the unit counters re-arm
    themselves after every launch)."""
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(11)
    M, N, K = 48, 3584, 18944
    a = _rand(g, M, K)
    b = _rand(g, N, K, scale=K ** -0.5)
    res = _rand(g, M, N)
    first = ops.gemm(a, b, residual=res)
    outs = [ops.gemm(a, b, residual=res) for _ in range(5)]
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, first)
    _close(first, a.float() @ b.float().t() + res.float())
    out = torch.empty_like(first)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ops.gemm(a, b, out=out, residual=res)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for _ in range(3):
                ops.gemm(a, b, out=out, residual=res)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(4):
        out.zero_()
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, first)


def test_skinny_k_not_multiple_of_64_uses_tile_kernel():
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(2)
    a = _rand(g, 40, 200)
    b = _rand(g, 512, 200, scale=200 ** -0.5)
    out = ops.gemm(a, b)
    torch.cuda.synchronize()
    _close(out, a.float() @ b.float().t())
