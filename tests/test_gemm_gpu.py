"""tcgen05 GEMM vs a plain torch fp32 reference (bf16 output tolerance)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [
    (128, 128, 64), (1, 256, 64), (77, 96, 40), (300, 512, 640), (577, 3072, 1024),
    (1000, 4096, 4096), (4096, 11008, 4096), (256, 32000, 4096), (8192, 4096, 11008),
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
