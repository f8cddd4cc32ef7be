"""Row argmax (first tokens, decode steps): the chunked kernel (vocab split
in chunks over CTAs, one 64-bit (value, first index) key per chunk, a warp
per row reducing the keys) against a torch reference of the
same semantics — the first index of the maximum, NaNs ignored, 0 for a row
with nothing above -inf — on ties, -inf / NaN rows, unaligned views and
repeated launches (the per-row keys reset themselves)."""
import pytest
import torch

from paper_2507_10069_b200 import ops

pytestmark = pytest.mark.gpu


def ref_argmax(x: torch.Tensor) -> torch.Tensor:
    xf = x.float().clone()
    xf[torch.isnan(xf)] = -float("inf")
    mx = xf.max(dim=1, keepdim=True).values
    hit = (xf == mx) & (mx > -float("inf"))
    idx = torch.arange(x.shape[1], device=x.device).expand_as(xf)
    first = torch.where(hit, idx, torch.full_like(idx, x.shape[1])).min(dim=1).values
    return torch.where(first == x.shape[1], torch.zeros_like(first), first).to(torch.int32)


@pytest.mark.parametrize("T,V", [(64, 152064), (1, 152064), (7, 32000), (300, 128256),
                                 (5, 8192), (3, 8193), (2, 100)])
def test_argmax_rows_matches_reference(T, V):
    g = torch.Generator(device="cuda").manual_seed(T * 7 + V)
    x = torch.randn(T, V, device="cuda", generator=g).bfloat16()
    # coarse values -> many exact ties across chunks; a few special rows
    x = (x * 4).round() / 4
    if T >= 3:
        x[1] = -float("inf")
        x[2] = float("nan")
        x[2, V // 2] = 1.0
    for _ in range(3):  # repeated launches: the row keys reset themselves
        got = ops.argmax_rows(x)
        assert torch.equal(got.cpu(), ref_argmax(x).cpu())


def test_argmax_rows_strided_view():
    x = torch.randn(16, 152064 + 3, device="cuda").bfloat16()
    v = x[:, 1:1 + 152064]  # 2-byte offset rows: the scalar path
    assert torch.equal(ops.argmax_rows(v).cpu(), ref_argmax(v).cpu())


def test_argmax_rows_signed_zero_maximum():
    # a row whose maximum is a signed zero: -0.0 first, +0.0 later in another
    # chunk -> the first zero wins (torch semantics, -0.0 == +0.0)
    V = 152064
    x = torch.full((4, V), -1.0, device="cuda").bfloat16()
    x[0, 5] = -0.0
    x[0, V - 10] = 0.0
    x[1, 9000] = 0.0
    x[1, 20000] = -0.0
    x[2, :] = -0.0
    x[3, 100] = -0.0
    assert torch.equal(ops.argmax_rows(x).cpu(), ref_argmax(x).cpu())
    assert ops.argmax_rows(x).cpu().tolist() == [5, 9000, 0, 100]
