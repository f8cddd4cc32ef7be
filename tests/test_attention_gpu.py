"""tcgen05 varlen attention vs a plain torch fp32 reference (rtol 2e-2)."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(q, k, v, qs, ql, ks, kl, hq, hkv, hd, causal):
    out = torch.zeros(q.shape[0], hq * hd, dtype=torch.float32, device=q.device)
    g = hq // hkv
    for s in range(len(ql)):
        Q = q[qs[s]:qs[s] + ql[s]].float().view(ql[s], hq, hd).transpose(0, 1)
        K = k[ks[s]:ks[s] + kl[s]].float().view(kl[s], hkv, hd).transpose(0, 1)
        V = v[ks[s]:ks[s] + kl[s]].float().view(kl[s], hkv, hd).transpose(0, 1)
        K = K.repeat_interleave(g, 0)
        V = V.repeat_interleave(g, 0)
        S = Q @ K.transpose(1, 2) / math.sqrt(hd)
        if causal:
            qpos = torch.arange(kl[s] - ql[s], kl[s], device=q.device)
            kpos = torch.arange(kl[s], device=q.device)
            S = S.masked_fill(kpos[None, None, :] > qpos[None, :, None], float("-inf"))
        P = torch.softmax(S, -1)
        out[qs[s]:qs[s] + ql[s]] = (P @ V).transpose(0, 1).reshape(ql[s], hq * hd)
    return out


CASES = [
    # (q_lens, kv_lens, hq, hkv, hd, causal)
    ([128], [128], 1, 1, 128, False),
    ([1], [1], 2, 1, 128, True),
    ([5, 300, 129], [5, 300, 129], 4, 2, 128, True),          # plain causal prefill
    ([17, 64, 1], [1000, 64, 4500], 8, 2, 128, True),         # suffix over cached prefix
    ([577, 577, 577], [577, 577, 577], 16, 16, 64, False),    # CLIP-L/336 ViT
    ([64] * 6, [64] * 6, 4, 4, 64, False),                    # windowed ViT
    ([700], [3000], 28, 4, 128, True),                        # Qwen-7B GQA 7:1
    ([250, 3], [250, 131], 32, 32, 128, True),                # Llama MHA
    ([64, 64, 16, 48, 32, 64], [64, 64, 16, 48, 32, 64], 16, 16, 80, False),  # Qwen ViT windows
    ([1000, 260], [1000, 260], 16, 16, 80, False),            # Qwen ViT full-attention layers
    ([300], [700], 4, 2, 80, True),                           # hd 80 causal, GQA
]


@pytest.mark.parametrize("tile_rows", [128, 256])
@pytest.mark.parametrize("ql,kl,hq,hkv,hd,causal", CASES)
def test_attention_matches_fp32(ql, kl, hq, hkv, hd, causal, tile_rows):
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(sum(ql) + hq)
    qs = [0]
    for x in ql[:-1]:
        qs.append(qs[-1] + x)
    ks = [0]
    for x in kl[:-1]:
        ks.append(ks[-1] + x + 7)  # gaps between sequences in the KV buffer
    Tq, Tk = sum(ql), ks[-1] + kl[-1] + 3
    q = torch.randn(Tq, hq * hd, device="cuda", generator=g).bfloat16()
    k = torch.randn(Tk, hkv * hd, device="cuda", generator=g).bfloat16()
    v = torch.randn(Tk, hkv * hd, device="cuda", generator=g).bfloat16()
    meta = ops.AttnMeta(qs, ql, ks, kl, hq, causal, tile_rows=tile_rows)
    out = ops.attention(q, k, v, meta, hkv, hd)
    torch.cuda.synchronize()
    ref = _ref(q, k, v, qs, ql, ks, kl, hq, hkv, hd, causal)
    err = (out.float() - ref).abs()
    assert torch.isfinite(out.float()).all()
    assert err.max().item() < 2e-2 * max(1.0, ref.abs().max().item()) + 1e-2, err.max().item()
    assert (err.norm() / ref.norm()).item() < 1e-2


def test_attention_hd80_strided_qkv_views():
    """Qwen2.5-VL vision layout: q, k, v are column views of one fused
    [T, 3 * 16 * 80] QKV buffer (token pitch 3840), windows of 64 patches."""
    from paper_2507_10069_b200 import ops
    hq, hd = 16, 80
    g = torch.Generator(device="cuda").manual_seed(7)
    lens = [64] * 9 + [32, 16, 64]
    T = sum(lens)
    qkv = torch.randn(T, 3 * hq * hd, device="cuda", generator=g).bfloat16()
    q, k, v = qkv[:, :hq * hd], qkv[:, hq * hd:2 * hq * hd], qkv[:, 2 * hq * hd:]
    st = [0]
    for x in lens[:-1]:
        st.append(st[-1] + x)
    meta = ops.AttnMeta(st, lens, st, lens, hq, causal=False)
    out = ops.attention(q, k, v, meta, hq, hd)
    torch.cuda.synchronize()
    ref = _ref(q.contiguous(), k.contiguous(), v.contiguous(), st, lens, st, lens, hq, hq, hd,
               False)
    err = (out.float() - ref).abs()
    assert (err.norm() / ref.norm()).item() < 1e-2


@pytest.mark.parametrize("tile_rows", [128, 256, "packed"])
@pytest.mark.parametrize("wins", [[64] * 9 + [32, 16, 64], [64, 64, 48, 16, 64, 40, 24] * 7,
                                  [16] * 20, [128, 8, 120, 64, 100, 64]])
def test_attention_windowed_row_bounds(wins, tile_rows):
    """Windowed vision attention as ONE sequence per image whose rows see only
    their own window (row bounds), straight from the fused QKV buffer; must
    equal independent attention per window."""
    from paper_2507_10069_b200 import ops
    hq, hd = 16, 80
    g = torch.Generator(device="cuda").manual_seed(len(wins))
    imgs = [wins, wins[: max(1, len(wins) // 3)]]
    lens = [sum(w) for w in imgs]
    T = sum(lens)
    qkv = torch.randn(T, 3 * hq * hd, device="cuda", generator=g).bfloat16()
    q, k, v = qkv[:, :hq * hd], qkv[:, hq * hd:2 * hq * hd], qkv[:, 2 * hq * hd:]
    st = [0, lens[0]]
    if tile_rows == "packed":
        meta = ops.AttnMeta.window_packed(st, imgs, hq)
    else:
        meta = ops.AttnMeta(st, lens, st, lens, hq, causal=False, windows=imgs,
                            tile_rows=tile_rows)
    out = ops.attention(q, k, v, meta, hq, hd)
    torch.cuda.synchronize()
    segs = [x for w in imgs for x in w]
    ss = [0]
    for x in segs[:-1]:
        ss.append(ss[-1] + x)
    ref = _ref(q.contiguous(), k.contiguous(), v.contiguous(), ss, segs, ss, segs, hq, hq, hd,
               False)
    err = (out.float() - ref).abs()
    assert torch.isfinite(out.float()).all()
    assert (err.norm() / ref.norm()).item() < 1e-2
    assert meta.flops(hd) == 4.0 * hd * hq * sum(x * x for x in segs)


def test_work_queue_scheduling_across_launches_and_streams():
    """The pair kernel's work queue (per-stream self-resetting counters):
    many back-to-back launches on two streams, varlen causal items of very
    different lengths, every output equal to the round-robin schedule's
    (same per-item arithmetic, so bit-identical) and to fp32."""
    import os
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(5)
    ql, kl, hq, hkv, hd = [2048, 300, 1500, 900, 1], [9000, 5000, 1500, 8310, 700], 8, 2, 128
    qs = [sum(ql[:i]) for i in range(len(ql))]
    ks = [sum(kl[:i]) for i in range(len(kl))]
    q = torch.randn(sum(ql), hq * hd, device="cuda", generator=g).bfloat16()
    k = torch.randn(sum(kl), hkv * hd, device="cuda", generator=g).bfloat16()
    v = torch.randn(sum(kl), hkv * hd, device="cuda", generator=g).bfloat16()
    meta = ops.AttnMeta(qs, ql, ks, kl, hq, True, tile_rows=256)
    ref = _ref(q, k, v, qs, ql, ks, kl, hq, hkv, hd, True)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i in range(12):
        s = streams[i % 2]
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            outs.append(ops.attention(q, k, v, meta, hkv, hd))
    torch.cuda.synchronize()
    first = outs[0]
    err = (first.float() - ref).abs()
    assert (err.norm() / ref.norm()).item() < 1e-2
    for o in outs[1:]:
        assert torch.equal(o, first)


def test_single_tile_epilogue_waits_for_last_pv_cold_l2():
    """Regression (session 5): the single-tile kernel's epilogue waited on the
    per-PV barrier by parity while PV(L-1) and PV(L) could both be in flight,
    so with slow (cold-L2) V loads it read O one or two blocks early (first
    launch of [300] x [700] hd-80 causal: rows 18-30 of head 1 off by 0.1).
    Every launch here starts with a cold L2 and must give identical bytes."""
    from paper_2507_10069_b200 import ops
    ql, kl, hq, hkv, hd = [300], [700], 4, 2, 80
    g = torch.Generator(device="cuda").manual_seed(11)
    q = torch.randn(300, hq * hd, device="cuda", generator=g).bfloat16()
    k = torch.randn(703, hkv * hd, device="cuda", generator=g).bfloat16()
    v = torch.randn(703, hkv * hd, device="cuda", generator=g).bfloat16()
    meta = ops.AttnMeta([0], ql, [0], kl, hq, True, tile_rows=128)
    ref = _ref(q, k, v, [0], ql, [0], kl, hq, hkv, hd, True)
    bound = 2e-2 * max(1.0, ref.abs().max().item()) + 1e-2
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    first = None
    for it in range(40):
        flush.fill_(it & 255)
        out = ops.attention(q, k, v, meta, hkv, hd)
        torch.cuda.synchronize()
        assert (out.float() - ref).abs().max().item() < bound, it
        if first is None:
            first = out.clone()
        assert torch.equal(out, first), it
