"""Parity at the bench's REAL shapes (VERDICT r1 top item): the kernels and
the full-depth Qwen2.5-VL-7B model that produce the C3 headline, against the
fp32 oracle (oracle/model_ref.py, run on the GPU in fp32 with chunked exact
attention), at the sizes bench.py runs:

* ViT full attention: one 7 410-token image = 29 640 patches, 16 heads of 80,
  bidirectional, q / k / v read from the fused QKV rows;
* ViT windowed attention: 26 064 patches (a 6 516-token image) in the
  product's window order, windows packed <= 128 rows per tile;
* decoder attention: causal GQA 28 / 4 heads of 128, a 2 048-token suffix
  over a 14 336-token cached prefix, batched with a shorter request;
* the whole 32-layer vision tower on a 7 410-token image;
* the 28-layer prefix-cached prefill of real C3 batches (the trace the bench
  runs, in its batch order, from an empty cache): every request's KV of every
  layer and its last-token logits vs the oracle's full recompute.

Tolerances (north star: bf16 within rtol 2e-2 of the reference's fp32):
relative Frobenius error < 2e-2 per tensor, and element-wise
|got - ref| <= 2e-2 * |ref| + 2e-2 * rms(ref) on >= 99 % of the elements
(the rms term keeps the element-wise bound meaningful where ref ~ 0).

Full depth: the bf16 FORMAT itself drifts from fp32 layer after layer
(tools/depth_error_probe.py: the oracle's own math with activations rounded
to bf16 where any bf16-storage implementation stores them reaches 1.5-3.4e-2
by layer 28 on these random-init weights, and the product tracks it within
a few per cent).  So the 32-layer ViT and the 28-layer decoder are held to
the fp32 bound OR, where the format alone exceeds it, to 1.15x the bf16
emulation's own error (oracle model_ref round_bf16=True) — a kernel bug
shows up as a product error well above the format's.  Every measured error
(product and emulation) is written to gpurun_out/fullshape_errors.json."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import model_ref

pytestmark = pytest.mark.gpu

RTOL = 2e-2
ELEM_FRAC = 0.99
_LOG: dict = {}


def _errs(got, ref):
    got, ref = got.float(), ref.float()
    fro = ((got - ref).norm() / ref.norm()).item()
    rms = ref.pow(2).mean().sqrt()
    ok = (got - ref).abs() <= RTOL * ref.abs() + RTOL * rms
    return fro, ok.float().mean().item()


def _check(name, got, ref):
    fro, frac = _errs(got, ref)
    _LOG[name] = {"rel_fro": fro, "elem_within_rtol": frac}
    _dump()
    assert torch.isfinite(got.float()).all(), name
    assert fro < RTOL, (name, fro)
    assert frac >= ELEM_FRAC, (name, frac)


def _check_depth(name, got, ref, emu):
    """Full-depth bound: the fp32 tolerance, or 1.15x what the bf16 format
    alone costs (emu = the oracle with bf16 storage rounding)."""
    fro, frac = _errs(got, ref)
    efro, efrac = _errs(emu, ref)
    _LOG[name] = {"rel_fro": fro, "elem_within_rtol": frac, "bf16_emulation_rel_fro": efro,
                  "bf16_emulation_elem_within_rtol": efrac}
    _dump()
    assert torch.isfinite(got.float()).all(), name
    assert fro < max(RTOL, 1.15 * efro + 1e-3), (name, fro, efro)
    assert frac >= min(ELEM_FRAC, efrac - 0.02), (name, frac, efrac)


def _dump():
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "fullshape_errors.json"), "w") as fh:
        json.dump(_LOG, fh, indent=1, sort_keys=True)


def _qwen7b(vit_layers=None):
    import dataclasses

    from paper_2507_10069_b200 import shapes
    s = shapes.SHAPES["qwen-7b"]
    if vit_layers is not None:
        s = dataclasses.replace(s, vision=dataclasses.replace(s.vision, layers=vit_layers))
    return s


def _ref_heads(q, k, v, hq, hkv, hd, causal):
    Q = q.float().view(q.shape[0], hq, hd).transpose(0, 1)
    K = k.float().view(k.shape[0], hkv, hd).transpose(0, 1).repeat_interleave(hq // hkv, 0)
    V = v.float().view(v.shape[0], hkv, hd).transpose(0, 1).repeat_interleave(hq // hkv, 0)
    return model_ref.sdpa_ref(Q, K, V, causal=causal).transpose(0, 1).reshape(q.shape[0], -1)


def test_vit_full_attention_29640_patches():
    from paper_2507_10069_b200 import ops
    N, H, hd = 29640, 16, 80
    g = torch.Generator(device="cuda").manual_seed(1)
    qkv = torch.randn(N, 3 * H * hd, device="cuda", generator=g).bfloat16()
    q, k, v = qkv[:, :H * hd], qkv[:, H * hd:2 * H * hd], qkv[:, 2 * H * hd:]
    meta = ops.AttnMeta([0], [N], [0], [N], H, causal=False)
    out = ops.attention(q, k, v, meta, H, hd)
    torch.cuda.synchronize()
    _check("attn_vit_full_29640", out, _ref_heads(q, k, v, H, H, hd, False))


def test_vit_window_attention_26064_patches():
    from paper_2507_10069_b200 import ops
    from paper_2507_10069_b200.encoder import window_plan
    from paper_2507_10069_b200.pipeline import patch_grid
    shape = _qwen7b()
    gh, gw = patch_grid(6516, shape.vision.merge)
    assert gh * gw == 26064
    v = shape.vision
    plan = window_plan(gh, gw, v.merge, v.window)
    wins = plan["window_lens"]
    N, H, hd = gh * gw, v.heads, v.head_dim
    g = torch.Generator(device="cuda").manual_seed(2)
    qkv = torch.randn(N, 3 * H * hd, device="cuda", generator=g).bfloat16()
    q, k, vv = qkv[:, :H * hd], qkv[:, H * hd:2 * H * hd], qkv[:, 2 * H * hd:]
    meta = ops.AttnMeta.window_packed(np.array([0]), [wins], H, device="cuda")
    out = ops.attention(q, k, vv, meta, H, hd)
    torch.cuda.synchronize()
    ref = torch.empty(N, H * hd, device="cuda")
    a = 0
    for w in wins.tolist():
        ref[a:a + w] = _ref_heads(q[a:a + w], k[a:a + w], vv[a:a + w], H, H, hd, False)
        a += w
    _check("attn_vit_window_26064", out, ref)


def test_decoder_attention_14k_prefix_2k_suffix():
    from paper_2507_10069_b200 import ops
    hq, hkv, hd = 28, 4, 128
    ql, kl = [2048, 300], [14336 + 2048, 5000]
    qs, ks = [0, 2048], [0, kl[0] + 64]
    g = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn(sum(ql), hq * hd, device="cuda", generator=g).bfloat16()
    k = torch.randn(ks[1] + kl[1], hkv * hd, device="cuda", generator=g).bfloat16()
    v = torch.randn(ks[1] + kl[1], hkv * hd, device="cuda", generator=g).bfloat16()
    meta = ops.AttnMeta(qs, ql, ks, kl, hq, causal=True)
    out = ops.attention(q, k, v, meta, hkv, hd)
    torch.cuda.synchronize()
    for s in range(2):
        ref = _ref_heads(q[qs[s]:qs[s] + ql[s]], k[ks[s]:ks[s] + kl[s]], v[ks[s]:ks[s] + kl[s]],
                         hq, hkv, hd, True)
        _check(f"attn_decoder_gqa_seq{s}_q{ql[s]}_kv{kl[s]}", out[qs[s]:qs[s] + ql[s]], ref)


def test_vit_32_layers_7410_token_image():
    """The whole Qwen2.5-VL-7B vision tower (32 layers, full attention in
    layers 7 / 15 / 23 / 31) + merger on one 7 410-token image."""
    from paper_2507_10069_b200.pipeline import HotPath, synthetic_pixels
    from paper_2507_10069_b200.workload import ImageInput
    shape = _qwen7b()
    assert shape.vision.layers == 32
    hp = HotPath(shape, budget_tokens=20000)
    img = ImageInput("7" * 32, 7410, (0, 0))
    assert hp.encode([img]) == 1
    torch.cuda.synchronize()
    gh, gw = hp.image_grid(7410)
    assert gh * gw == 29640
    P = shape.vision.patch
    px = synthetic_pixels(img.content_hash, gh * P, gw * P)
    pxd = torch.from_numpy(px).cuda()
    with torch.no_grad():
        ref = model_ref.qwen_vit_ref(shape, hp.Wv, pxd, (gh, gw))
        emu = model_ref.qwen_vit_ref(shape, hp.Wv, pxd, (gh, gw), round_bf16=True)
    got = hp.slabs[img.content_hash]
    assert got.shape == ref.shape == (7410, shape.decoder.d)
    _check_depth("vit32_7410_tokens", got, ref, emu)


def _oracle_request(hp, req):
    from paper_2507_10069_b200.keys import TAG_IMG, request_keys
    keys, w = request_keys(hp.codec, req)
    rows = []
    for k, ww in zip(keys, w):
        if int(k) >> 62 == TAG_IMG:
            rows.append(hp.slabs[hp.codec.symbol(int(k))[1]].float())
        else:
            rows.append(hp.Wd["embed"][int(k) % hp.shape.decoder.vocab].float()[None])
    x = torch.cat(rows, 0)
    syms = [("img", int(ww)) if int(k) >> 62 == TAG_IMG else ("txt", 1)
            for k, ww in zip(keys, w)]
    pos3 = model_ref.mrope_positions_ref(syms)
    with torch.no_grad():
        return (model_ref.decoder_ref(hp.shape, hp.Wd, x, pos3=pos3),
                model_ref.decoder_ref(hp.shape, hp.Wd, x, pos3=pos3, round_bf16=True))


def test_prefill_28_layers_real_c3_batches():
    """Full-depth Qwen2.5-VL-7B on the C3 trace in the bench's batch order
    from an empty cache (16 384-token batches).  Checked: batch 0 (computed
    from scratch), batch 45 (two requests over 6 516-token cached image
    prefixes, 2.2k computed) and batch 54 (14.1k of 14.6k tokens cached:
    a 7 410-token image prefix + system prefixes)."""
    from goldens import trace_path
    from paper_2507_10069_b200.driver import PassStats, TraceDriver, form_batches
    from paper_2507_10069_b200.keys import KeySeq, request_keys
    from paper_2507_10069_b200.pipeline import HotPath
    from paper_2507_10069_b200.workload import read_trace
    shape = _qwen7b()
    assert shape.decoder.layers == 28
    hp = HotPath(shape, budget_tokens=600_000, image_fraction=0.25)
    drv = TraceDriver(hp, 16384)
    hp.new_cache()
    st = PassStats()
    batches = form_batches(read_trace(trace_path("c3")), 16384)
    check_at = {0, 45, 54}
    for bi, batch in enumerate(batches[:55]):
        if bi not in check_at:
            drv.run_batch(batch, float(bi), st)
            continue
        _check_batch(hp, batch, bi, "c3")


def _check_batch(hp, batch, bi, tag, only=None):
    """Run one batch through the hot path by hand (image-pool lookups, encode
    of the misses, host match, prefill) and check every request's KV of every
    layer and its first token against the oracle's full recompute."""
    from paper_2507_10069_b200.keys import KeySeq, request_keys
    cache = hp.cache
    missed, seen = [], set()
    for r in batch:
        for img in r.images:
            if img.content_hash not in seen:
                seen.add(img.content_hash)
                if cache.image_lookup(img.content_hash, bi) is None or \
                        img.content_hash not in hp.slabs:
                    missed.append(img)
    if missed:
        hp.encode(missed, float(bi))
        for img in missed:
            cache.image_insert(img.content_hash, img.token_count, float(bi), 0)
    handles, cached = [], []
    for r in batch:
        k, w = request_keys(hp.codec, r)
        s = KeySeq(k, w, hp.codec)
        m, h = cache.match_prefix(s, s.weights, float(bi))
        handles.append(h)
        cached.append(min(m, r.total_input_len - 1))
    res = hp.prefill(batch, cached)
    torch.cuda.synchronize()
    bk = res.kv
    ids = res.next_ids.cpu().tolist()
    for j, r in enumerate(batch):
        if only is not None and j not in only(cached, batch):
            continue
        N, row0 = r.total_input_len, int(bk.row0[j])
        (ks, vs, hl, logits), (eks, evs, _, _) = _oracle_request(hp, r)
        got_k = bk.req_kv[:, 0, row0:row0 + N]
        got_v = bk.req_kv[:, 1, row0:row0 + N]
        _check_depth(f"{tag}_b{bi}_r{r.id}_K_all_layers(N={N},cached={cached[j]})", got_k,
                     torch.stack(ks), torch.stack(eks))
        _check_depth(f"{tag}_b{bi}_r{r.id}_V_all_layers", got_v, torch.stack(vs),
                     torch.stack(evs))
        # the first two layers stay inside the plain fp32 bound
        _check(f"{tag}_b{bi}_r{r.id}_K_layers0-1", got_k[:2], torch.stack(ks[:2]))
        top2 = logits.topk(2).values
        if (top2[0] - top2[1]).item() > 0.05 * logits.abs().max().item():
            assert ids[j] == int(logits.argmax()), (bi, r.id)
        del ks, vs, eks, evs
        torch.cuda.empty_cache()
    for h in handles:
        cache.release(h)
    return cached


def test_prefill_c5_true_width_4_layers():
    """Qwen2.5-VL-72B at its TRUE width (d 8192, GQA 64 / 8, d_ff 29 568,
    152k vocabulary) with 4 decoder layers, on the C5 trace in the bench's
    batch order from an empty cache with the bench's 80k-token budget
    (bench.py --config c5).  Checked: batch 0 from scratch and the first
    batch whose requests reuse a cached prefix of >= 1 000 tokens (the
    request with the longest cached prefix, plus the batch's first)."""
    import dataclasses

    from goldens import trace_path
    from paper_2507_10069_b200 import shapes
    from paper_2507_10069_b200.driver import PassStats, TraceDriver, form_batches
    from paper_2507_10069_b200.pipeline import HotPath
    from paper_2507_10069_b200.workload import read_trace
    s = shapes.SHAPES["qwen-72b"]
    shape = dataclasses.replace(
        s, decoder=dataclasses.replace(s.decoder, layers=4),
        vision=dataclasses.replace(s.vision, layers=2, full_layers=(1,)))
    assert shape.decoder.d == 8192 and shape.decoder.hq == 64 and shape.decoder.hkv == 8
    hp = HotPath(shape, budget_tokens=80_000, image_fraction=0.25)
    drv = TraceDriver(hp, 16384)
    hp.new_cache()
    st = PassStats()
    batches = form_batches(read_trace(trace_path("c5")), 16384)

    def pick(cached, batch):
        return {0, max(range(len(batch)), key=lambda j: cached[j])}

    _check_batch(hp, batches[0], 0, "c5w4", only=pick)
    hp.insert_batch(batches[0], now=0.0)
    hp.release_batch_kv()
    hit = False
    for bi, batch in enumerate(batches[1:40], start=1):
        from paper_2507_10069_b200.keys import KeySeq, request_keys
        best = 0
        for r in batch:
            k, w = request_keys(hp.codec, r)
            q = KeySeq(k, w, hp.codec)
            m, h = hp.cache.match_prefix(q, q.weights, float(bi))
            hp.cache.release(h)
            best = max(best, m)
        if best >= 1000:
            _check_batch(hp, batch, bi, "c5w4", only=pick)
            hit = True
            break
        drv.run_batch(batch, float(bi), st)
    assert hit, "no C5 batch with a cached prefix in the first 40 batches"
