"""Cross-attention model (Llama-3.2-Vision) on the GPU:
image tokens carry their cross-attention K/V in the token-granular prefix
cache, text tokens their self-attention K/V; prefill (fresh and
prefix-cached, mixed with text-only requests) vs the fp32 oracle
(oracle/model_ref.decoder_ref with img=..., whose cross layer is pinned
against transformers' Mllama layer in test_mllama_cross_cpu.py)."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import model_ref

pytestmark = pytest.mark.gpu

RTOL = 2e-2


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm()).item()


def _shape(name, layers):
    from paper_2507_10069_b200 import shapes
    s = shapes.SHAPES[name]
    s = dataclasses.replace(s, vision=dataclasses.replace(s.vision, layers=1))
    if layers is not None:
        s = dataclasses.replace(s, decoder=dataclasses.replace(s.decoder, layers=layers))
    return s


def _oracle(hp, req):
    from paper_2507_10069_b200.keys import TAG_IMG, request_keys
    keys, w = request_keys(hp.codec, req)
    txt, img = [], []
    for k, ww in zip(keys, w):
        if int(k) >> 62 == TAG_IMG:
            img.append(hp.slabs[hp.codec.symbol(int(k))[1]].float())
        else:
            txt.append(hp.Wd["embed"][int(k) % hp.shape.decoder.vocab].float()[None])
    x = torch.cat(txt, 0)
    return model_ref.decoder_ref(hp.shape, hp.Wd, x, img=torch.cat(img, 0) if img else None)


def _check(hp, req, kv, row0, rid):
    d = hp.shape.decoder
    ks, vs, hl, logits = _oracle(hp, req)
    n_img = sum(i.token_count for i in req.images)
    N = req.total_input_len
    n_self = d.kv_layers
    for p in range(n_self):                      # text rows, self planes
        assert rel(kv[p, 0, row0 + n_img:row0 + N], ks[p]) < RTOL
        assert rel(kv[p, 1, row0 + n_img:row0 + N], vs[p]) < RTOL
    if n_img:                                    # image rows, cross planes
        for c in range(len(d.cross)):
            assert rel(kv[c, 0, row0:row0 + n_img], ks[n_self + c]) < RTOL
            assert rel(kv[c, 1, row0:row0 + n_img], vs[n_self + c]) < RTOL
    top = logits.topk(2).values
    if (top[0] - top[1]).item() > 0.05 * logits.abs().max().item():
        assert rid == int(logits.argmax())


@pytest.mark.parametrize("name,layers", [("tiny-x", None), ("llama-11b-v", 5)])
def test_cross_prefill_fresh_and_prefix_cached(name, layers):
    from paper_2507_10069_b200.keys import KeySeq, request_keys
    from paper_2507_10069_b200.pipeline import HotPath
    from paper_2507_10069_b200.workload import ImageInput, Request
    shape = _shape(name, layers)
    assert shape.decoder.cross, "the shape must contain a cross-attention layer"
    hp = HotPath(shape, budget_tokens=60000)
    tok = 576 if name == "llama-11b-v" else 64
    X = ImageInput("5" * 32, tok, (0, 0))
    Y = ImageInput("6" * 32, tok + 36, (0, 0))
    a = Request(0, 0.0, "multimodal", 40, (X,), 2, prefix_id=4, prefix_len=16)
    b = Request(1, 0.0, "multimodal", 25, (X,), 2, prefix_id=4, prefix_len=16)
    c = Request(2, 0.0, "text", 30, (), 2)
    e = Request(3, 0.0, "multimodal", 20, (Y, X), 2)
    hp.encode([X, Y])
    r1 = hp.prefill([c, a, e], [0, 0, 0])          # text-only first: reordered inside
    torch.cuda.synchronize()
    kv1 = hp._req_kv.clone()
    rows = hp._last.row0
    ids1 = r1.next_ids.cpu().tolist()
    for req, row0, rid in ((c, rows[0], ids1[0]), (a, rows[1], ids1[1]), (e, rows[2], ids1[2])):
        _check(hp, req, kv1, int(row0), rid)
    hp.insert_batch([c, a, e], now=1.0)
    hp.release_batch_kv()
    # b shares a's image and system prefix: its cross K/V and prefix text K/V
    # come from the pool (K3 gather), bit-identical to a's
    k, w = request_keys(hp.codec, b)
    s = KeySeq(k, w, hp.codec)
    matched, h = hp.cache.match_prefix(s, s.weights, 2.0)
    assert matched == tok + 16
    r2 = hp.prefill([b], [matched])
    torch.cuda.synchronize()
    assert int(r2.matched_kv[0]) == matched
    n_cross = len(shape.decoder.cross)
    a0 = int(rows[1])
    assert torch.equal(hp._req_kv[:n_cross, :, :tok], kv1[:n_cross, :, a0:a0 + tok])
    assert torch.equal(hp._req_kv[:, :, tok:matched], kv1[:, :, a0 + tok:a0 + matched])
    _check(hp, b, hp._req_kv, 0, int(r2.next_ids.cpu()[0]))
    hp.cache.release(h)


def test_cross_prefill_on_nan_filled_memory():
    """Image rows leave the self planes unused; a neighbouring request's
    masked 128-key block may still read them, so they must not carry NaN
    (fresh cudaMalloc memory is zero and would hide this)."""
    from paper_2507_10069_b200.pipeline import HotPath
    from paper_2507_10069_b200.workload import ImageInput, Request
    shape = _shape("llama-11b-v", 5)
    hp = HotPath(shape, budget_tokens=20000)
    X = ImageInput("8" * 32, 576, (0, 0))
    Y = ImageInput("9" * 32, 288, (0, 0))
    reqs = [Request(0, 0.0, "multimodal", 30, (X,), 5, prefix_id=2, prefix_len=8),
            Request(1, 0.0, "text", 19, (), 4),
            Request(2, 0.0, "multimodal", 11, (Y, X), 6)]
    hp.encode([X, Y])
    junk = torch.full((1 << 31,), float("nan"), device="cuda", dtype=torch.bfloat16)
    del junk       # the caching allocator hands these NaN bytes to the next buffers
    res = hp.prefill(reqs, [0, 0, 0])
    torch.cuda.synchronize()
    kv, rows = hp._req_kv, hp._last.row0
    for r, req in enumerate(reqs):
        n_img = sum(i.token_count for i in req.images)
        seg = kv[:, :, int(rows[r]):int(rows[r]) + req.total_input_len]
        assert torch.isfinite(seg[:, :, n_img:].float()).all()
        _check(hp, req, kv, int(rows[r]), int(res.next_ids[r]))
