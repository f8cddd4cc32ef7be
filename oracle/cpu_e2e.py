"""CPU port of the whole hot path, end to end — TEST / BASELINE
INFRASTRUCTURE ONLY (bench.py's cpu_baseline leg; never the product).

SURVEY.md §8d CPU leg 3 / BASELINE.md §4.3: a trace served on the host's
cores in fp32 with the SAME cache decisions as the product, made by the
reference's own `mmsim.cache.UnifiedCache` (pkg/src/mmsim/cache.py:363-406,
imported from baseline/_ref — no repo native code is loaded here):

  per prefill batch (arrival order, <= max_batch_tokens input tokens):
    image_lookup / encode the misses with the fp32 ViT (model_ref.vit_ref /
      qwen_vit_ref) / image_insert            (engine.py:474-501, 582-600)
    match_prefix -> cached = min(matched, total - 1)   (engine.py:539-547)
    prefill ONLY the uncached suffix with model_ref.decoder_ref(past=...),
      reusing the cached prefix's fp32 KV (taken from an earlier request
      with the same leading symbols: KV is causal, so it depends on nothing
      else)                                      (engine.py:602-632)
    insert_prefix + release                      (engine.py:653-657)

Returns the wall time and the work done, so the CPU number is measured on
the same work the GPU path does (not extrapolated).
"""
from __future__ import annotations

import time

import numpy as np
import torch

from . import model_ref

_TAG_PFX, _TAG_TXT = 1 << 62, 2 << 62


def unified_sequence(req):
    """Engine.unified_sequence (pkg/src/mmsim/engine.py:448-461)."""
    syms, w = [], []
    for img in req.images:
        syms.append(("img", img.content_hash))
        w.append(img.token_count)
    plen = req.prefix_len if req.prefix_id is not None else 0
    syms += [("pfx", req.prefix_id, i) for i in range(plen)]
    syms += [("txt", req.id, i) for i in range(req.text_input_len - plen)]
    w += [1] * (len(syms) - len(req.images))
    return syms, w


def _token_id(sym, vocab: int) -> int:
    """Text token id of a symbol: its injective key (keys.py, SURVEY App. A
    H3) mod vocab — the same ids the product embeds."""
    tag = _TAG_PFX if sym[0] == "pfx" else _TAG_TXT
    return (tag | (sym[1] << 32) | sym[2]) % vocab


def _pixels(content_hash: str, h: int, w: int) -> torch.Tensor:
    px = np.random.default_rng(int(content_hash[:16], 16)).integers(
        0, 256, (h, w, 3), dtype=np.uint8)
    return torch.from_numpy(px)


def run_trace(reqs, shape, budget_tokens: int, image_fraction: float,
              max_batch_tokens: int, threads: int, form_batches, grid_of,
              seed: int = 0, time_budget_s: float | None = None) -> dict:
    """Serve `reqs` end to end on the CPU.  form_batches / grid_of: the
    product's pure batching and patch-grid helpers (same batches, same
    image grids).  Stops early (and says so) after time_budget_s."""
    from mmsim.cache import UnifiedCache  # the reference cache (baseline/_ref)
    torch.set_num_threads(threads)
    v, d = shape.vision, shape.decoder
    Wv, Wd = model_ref.random_weights_f32(shape, seed=seed)
    vit = model_ref.qwen_vit_ref if v.arch == "qwen" else model_ref.vit_ref
    cache = UnifiedCache(budget_tokens, image_fraction)
    slabs: dict = {}
    done: list = []          # (symbols, k_list, v_list) of prefilled requests
    st = {"requests": 0, "batches": 0, "input_tokens": 0, "computed_tokens": 0,
          "cached_tokens": 0, "images_encoded": 0, "encode_tokens": 0, "first_tokens": []}
    t0 = time.perf_counter()
    truncated = False
    with torch.no_grad():
        for bi, batch in enumerate(form_batches(reqs, max_batch_tokens)):
            if time_budget_s is not None and time.perf_counter() - t0 > time_budget_s:
                truncated = True
                break
            now = float(bi)
            # every lookup of the batch first, then encode + insert the misses
            # (the engine's order: engine.py:474-501, then 593)
            seen, missed = set(), []
            for r in batch:
                for img in r.images:
                    h = img.content_hash
                    if h in seen:
                        continue
                    seen.add(h)
                    if cache.image_lookup(h, now) is None or h not in slabs:
                        missed.append(img)
            for img in missed:
                h = img.content_hash
                gh, gw = grid_of(img.token_count)
                slabs[h] = vit(shape, Wv, _pixels(h, gh * v.patch, gw * v.patch), (gh, gw))
                st["images_encoded"] += 1
                st["encode_tokens"] += img.token_count
                cache.image_insert(h, img.token_count, now,
                                   img.token_count * d.kv_bytes_per_token)
            handles, seqs = [], []
            for r in batch:
                syms, w = unified_sequence(r)
                m, handle = cache.match_prefix(syms, w, now)
                handles.append(handle)
                seqs.append((syms, w))
                total = r.total_input_len
                cached = min(m, total - 1)
                past = _donor(done, syms, w, cached) if cached > 0 else None
                if past is None:
                    cached = 0
                rows, pos3_syms = [], []
                acc = 0
                for s, ww in zip(syms, w):
                    if acc + ww > cached:   # rows of this symbol past the cached prefix
                        lo = max(0, cached - acc)
                        if s[0] == "img":
                            rows.append(slabs[s[1]][lo:])
                        else:
                            rows.append(Wd["embed"][_token_id(s, d.vocab)][None])
                    pos3_syms.append(("img", ww) if s[0] == "img" else ("txt", 1))
                    acc += ww
                x = torch.cat(rows, 0)
                pos3 = model_ref.mrope_positions_ref(pos3_syms) if d.mrope_section else None
                ks, vs, _, logits = model_ref.decoder_ref(shape, Wd, x, pos3=pos3, past=past)
                done.append((syms, ks, vs))
                st["first_tokens"].append(int(logits.argmax()))
                st["computed_tokens"] += total - cached
                st["cached_tokens"] += cached
                st["input_tokens"] += total
                st["requests"] += 1
            for syms, w in seqs:
                cache.insert_prefix(syms, w, now)
            for handle in handles:
                cache.release(handle)
            st["batches"] += 1
    st["seconds"] = time.perf_counter() - t0
    st["truncated"] = truncated
    st["cores"] = threads
    return st


def _donor(done, syms, w, cached):
    """fp32 KV of positions [0, cached) from the newest prefilled request
    whose leading symbols cover those positions."""
    acc, s = 0, 0
    while acc < cached:
        acc += w[s]
        s += 1
    head = syms[:s]
    for dsyms, ks, vs in reversed(done):
        if len(dsyms) >= s and dsyms[:s] == head:
            return [k[:cached] for k in ks], [v[:cached] for v in vs]
    return None
