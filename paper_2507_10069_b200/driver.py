"""Trace drivers over a HotPath (one GPU).

* run_backlog  — throughput: the whole trace is queued at t=0 and served in
                 arrival order in prefill batches of at most
                 `max_batch_tokens` input tokens (the reference's per-instance
                 batch cap, RunConfig.max_batch_tokens_per_instance,
                 pkg/src/mmsim/engine.py:80, budgeted on total_input_len like
                 dispatch, engine.py:1057-1060).
* run_replay   — TTFT: open-loop replay of the trace's arrival times on a
                 virtual clock; whenever the GPU is idle it takes every
                 arrived request (same cap), runs encode + prefill and the
                 clock advances by the MEASURED device time of that batch.
                 TTFT = batch completion - arrival  (simulated queueing +
                 measured compute, SURVEY.md §8d "mode B").

Per batch the cache protocol is the engine's: image_lookup per image
(split_encode_work, engine.py:474-501), encode the misses once,
image_insert (engine.py:593), match_prefix + cached_prefix = min(matched,
total-1) (engine.py:539-547), prefill, insert_prefix + release
(engine.py:653-657).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .keys import KeySeq, request_keys


@dataclass
class PassStats:
    requests: int = 0
    batches: int = 0
    input_tokens: int = 0
    computed_tokens: int = 0
    cached_tokens: int = 0
    images_encoded: int = 0
    encode_tokens: int = 0
    flops: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    gpu_ms: float = 0.0
    first_tokens: list = field(default_factory=list)
    ttft: list = field(default_factory=list)


from .batching import affinity_key, form_batches, route, route_balanced, shard  # noqa: F401


class TraceDriver:
    def __init__(self, hp, max_batch_tokens: int = 16384):
        self.hp = hp
        self.max_batch_tokens = max_batch_tokens

    def identify_images(self, reqs, host_pixels, stats: PassStats):
        """Image identity from the pixels (the serving path):
        every image payload of the batch (each occurrence, as requests carry
        them) is copied H2D from pinned host memory, the K1 pixel digest runs
        on the GPU and the 122-bit digests come back (16 B per image).  The
        requests are re-keyed by the digest (32 hex digits), so the cache, the
        symbol keys and the slabs see the pixels' digest, not the trace's
        content_hash; the payloads stay staged on the device for the encode
        of the misses.  Returns (re-keyed requests, {digest: device bytes})."""
        import dataclasses

        from . import dataplane
        occ = [img for r in reqs for img in r.images]
        if not occ:
            return list(reqs), {}
        srcs = [host_pixels[img.content_hash].reshape(-1) for img in occ]
        sizes = np.array([int(t.numel()) for t in srcs], np.int64)
        offs = np.zeros(len(occ) + 1, np.int64)
        np.cumsum((sizes + 15) // 16 * 16, out=offs[1:])
        # upload + digest on a high-priority side stream: the host waits for
        # the digests only, not for the previous batch still on the main stream
        main = torch.cuda.current_stream(self.hp.device)
        if getattr(self, "_id_stream", None) is None:
            self._id_stream = torch.cuda.Stream(self.hp.device, priority=-1)
        with torch.cuda.stream(self._id_stream):
            buf = torch.empty(int(offs[-1]), dtype=torch.uint8, device=self.hp.device)
            for i, t in enumerate(srcs):
                buf[offs[i]:offs[i] + sizes[i]].copy_(t, non_blocking=True)
            dig_d = dataplane.pixel_digest_ranges(buf, offs[:-1], sizes)
            dig_h = torch.empty(dig_d.shape, dtype=dig_d.dtype, pin_memory=True)
            dig_h.copy_(dig_d, non_blocking=True)
            done = torch.cuda.Event()
            done.record()
        done.synchronize()
        main.wait_event(done)                # the encode reads the staged payloads
        buf.record_stream(main)
        dig = dig_h.numpy().view(np.uint64)
        stats.h2d_bytes += int(sizes.sum())
        stats.d2h_bytes += int(dig.nbytes)
        ident = [f"{int(d[0]):016x}{int(d[1]):016x}" for d in dig]
        staged, it = {}, iter(range(len(occ)))
        out = []
        for r in reqs:
            imgs = []
            for img in r.images:
                i = next(it)
                staged.setdefault(ident[i], buf[offs[i]:offs[i] + sizes[i]])
                imgs.append(dataclasses.replace(img, content_hash=ident[i]))
            out.append(dataclasses.replace(r, images=tuple(imgs)) if r.images else r)
        return out, staged

    def run_batch(self, reqs, now: float, stats: PassStats, host_pixels=None,
                  identity: str = "hash"):
        hp = self.hp
        staged = None
        if identity == "pixels":
            assert host_pixels is not None, "pixel identity needs the host payloads"
            reqs, staged = self.identify_images(reqs, host_pixels, stats)
            host_pixels = None
        hp.staged_pixels = staged
        try:
            return self._run_batch(reqs, now, stats, host_pixels, staged)
        finally:
            hp.staged_pixels = None

    def _run_batch(self, reqs, now, stats, host_pixels, staged):
        hp = self.hp
        cache = hp.cache
        dec = hp.shape.decoder
        # image cache (split_encode_work): lookups, in-batch de-dup, encode misses
        missed, seen = [], set()
        for r in reqs:
            for img in r.images:
                h = img.content_hash
                if h in seen:
                    continue
                seen.add(h)
                if cache.image_lookup(h, now) is None or h not in hp.slabs:
                    missed.append(img)
        if missed:
            stats.images_encoded += hp.encode(missed, now, host_pixels=host_pixels,
                                              device_pixels=staged)
            stats.encode_tokens += sum(i.token_count for i in missed)
            stats.flops += hp.encoder.last_flops
            if host_pixels is not None:
                stats.h2d_bytes += sum(int(host_pixels[i.content_hash].numel()) for i in missed)
            for img in missed:
                cache.image_insert(img.content_hash, img.token_count, now,
                                   img.token_count * dec.kv_bytes_per_token)
        # prefix match on the host tree (authoritative), then the device batch
        handles, cached = [], []
        for r in reqs:
            k, w = request_keys(hp.codec, r)
            seq = KeySeq(k, w, hp.codec)
            m, h = cache.match_prefix(seq, seq.weights, now)
            handles.append(h)
            cached.append(min(m, r.total_input_len - 1))
            stats.h2d_bytes += k.nbytes + w.nbytes
        res = hp.prefill(reqs, cached)
        hp.insert_batch(reqs, now)
        for h in handles:
            cache.release(h)
        hp.release_batch_kv()
        stats.requests += len(reqs)
        stats.batches += 1
        stats.input_tokens += res.input_tokens
        stats.computed_tokens += res.computed_tokens
        stats.cached_tokens += int(sum(cached))
        stats.flops += res.flops
        return res

    def run_backlog(self, reqs, host_pixels=None, fetch_results: bool = False,
                    identity: str = "hash") -> PassStats:
        """One pass over the trace from an empty cache (one bench step).
        identity="pixels": images are identified by the K1 digest of their
        host payloads (identify_images), as a server receiving pixels would."""
        self.hp.new_cache()
        st = PassStats()
        outs = []
        for bi, batch in enumerate(form_batches(reqs, self.max_batch_tokens)):
            res = self.run_batch(batch, float(bi), st, host_pixels, identity)
            outs.append(res.next_ids)
        if fetch_results:
            ids = torch.cat(outs).cpu()  # D2H of the step's result (first tokens)
            st.d2h_bytes += ids.numel() * ids.element_size()
            st.first_tokens = ids.tolist()
        return st

    def run_replay(self, reqs, host_pixels=None) -> PassStats:
        """Open-loop arrival replay; TTFT from measured batch device time."""
        self.hp.new_cache()
        st = PassStats()
        pending = sorted(reqs, key=lambda r: (r.arrival_time, r.id))
        clock, i = 0.0, 0
        queue = []
        while i < len(pending) or queue:
            while i < len(pending) and pending[i].arrival_time <= clock:
                queue.append(pending[i])
                i += 1
            if not queue:
                clock = pending[i].arrival_time
                continue
            batch, tok = [], 0
            while queue and (not batch or tok + queue[0].total_input_len <= self.max_batch_tokens):
                tok += queue[0].total_input_len
                batch.append(queue.pop(0))
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            res = self.run_batch(batch, clock, st, host_pixels)
            ids = res.next_ids.cpu()  # first tokens reach the host
            e.record()
            e.synchronize()
            dt = s.elapsed_time(e) / 1e3
            st.gpu_ms += dt * 1e3
            clock += dt
            for r in batch:
                st.ttft.append(clock - r.arrival_time)
        return st

    def run_decode(self, reqs, max_active: int = 64, n_slots: int = 600_000,
                   graphs: bool = True, step_log: list | None = None) -> dict:
        """Decode leg: the requests are prefilled in
        arrival order (untimed, from scratch) and admitted into a paged
        decode arena as they finish, keeping up to `max_active` decoding;
        every decode step is timed with CUDA events.  Returns generated
        tokens, steps, device seconds of the steps and the HBM bytes they
        read (decoder weights once per step + every attended KV row).
        `step_log` (optional) receives one [batch, kv rows read, longest kv
        row, kv lengths, ms, requests admitted just before] record per step."""
        from .decode import DecodeSession
        hp = self.hp
        dec = hp.shape.decoder
        sess = DecodeSession(hp, n_slots, graphs=graphs)
        pending = list(reqs)
        ev = []
        wbytes = sum(t.numel() * t.element_size() for L in hp.Wd["layers"]
                     for t in L.values() if isinstance(t, torch.Tensor))
        wbytes += hp.Wd["lm_head"].numel() * hp.Wd["lm_head"].element_size()
        kv_row_bytes = dec.kv_layers * 2 * dec.kv_dim * 2
        steps = gen = 0
        kv_rows = 0
        admitted = 0
        while pending or sess.active:
            room = max_active - len(sess.active)
            if pending and room > 0:
                batch, tok, slots = [], 0, 0
                free = sess.arena.free_slots
                while (pending and len(batch) < room
                       and (not batch or tok + pending[0].total_input_len <= self.max_batch_tokens)
                       and slots + pending[0].total_input_len + pending[0].output_len <= free):
                    tok += pending[0].total_input_len
                    slots += pending[0].total_input_len + pending[0].output_len
                    batch.append(pending.pop(0))
                if not batch:
                    if not sess.active:
                        raise MemoryError("decode arena too small for the next request")
                    pending_blocked = True
                else:
                    pending_blocked = False
                if not pending_blocked:
                    imgs = {i.content_hash: i for r in batch for i in r.images}
                    hp.encode(list(imgs.values()))
                    res = hp.prefill(batch, [0] * len(batch))
                    sess.admit(res.kv, batch, res.next_ids)
                    hp.release_batch_kv()
                    admitted += len(batch)
                    continue
            b = len(sess.active)
            rows_before = sess.kv_rows_read
            lens = [a.kv_len + 1 for a in sess.active] if step_log is not None else None
            sess.prepare()   # composition change: static buffers / graph capture, untimed
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            sess.step()
            e.record()
            ev.append((s, e))
            steps += 1
            gen += b
            kv_rows += sess.kv_rows_read - rows_before
            if step_log is not None:
                step_log.append([b, sess.kv_rows_read - rows_before, max(lens), lens, admitted])
                admitted = 0
        torch.cuda.synchronize()
        secs = sum(a.elapsed_time(b) for a, b in ev) / 1e3
        if step_log is not None:
            for rec, (a, b) in zip(step_log[-len(ev):], ev):
                rec.insert(4, a.elapsed_time(b))
        return {"requests": len(reqs), "generated_tokens": gen, "steps": steps,
                "device_s": secs, "tokens_per_s": gen / secs if secs else 0.0,
                "tpot_ms_mean": secs / steps * 1e3 if steps else 0.0,
                "mean_batch": gen / steps if steps else 0.0,
                "hbm_bytes": steps * wbytes + kv_rows * kv_row_bytes}


def nearest_rank(values, pct: float) -> float:
    """metrics.nearest_rank (pkg/src/mmsim/metrics.py:20-25)."""
    v = sorted(values)
    if not v:
        return float("nan")
    k = int(np.ceil(pct / 100.0 * len(v)))
    return float(v[max(0, k - 1)])
