"""Decode stage on one B200.

The reference models decode analytically: every decoding request ticks once
per `decode_step_time(batch, instances, resident_kv)` seconds
(pkg/src/mmsim/costmodel.py:121-136, engine.py:670-693), after its prefill
reserved `kv_need = input + output` KV tokens on its home instance
(engine.py:146-148, 623).  Here the step really runs:

  DecodeArena    token-granular paged KV arena [L, 2, slots, kv_dim] of one
                 GPU (the prefix pool's layout); a request admitted after
                 prefill reserves input + output - 1 slots (the reference's
                 kv_need; the first output token comes from prefill), its
                 prefill KV rows are copied in by K3 (one launch per batch),
                 and its block table is fixed for its lifetime.
  DecodeSession  continuous batching: every step feeds each active request's
                 previous token (device-resident, no host round trip) through
                 Decoder.decode_step — the fused QKV epilogue writes the new
                 K/V row straight into the request's next slot, the paged
                 decode attention kernel reads the whole history — and
                 retires requests that produced output_len tokens.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import dataplane, ops
from .keys import TAG_IMG
from .prefill import mrope_positions


class DecodeArena:
    def __init__(self, shape, n_slots: int, device="cuda"):
        dec = shape.decoder
        self.shape = shape
        self.device = torch.device(device)
        self.n_slots = int(n_slots)
        self.kv = torch.empty(dec.kv_layers, 2, self.n_slots, dec.kv_dim, dtype=torch.bfloat16,
                              device=self.device)
        # free list as a stack (top = end); slots handed out scattered over time
        self._free = np.arange(self.n_slots - 1, -1, -1, dtype=np.int32)
        self._top = self.n_slots

    @property
    def free_slots(self) -> int:
        return self._top

    def alloc(self, n: int) -> np.ndarray:
        if n > self._top:
            raise MemoryError(f"decode arena: {n} slots requested, {self._top} free")
        out = self._free[self._top - n:self._top][::-1].copy()
        self._top -= n
        return out

    def release(self, slots: np.ndarray) -> None:
        n = len(slots)
        self._free[self._top:self._top + n] = slots[::-1]
        self._top += n


@dataclass
class _Active:
    rid: object
    slots: np.ndarray      # reserved arena rows: prompt then generated tokens
    kv_len: int            # rows holding KV now
    next_pos: int          # RoPE position of the next input token
    left: int              # decode steps still to run
    tokens: list           # generated ids (host copy, filled when fetched)
    n_img: int = 0         # cross-attention models: slots[:n_img] hold the image rows
                           # (cross K/V); kv_len / next_pos then count text tokens


class _Static:
    """Graph-static device buffers of one batch bucket."""

    def __init__(self, Bp: int, bt_cap: int, device):
        i32 = dict(dtype=torch.int32, device=device)
        self.Bp = Bp
        self.tok = torch.zeros(Bp, **i32)
        self.bt = torch.zeros(bt_cap, **i32)
        self.bt_off = torch.zeros(Bp + 1, dtype=torch.int64, device=device)
        self.kv_len = torch.zeros(Bp, **i32)
        self.next_pos = torch.zeros(Bp, **i32)
        self.slot = torch.zeros(Bp, **i32)
        self.pos = torch.zeros(Bp, **i32)
        # cross-attention models: the image rows of each request
        self.bt_x = torch.zeros(bt_cap, **i32)
        self.bt_x_off = torch.zeros(Bp + 1, dtype=torch.int64, device=device)
        self.kv_len_x = torch.zeros(Bp, **i32)
        self.xmask = torch.zeros(Bp, dtype=torch.float32, device=device)
        self.graphs: dict = {}   # (kv bucket, image kv bucket) -> (CUDAGraph, ids, logits)


class DecodeSession:
    """Continuous-batching decode over one GPU's arena.

    graphs=True: every step is one CUDA-graph replay (a decode step is ~250
    small launches — eager, the host's per-launch cost would bound it).  The
    graph of a (batch bucket, KV-length bucket) pair is captured once: its
    inputs live in static buffers (block tables, lengths, positions, the
    previous tokens), the step advances them on the device
    (emm_decode_advance) and writes its argmax back into the token buffer,
    so consecutive replays need no host input until the batch composition
    changes.  Rows beyond the live requests are padding that attends to one
    scratch slot."""

    B_BUCKETS = (1, 2, 4, 8, 16, 32, 64, 128, 256)
    SCRATCH_SEG = 1 << 16

    def __init__(self, hp, n_slots: int, graphs: bool = True):
        self.hp = hp
        self.cross = bool(hp.shape.decoder.cross)
        self.shape = hp.shape
        # one extra slot: the scratch row every padding request writes / reads
        self.arena = DecodeArena(hp.shape, n_slots + 1, device=hp.device)
        self._scratch = int(self.arena.alloc(1)[0])
        self.active: list[_Active] = []
        self.tok = torch.zeros(0, dtype=torch.int32, device=hp.device)
        self._tables = None   # eager mode: device block tables of the composition
        self.graphs = graphs
        self._static: dict[int, _Static] = {}
        self._cur = None      # (static, kv bucket) loaded with the current composition
        self._pool = None
        self.steps = 0
        self.generated = 0
        self.kv_rows_read = 0   # sum over steps of attended KV rows (roofline)
        self.finished: dict = {}

    # ------------------------------------------------------------- admit
    def admit(self, batch_kv, reqs, first_ids: torch.Tensor, out_lens=None) -> None:
        """Requests just prefilled (their KV in batch_kv.req_kv rows
        [row0, row0 + total)), with their first token (prefill's argmax,
        device int32)."""
        dec = self.shape.decoder
        src, dst, new = [], [], []
        need = sum(int(req.total_input_len) + max(0, int(out_lens[r] if out_lens is not None
                                                          else req.output_len) - 1)
                   for r, req in enumerate(reqs))
        if need > self.arena.free_slots:   # all or nothing: no partial admission
            raise MemoryError(f"decode arena: {need} slots needed, {self.arena.free_slots} free")
        for r, req in enumerate(reqs):
            n = int(req.total_input_len)
            out_len = int(out_lens[r]) if out_lens is not None else int(req.output_len)
            steps = max(0, out_len - 1)          # token 1 came from prefill
            slots = self.arena.alloc(n + steps)
            row0 = int(batch_kv.row0[r])
            src.append(np.arange(row0, row0 + n, dtype=np.int32))
            dst.append(slots[:n])
            n_img = 0
            if dec.cross:    # images first (engine.py:448-461): text positions only
                keys, w = batch_kv.keys[r], batch_kv.weights[r]
                is_img = (np.asarray(keys, np.uint64) >> np.uint64(62)) == np.uint64(TAG_IMG)
                n_img = int(np.asarray(w)[is_img].sum())
                kv0 = nxt = n - n_img
            elif dec.mrope_section:
                pt, ph, pw = mrope_positions(batch_kv.keys[r], batch_kv.weights[r])
                kv0, nxt = n, int(max(pt.max(), ph.max(), pw.max())) + 1
            else:
                kv0 = nxt = n
            new.append(_Active(getattr(req, "id", r), slots, kv0, nxt, steps, [], n_img))
        if src:
            s = ops.h2d(np.concatenate(src), self.hp.device)
            d = ops.h2d(np.concatenate(dst), self.hp.device)
            dataplane.kv_copy_rows(batch_kv.req_kv, s, self.arena.kv, d, int(s.shape[0]))
        keep = [a for a in new if a.left > 0]
        for a in new:
            if a.left == 0:
                self.arena.release(a.slots)
                self.finished[a.rid] = a
        if keep:
            idx = [i for i, a in enumerate(new) if a.left > 0]
            ids = first_ids[torch.as_tensor(idx, device=first_ids.device)] if len(idx) != len(
                new) else first_ids
            self._sync_tok()
            self.tok = torch.cat([self.tok, ids.to(torch.int32)])
            self.active.extend(keep)
            self._tables = None
            self._cur = None

    # -------------------------------------------------------------- step
    def _build_tables(self):
        dev = self.hp.device
        selfs = [a.slots[a.n_img:] for a in self.active]
        bt = np.concatenate(selfs)
        off = np.zeros(len(self.active) + 1, np.int64)
        np.cumsum([len(x) for x in selfs], out=off[1:])
        self._tables = (ops.h2d(bt, dev, np.int32), ops.h2d(off, dev, np.int64))
        self._xtables = self._cross_tables(len(self.active)) if self.cross else None

    def _cross_tables(self, Bp: int):
        """Host arrays of the image rows (cross layers) for Bp rows."""
        d = self.shape.decoder
        B = len(self.active)
        imgs = [a.slots[:a.n_img] for a in self.active]
        bt = np.concatenate(imgs + [np.zeros(1, np.int32)])
        off = np.zeros(Bp + 1, np.int64)
        np.cumsum([len(x) for x in imgs], out=off[1:B + 1])
        off[B + 1:] = off[B]
        kvx = np.zeros(Bp, np.int32)
        mask = np.full(Bp, np.inf, np.float32)
        for i, a in enumerate(self.active):
            kvx[i] = a.n_img
            if a.n_img:
                mask[i] = (1.0 - d.eps) * d.d
        return bt, off, kvx, mask

    def _sync_tok(self):
        """Graph mode keeps the live tokens in the static buffer: pull them."""
        if self._cur is not None:
            st = self._cur[0]
            self.tok = st.tok[:len(self.active)].clone()

    def _bucket(self, B: int) -> int:
        for b in self.B_BUCKETS:
            if b >= B:
                return b
        return B

    def _load(self):
        """Write the current composition into the static buffers of its
        bucket (padding rows -> scratch segment)."""
        B = len(self.active)
        Bp = self._bucket(B)
        st = self._static.get(Bp)
        if st is None:
            st = _Static(Bp, self.arena.n_slots + self.SCRATCH_SEG, self.hp.device)
            self._static[Bp] = st
        selfs = [a.slots[a.n_img:] for a in self.active]
        real = np.concatenate(selfs)
        n_real = len(real)
        bt = np.concatenate([real, np.full(self.SCRATCH_SEG, self._scratch, np.int32)])
        off = np.zeros(Bp + 1, np.int64)
        np.cumsum([len(x) for x in selfs], out=off[1:B + 1])
        off[B + 1:] = n_real                       # padding rows: the scratch segment
        kv_len = np.zeros(Bp, np.int32)
        nxt = np.zeros(Bp, np.int32)
        for i, a in enumerate(self.active):
            kv_len[i], nxt[i] = a.kv_len, a.next_pos
        dev = self.hp.device
        st.bt[:len(bt)].copy_(ops.h2d(bt, dev, np.int32))
        st.bt_off.copy_(ops.h2d(off, dev, np.int64))
        st.kv_len.copy_(ops.h2d(kv_len, dev, np.int32))
        st.next_pos.copy_(ops.h2d(nxt, dev, np.int32))
        st.tok.zero_()
        st.tok[:B].copy_(self.tok)
        kvb = 256
        need = max(len(a.slots) - a.n_img for a in self.active)
        while kvb < need:
            kvb *= 2
        kvbx = 0
        if self.cross:
            xb, xo, xk, xm = self._cross_tables(Bp)
            st.bt_x[:len(xb)].copy_(ops.h2d(xb, dev, np.int32))
            st.bt_x_off.copy_(ops.h2d(xo, dev, np.int64))
            st.kv_len_x.copy_(ops.h2d(xk, dev, np.int32))
            st.xmask.copy_(ops.h2d(xm, dev, np.float32))
            kvbx = 256
            while kvbx < int(xk.max()):
                kvbx *= 2
        self._cur = (st, (kvb, kvbx))

    def _graph(self, st: _Static, key):
        g = st.graphs.get(key)
        if g is not None:
            return g
        dec = self.hp.decoder
        kvb, kvbx = key
        cross = (dict(bt=st.bt_x, bt_off=st.bt_x_off, kv_len=st.kv_len_x, max_kv_len=kvbx,
                      xmask=st.xmask) if self.cross else None)

        def body():
            ops.decode_advance(st.bt, st.bt_off, st.kv_len, st.next_pos, st.slot, st.pos)
            ids, logits = dec.decode_step(st.tok, self.arena.kv, st.slot, st.pos, st.bt,
                                          st.bt_off, st.kv_len, kvb, return_logits=True,
                                          cross=cross)
            st.tok.copy_(ids)
            return ids, logits
        # warm-up outside capture on a padding-only state (lazy allocations,
        # kernel attributes), then restore the real state
        state = (st.tok, st.bt_off, st.kv_len, st.next_pos, st.kv_len_x, st.xmask)
        saved = [t.clone() for t in state]
        st.bt_off.fill_(self.arena.n_slots)       # beyond any real slot list: scratch
        st.bt[self.arena.n_slots:self.arena.n_slots + self.SCRATCH_SEG].fill_(self._scratch)
        st.kv_len.zero_()
        st.kv_len_x.zero_()
        st.xmask.fill_(float("inf"))
        body()
        torch.cuda.current_stream().synchronize()
        for t, v in zip(state, saved):
            t.copy_(v)
        graph = torch.cuda.CUDAGraph()
        if self._pool is None:
            self._pool = torch.cuda.graph_pool_handle()
        with torch.cuda.graph(graph, pool=self._pool):
            ids, logits = body()
        st.graphs[key] = (graph, ids, logits)
        return st.graphs[key]

    def prepare(self) -> None:
        """Graph mode: load the current composition into its static buffers
        and capture its graph if new (the bench keeps this out of the timed
        step; step() does it itself otherwise)."""
        if self.graphs and self.active:
            if self._cur is None:
                self._load()
            self._graph(*self._cur)

    @ops.nvtx_stage("emm.decode_step")
    def step(self, return_logits: bool = False):
        """One decode step for every active request; retires the finished.
        Graph mode returns views of the graph's static output buffers: they
        hold this step's ids / logits until the next step() replays."""
        if not self.active:
            return None
        B = len(self.active)
        kv_now = np.array([a.kv_len + 1 for a in self.active], np.int64)
        if self.graphs:
            if self._cur is None:
                self._load()
            st, key = self._cur
            graph, ids_s, logits_s = self._graph(st, key)
            graph.replay()
            ids = ids_s[:B]
            out = (ids, logits_s[:B]) if return_logits else ids
        else:
            if self._tables is None:
                self._build_tables()
            bt, bt_off = self._tables
            slots = np.empty(B, np.int32)
            pos = np.empty(B, np.int32)
            for i, a in enumerate(self.active):
                slots[i] = a.slots[a.n_img + a.kv_len]
                pos[i] = a.next_pos
            dev = self.hp.device
            cross = None
            if self.cross:
                xb, xo, xk, xm = self._xtables
                cross = dict(bt=ops.h2d(xb, dev, np.int32), bt_off=ops.h2d(xo, dev, np.int64),
                             kv_len=ops.h2d(xk, dev, np.int32), max_kv_len=int(xk.max()),
                             xmask=ops.h2d(xm, dev, np.float32))
            out = self.hp.decoder.decode_step(self.tok, self.arena.kv, ops.h2d(slots, dev),
                                              ops.h2d(pos, dev), bt, bt_off,
                                              ops.h2d(kv_now.astype(np.int32), dev),
                                              int(kv_now.max()), return_logits=return_logits,
                                              cross=cross)
            ids = out[0] if return_logits else out
            self.tok = ids
        self.steps += 1
        self.generated += B
        self.kv_rows_read += int(kv_now.sum())
        for a in self.active:
            a.kv_len += 1
            a.next_pos += 1
            a.left -= 1
        done = [i for i, a in enumerate(self.active) if a.left == 0]
        if done:
            keep = [i for i, a in enumerate(self.active) if a.left > 0]
            for i in done:
                a = self.active[i]
                self.arena.release(a.slots)
                self.finished[a.rid] = a
            self.active = [self.active[i] for i in keep]
            self.tok = (ids[torch.as_tensor(keep, device=ids.device)] if keep
                        else ids[:0]).clone()
            self._tables = None
            self._cur = None
        return out

    def run(self, max_steps: int | None = None) -> int:
        """Step until every active request finished (or max_steps)."""
        n = 0
        while self.active and (max_steps is None or n < max_steps):
            self.step()
            n += 1
        return n


class DecodeStepModel:
    """Measured decode step time on this GPU, for the engine's mode B
    (B200Engine.decode_step_seconds replaces CostProfile.decode_step_time,
    costmodel.py:121-136, the way the prefill / encode hooks replace theirs).

    A decode step streams the decoder weights once (cost depends on the batch
    only) and every resident KV row of the batch once.  Both terms are
    measured here, once per GPU and model: t_fixed(b) = CUDA-graph replay of
    a real decode step of b requests with short contexts, for b in powers of
    two (interpolated between them), and the paged decode attention kernel's
    seconds per KV byte on a long-context batch.  step(b, kv) = t_fixed(b) +
    b * kv * bytes_per_kv_token * s_per_byte."""

    def __init__(self, hp, max_batch: int = 128):
        self.hp = hp
        dec = hp.shape.decoder
        self.kv_token_bytes = dec.kv_layers * 2 * dec.kv_dim * 2
        self.b_points = [b for b in DecodeSession.B_BUCKETS if b <= max_batch]
        self.t_fixed = {}
        self.s_per_byte = 0.0
        self._measure()

    def _time_replays(self, fn, reps: int = 10) -> float:
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps / 1e3

    def _measure(self):
        hp = self.hp
        dec = hp.shape.decoder
        ctx = 32
        bmax = self.b_points[-1]
        sess = DecodeSession(hp, bmax * (ctx + 4) + 16, graphs=True)
        sess.arena.kv.normal_()
        for b in self.b_points:
            # b padding-free requests of ctx tokens, static state rebuilt per replay
            slots = sess.arena.alloc(b * (ctx + 4)).reshape(b, ctx + 4)
            sess.active = [_Active(i, slots[i], ctx, ctx, 10 ** 9, []) for i in range(b)]
            sess.tok = torch.zeros(b, dtype=torch.int32, device=hp.device)
            sess._cur = None
            sess.prepare()
            st, kvb = sess._cur
            graph = st.graphs[kvb][0]
            kv0 = st.kv_len.clone()

            def one():
                st.kv_len.copy_(kv0)
                graph.replay()
            self.t_fixed[b] = self._time_replays(one)
            sess.arena.release(slots.reshape(-1))
            sess.active = []
        # attention seconds per KV byte (long contexts: bandwidth regime;
        # 16 x 4096 rows = 1 GB of K/V per layer at Qwen2-7B width)
        n_req, L = 16, 4096
        arena = DecodeArena(hp.shape, n_req * L, device=hp.device)
        arena.kv.normal_()
        q = torch.randn(n_req, dec.q_dim, device=hp.device).bfloat16()
        bt = torch.randperm(n_req * L, device=hp.device).to(torch.int32)
        bt_off = torch.arange(0, n_req * L + 1, L, dtype=torch.int64, device=hp.device)
        kv_len = torch.full((n_req,), L, dtype=torch.int32, device=hp.device)
        t = self._time_replays(lambda: ops.decode_attention(
            q, arena.kv[0, 0], arena.kv[0, 1], bt, bt_off, kv_len, dec.hkv, dec.hd, L))
        self.s_per_byte = t / (n_req * L * 2 * dec.kv_dim * 2)
        del arena

    def fixed(self, b: int) -> float:
        pts = self.b_points
        if b <= pts[0]:
            return self.t_fixed[pts[0]]
        for lo, hi in zip(pts, pts[1:]):
            if b <= hi:
                w = (b - lo) / (hi - lo)
                return (1 - w) * self.t_fixed[lo] + w * self.t_fixed[hi]
        # beyond the largest point: extrapolate the last segment's slope
        lo, hi = pts[-2], pts[-1]
        return self.t_fixed[hi] + (b - hi) * (self.t_fixed[hi] - self.t_fixed[lo]) / (hi - lo)

    def step_seconds(self, batch: int, kv_tokens_total: float) -> float:
        return self.fixed(max(1, batch)) + kv_tokens_total * self.kv_token_bytes * self.s_per_byte

    def as_dict(self) -> dict:
        return {"t_fixed_s": {str(k): v for k, v in self.t_fixed.items()},
                "attn_s_per_kv_byte": self.s_per_byte,
                "kv_token_bytes": self.kv_token_bytes}
