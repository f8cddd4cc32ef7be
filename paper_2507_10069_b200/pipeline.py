"""HotPath: the unified multimodal prefix cache feeding encode and prefill on
one B200 — the object B200Engine drives at the reference's stage entry
points (pkg/src/mmsim/engine.py:565 start_encode, :602 start_prefill,
:653-657 insert_prefix/release) and that bench.py times.

State on the device:
  * decoder / vision weights (bf16, random init of the named shapes)
  * the prefix KV pool  [L, 2, slots, kv_dim]  + its DeviceIndex (K2)
  * image slabs: content_hash -> [token_count, d] decoder-space embeddings,
    referenced by the image pool (C++ LRU, cache.py:31-74) and by every
    in-flight request that needs them (the pool has no
    pins, so a slab outlives its pool entry while a request holds it)
"""
from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import dataplane, ops
from ._lib import check, lib
from .cache import GpuUnifiedCache
from .encoder import make_encoder
from .cache import DEFAULT_CODEC
from .keys import TAG_IMG, KeySeq, request_keys
from .prefill import Decoder, mrope_positions
from .shapes import ModelShape, patch_grid
from .weights import init_decoder, init_vision


def synthetic_pixels(content_hash: str, height: int, width: int) -> np.ndarray:
    """Deterministic uint8 HWC pixels of an image identity."""
    return np.random.default_rng(int(content_hash[:16], 16)).integers(
        0, 256, (height, width, 3), dtype=np.uint8)


@dataclass
class BatchResult:
    next_ids: torch.Tensor               # int32 [n_req] on device
    matched_kv: torch.Tensor             # device-computed matched KV tokens (K2)
    computed_tokens: int = 0
    input_tokens: int = 0
    encode_images: int = 0
    flops: float = 0.0
    kv: object = None
    keep: object = None   # buffers other streams may still read (peer match outputs)


class HotPath:
    def __init__(self, shape: ModelShape, budget_tokens: int, image_fraction: float = 0.25,
                 device="cuda", seed: int = 0, max_batch_rows: int = 1 << 16,
                 weights: tuple | None = None, own_cache: bool = True):
        self.shape = shape
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(self.device):
            if weights is not None:  # (Wv, Wd) already on this device
                self.Wv, self.Wd = weights
            else:
                self.Wv = init_vision(shape, seed=seed, device=self.device)
                self.Wd = init_decoder(shape, seed=seed + 1, device=self.device)
            self.encoder = make_encoder(shape, self.Wv)
            self.decoder = Decoder(shape, self.Wd)
        self.budget_tokens, self.image_fraction = budget_tokens, image_fraction
        self.codec = DEFAULT_CODEC
        self.pixels: dict[str, torch.Tensor] = {}   # device-resident inputs (optional)
        # payloads staged by driver.identify_images for the current batch (a
        # lost slab is re-encoded from them, never from synthetic pixels)
        self.staged_pixels: dict[str, torch.Tensor] | None = None
        self._last = None
        self.cd = self.cache = self.index = None
        self._free_pools: list = []
        self._pool_users: dict = {}
        if own_cache:
            self.new_cache()

    # ------------------------------------------------------------ cache state
    def attach(self, cache: GpuUnifiedCache, pool: torch.Tensor | None = None) -> "CacheDevice":
        """Attach the device data plane (index + KV pool + image slabs) to a
        GpuUnifiedCache, e.g. one the unchanged reference driver created.
        Pools of caches that are gone (a finished engine run) are reused, so
        repeated runs on one HotPath do not accumulate 25 GB pools."""
        if pool is None:
            pool = self._free_pool(cache)
        with torch.cuda.device(self.device):
            cd = CacheDevice(self, cache, pool)
        p = cd.index.pool
        self._pool_users[id(p)] = self._pool_users.get(id(p), 0) + 1
        # the finalizer must not own the HotPath: hp.cd -> cd would keep the
        # referent reachable from its own finalizer and leak every model
        weakref.finalize(cd, HotPath._release_pool_of, weakref.ref(self), p)
        self._use(cd)
        return cd

    @staticmethod
    def _release_pool_of(hp_ref, pool: torch.Tensor) -> None:
        hp = hp_ref()
        if hp is not None:
            hp._release_pool(pool)

    def _release_pool(self, pool: torch.Tensor) -> None:
        n = self._pool_users.get(id(pool), 1) - 1
        if n > 0:
            self._pool_users[id(pool)] = n
            return
        self._pool_users.pop(id(pool), None)
        self._free_pools.append(pool)

    def _free_pool(self, cache: GpuUnifiedCache):
        dec = self.shape.decoder
        shape = (dec.kv_layers, 2, max(cache.prefixes.capacity, 1), dec.kv_dim)
        for attempt in range(2):
            for i, p in enumerate(self._free_pools):
                if tuple(p.shape) == shape:
                    return self._free_pools.pop(i)
            if attempt == 0:
                import gc
                gc.collect()   # engines hold their caches in reference cycles
        return None

    def new_cache(self) -> GpuUnifiedCache:
        """Fresh UnifiedCache + device index, reusing the previous KV pool."""
        pool = self.index.pool if getattr(self, "index", None) is not None else None
        self.cache = self.index = self.cd = None
        cache = GpuUnifiedCache(self.budget_tokens, self.image_fraction, codec=self.codec)
        self.attach(cache, pool)
        return cache

    def _use(self, cd: "CacheDevice"):
        self.cd, self.cache, self.index = cd, cd.cache, cd.index

    @property
    def slabs(self) -> dict:
        return self.cd.slabs

    # ------------------------------------------------------------- pixels
    def image_grid(self, token_count: int) -> tuple[int, int]:
        return patch_grid(token_count, self.shape.vision.merge)

    def stage_pixels(self, images) -> None:
        """Pre-stage pixels of `images` on the device (inputs resident in HBM)."""
        P = self.shape.vision.patch
        for img in images:
            if img.content_hash in self.pixels:
                continue
            gh, gw = self.image_grid(img.token_count)
            px = synthetic_pixels(img.content_hash, gh * P, gw * P)
            self.pixels[img.content_hash] = torch.from_numpy(px).to(self.device)

    # ------------------------------------------------------------- encode
    @ops.nvtx_stage("emm.encode")
    def encode(self, images, now: float | None = None, host_pixels: dict | None = None,
               verify_digest: bool = False, cd: "CacheDevice | None" = None,
               device_pixels: dict | None = None) -> int:
        """K1 + K4 for the missed images of an encode job: pixels -> slabs.
        Returns the number of images encoded.  `host_pixels` (pinned uint8
        tensors) are copied H2D here (end-to-end mode); `device_pixels` are
        payloads already staged on this device (driver.identify_images)."""
        slabs = (cd or self.cd).slabs
        todo = [img for img in images if img.content_hash not in slabs]
        seen, uniq = set(), []
        for img in todo:
            if img.content_hash not in seen:
                seen.add(img.content_hash)
                uniq.append(img)
        if not uniq:
            return 0
        P = self.shape.vision.patch
        grids = [self.image_grid(img.token_count) for img in uniq]
        sizes = [gh * P * gw * P * 3 for gh, gw in grids]
        offs = np.zeros(len(uniq) + 1, np.int64)
        np.cumsum([(s + 15) // 16 * 16 for s in sizes], out=offs[1:])
        buf = torch.empty(int(offs[-1]), dtype=torch.uint8, device=self.device)
        for i, img in enumerate(uniq):
            src = None
            if device_pixels is not None and img.content_hash in device_pixels:
                src = device_pixels[img.content_hash]
            elif host_pixels is not None:
                src = host_pixels[img.content_hash]
            else:
                src = self.pixels.get(img.content_hash)
                if src is None:
                    gh, gw = grids[i]
                    src = torch.from_numpy(synthetic_pixels(img.content_hash, gh * P, gw * P))
            buf[offs[i]:offs[i] + sizes[i]].copy_(src.reshape(-1), non_blocking=True)
        if verify_digest:
            self.last_digests = dataplane.pixel_digest_ranges(buf, offs[:-1],
                                                              np.asarray(sizes, np.int64))
        rows, spans = self.encoder.encode(buf, offs[:-1], grids)
        for img, (a, b) in zip(uniq, spans):
            assert b - a == img.token_count, "encoder must emit token_count rows (H5)"
            slabs[img.content_hash] = rows[a:b]
        return len(uniq)

    # ------------------------------------------------------------- prefill
    @ops.nvtx_stage("emm.prefill")
    def prefill(self, reqs, cached_prefix, cd: "CacheDevice | None" = None) -> BatchResult:
        """K1 + K2 + K3 + decoder for a batch whose cached_prefix[r] was set
        by the host tree (consult_prefix_cache, engine.py:539-547).  Leaves
        the batch's KV registered as the scatter source for insert()."""
        dec = self.shape.decoder
        dev = self.device
        cd = cd or self.cd
        index = cd.index
        n = len(reqs)
        keys_l, w_l = zip(*[request_keys(self.codec, r) for r in reqs])
        totals = np.array([int(w.sum()) for w in w_l], np.int64)
        P_ = np.asarray(cached_prefix, np.int64)
        S_ = totals - P_
        assert (S_ >= 1).all(), "at least one token is recomputed (engine.py:546)"
        # K1 + K2: block hashes, device match, block tables for the prefix
        if index.device == dev:
            batch = dataplane.block_hash(list(keys_l), list(w_l), device=dev)
            res = index.match(batch, P_)
        else:
            # the group's index and pool live on another GPU: hash + match
            # there, then this GPU's stream waits for the block table and
            # gathers the prefix rows peer-to-peer (SURVEY §8e exchange 2)
            with torch.cuda.device(index.device):
                batch = dataplane.block_hash(list(keys_l), list(w_l), device=index.device)
                res = index.match(batch, P_)
                ev = torch.cuda.Event()
                ev.record()
            torch.cuda.current_stream(dev).wait_event(ev)
        # request KV buffer rows
        row0 = np.zeros(n, np.int64)
        np.cumsum(totals[:-1], out=row0[1:])
        R = int(totals.sum())
        req_kv = torch.empty(dec.kv_layers, 2, R, dec.kv_dim, device=dev, dtype=torch.bfloat16)
        # K3: gather cached prefix KV from the paged pool
        n_pref = int(P_.sum())
        if n_pref:
            dst_rows = ops.h2d(np.concatenate(
                [np.arange(row0[r], row0[r] + P_[r], dtype=np.int32) for r in range(n)]), dev)
            dataplane.kv_copy_rows(index.pool, res["bt"][:n_pref], req_kv, dst_rows, n_pref)
        if dec.cross:
            return self._prefill_cross(reqs, keys_l, w_l, totals, P_, row0, req_kv, res, cd,
                                       batch)
        # suffix token sources: text embedding rows or image slab rows
        S_total = int(S_.sum())
        src_ptr = np.empty(S_total, np.int64)
        kv_row = np.empty(S_total, np.int32)
        pos = np.empty(S_total, np.int32)
        mrope = bool(dec.mrope_section)
        if mrope:
            pos_h = np.empty(S_total, np.int32)
            pos_w = np.empty(S_total, np.int32)
        last_rows = np.empty(n, np.int32)
        # H9: the image pool has no pins, so a slab may have been evicted
        # between this request's image hit and its prefill -> re-encode it
        need = {img.content_hash: img for r, req in enumerate(reqs) for img in req.images}
        lost = [img for h, img in need.items() if h not in cd.slabs]
        if lost:
            self.encode(lost, cd=cd, device_pixels=self.staged_pixels)
        emb = self.Wd["embed"]
        emb_base, row_bytes = emb.data_ptr(), dec.d * 2
        o = 0
        for r, req in enumerate(reqs):
            keys, w = keys_l[r], w_l[r]
            p0, tot = int(P_[r]), int(totals[r])
            t = np.arange(p0, tot, dtype=np.int64)
            cum = np.cumsum(w)
            sym = np.searchsorted(cum, t, side="right")
            within = t - (cum[sym] - w[sym])
            k_sym = keys[sym]
            is_img = (k_sym >> np.uint64(62)) == np.uint64(TAG_IMG)
            ptrs = emb_base + (k_sym % np.uint64(dec.vocab)).astype(np.int64) * row_bytes
            if is_img.any():
                for j in np.unique(sym[is_img]):
                    h = self.codec.symbol(int(keys[j]))[1]
                    slab = cd.slabs.get(h)
                    if slab is None:
                        raise RuntimeError(f"image {h} has no encoded slab for prefill")
                    m = sym == j
                    ptrs[m] = slab.data_ptr() + within[m] * row_bytes
            L = tot - p0
            src_ptr[o:o + L] = ptrs
            kv_row[o:o + L] = row0[r] + t
            if mrope:
                pt, ph, pw = mrope_positions(keys, w)
                pos[o:o + L], pos_h[o:o + L], pos_w[o:o + L] = pt[p0:], ph[p0:], pw[p0:]
            else:
                pos[o:o + L] = t
            last_rows[r] = o + L - 1
            o += L
        to_dev = lambda a: ops.h2d(a, dev)
        x = torch.empty(S_total, dec.d, device=dev, dtype=torch.bfloat16)
        ops.gather_rows(to_dev(src_ptr), x)
        meta = ops.AttnMeta(np.concatenate([[0], np.cumsum(S_)[:-1]]), S_, row0, totals,
                            dec.hq, causal=True, device=dev)
        ids = self.decoder.forward(x, req_kv, to_dev(kv_row), to_dev(pos), meta,
                                   to_dev(last_rows),
                                   pos_h=to_dev(pos_h) if mrope else None,
                                   pos_w=to_dev(pos_w) if mrope else None)
        batch_kv = BatchKV(req_kv=req_kv, keys=keys_l, weights=w_l, row0=row0,
                           rids=[getattr(r, "id", i) for i, r in enumerate(reqs)])
        self._last = batch_kv
        flops = S_total * dec.linear_flops_per_token() + meta.flops(dec.hd) * dec.layers \
            + n * 2.0 * dec.d * dec.vocab
        return BatchResult(next_ids=ids, matched_kv=res["matched_kv"], computed_tokens=S_total,
                           input_tokens=int(totals.sum()), flops=flops, kv=batch_kv,
                           keep=(batch, res) if index.device != dev else None)

    def _prefill_cross(self, reqs, keys_l, w_l, totals, P_, row0, req_kv, res, cd, batch):
        """Prefill of a cross-attention model (Llama-3.2-Vision).

        The unified sequence puts a request's images first (engine.py:448-
        461); here image tokens take no self-attention positions.  The KV
        row of an image token holds that image's cross-attention K/V (planes
        0..n_cross-1: k_norm'ed keys, values), a text token's row its
        self-attention K/V (planes = self layers), so the token-granular
        prefix cache, its K3 gather and the insert scatter carry both
        unchanged.  Uncached image tokens get their cross K/V projected from
        the image slab here; text tokens run the 40-layer stack with the
        cross layers on the rows of requests that have images (those come
        first in the token order)."""
        dec = self.shape.decoder
        dev = self.device
        n = len(reqs)
        emb = self.Wd["embed"]
        emb_base, row_bytes = emb.data_ptr(), dec.d * 2
        need = {img.content_hash: img for req in reqs for img in req.images}
        lost = [img for h, img in need.items() if h not in cd.slabs]
        if lost:
            self.encode(lost, cd=cd, device_pixels=self.staged_pixels)
        n_img = np.zeros(n, np.int64)
        img_ptr, img_row = [], []
        for r in range(n):
            keys, w = keys_l[r], w_l[r]
            is_img = (keys >> np.uint64(62)) == np.uint64(TAG_IMG)
            k_img = int(is_img.sum())
            if k_img and not is_img[:k_img].all():
                raise ValueError("cross-attention model: images must precede text "
                                 "(engine.py:448-461 order)")
            n_img[r] = int(w[:k_img].sum())
            if n_img[r] >= totals[r]:
                raise ValueError("cross-attention model: a request needs a text token")
            for j in range(k_img):          # uncached image tokens -> cross K/V
                t0 = int(w[:j].sum())
                lo, hi = max(int(P_[r]), t0), t0 + int(w[j])
                if lo >= hi:
                    continue
                slab = cd.slabs.get(self.codec.symbol(int(keys[j]))[1])
                if slab is None:
                    raise RuntimeError("image has no encoded slab for prefill")
                img_ptr.append(slab.data_ptr() + np.arange(lo - t0, hi - t0,
                                                           dtype=np.int64) * row_bytes)
                img_row.append(np.arange(row0[r] + lo, row0[r] + hi, dtype=np.int32))
        n_cross = len(dec.cross)
        T_img = int(sum(len(x) for x in img_row))
        flops = 0.0
        if T_img:
            x_img = torch.empty(T_img, dec.d, device=dev, dtype=torch.bfloat16)
            ops.gather_rows(ops.h2d(np.concatenate(img_ptr), dev), x_img)
            kvs = torch.empty(n_cross, 2, T_img, dec.kv_dim, device=dev, dtype=torch.bfloat16)
            for ci, li in enumerate(dec.cross):
                L = self.Wd["layers"][li]
                ops.gemm(x_img, L["xk_w"], out=kvs[ci, 0])
                ops.gemm(x_img, L["xv_w"], out=kvs[ci, 1])
                kh = kvs[ci, 0].view(T_img * dec.hkv, dec.hd)
                ops.norm(kh, self.decoder.ones_hd, None, dec.eps, out=kh)
            rows_d = ops.h2d(np.concatenate(img_row), dev)
            dataplane.kv_copy_rows(kvs, None, req_kv[:n_cross], rows_d, T_img)
            # the self planes of an image row are never attended to, but a
            # 128-key block of a neighbouring request's self attention can
            # cover them (masked, P = 0) and 0 * NaN garbage would poison the
            # PV product: zero them (one K3 launch from a single zero row);
            # the pool and the decode arena then inherit zeros
            nz = dec.kv_layers - n_cross
            if nz > 0:
                if getattr(self, "_zero_row", None) is None or self._zero_row.shape[0] != nz:
                    self._zero_row = torch.zeros(nz, 2, 1, dec.kv_dim, device=dev,
                                                 dtype=torch.bfloat16)
                zidx = torch.zeros(T_img, dtype=torch.int32, device=dev)
                dataplane.kv_copy_rows(self._zero_row, zidx, req_kv[n_cross:], rows_d, T_img)
            flops += T_img * dec.cross_kv_flops_per_image_token()
        # text suffix rows, requests with images first
        order = sorted(range(n), key=lambda r: (n_img[r] == 0, r))
        t_ptr, t_row, t_pos = [], [], []
        q_start = np.zeros(n, np.int64)
        q_len = np.zeros(n, np.int64)
        last_rows = np.zeros(n, np.int32)
        o = 0
        for r in order:
            keys, w = keys_l[r], w_l[r]
            lo = max(int(P_[r]), int(n_img[r]))
            t = np.arange(lo, int(totals[r]), dtype=np.int64)
            cum = np.cumsum(w)
            sym = np.searchsorted(cum, t, side="right")
            t_ptr.append(emb_base + (keys[sym] % np.uint64(dec.vocab)).astype(np.int64) * row_bytes)
            t_row.append((row0[r] + t).astype(np.int32))
            t_pos.append((t - n_img[r]).astype(np.int32))
            q_start[r], q_len[r] = o, len(t)
            o += len(t)
            last_rows[r] = o - 1
        S_text = o
        img_reqs = [r for r in order if n_img[r] > 0]
        n_img_rows = int(sum(q_len[r] for r in img_reqs))
        to_dev = lambda a: ops.h2d(a, dev)
        x = torch.empty(S_text, dec.d, device=dev, dtype=torch.bfloat16)
        ops.gather_rows(to_dev(np.concatenate(t_ptr)), x)
        n_text = totals - n_img
        meta_self = ops.AttnMeta(q_start, q_len, row0 + n_img, n_text, dec.hq, causal=True,
                                 device=dev)
        meta_cross = None
        if img_reqs:
            ir = np.asarray(img_reqs)
            meta_cross = ops.AttnMeta(q_start[ir], q_len[ir], row0[ir], n_img[ir], dec.hq,
                                      causal=False, device=dev)
        ids = self.decoder.forward_cross(x, req_kv, to_dev(np.concatenate(t_row)),
                                         to_dev(np.concatenate(t_pos)), meta_self, meta_cross,
                                         n_img_rows, to_dev(last_rows))
        batch_kv = BatchKV(req_kv=req_kv, keys=keys_l, weights=w_l, row0=row0,
                           rids=[getattr(r, "id", i) for i, r in enumerate(reqs)])
        self._last = batch_kv
        flops += S_text * dec.linear_flops_per_token() + meta_self.flops(dec.hd) * dec.kv_layers \
            + (meta_cross.flops(dec.hd) * n_cross if meta_cross is not None else 0.0) \
            + n * 2.0 * dec.d * dec.vocab
        computed = int((totals - P_).sum())
        return BatchResult(next_ids=ids, matched_kv=res["matched_kv"], computed_tokens=computed,
                           input_tokens=int(totals.sum()), flops=flops, kv=batch_kv,
                           keep=(batch, res) if cd.index.device != dev else None)

    # ------------------------------------------------------------- insert
    def prepare_insert(self, batch_kv, cd: "CacheDevice | None" = None):
        """Register a prefill batch's KV buffer(s) as the scatter source of its
        requests' insert_prefix calls (matched by each sequence's final
        block hash).  `batch_kv` may be a list: the sub-batches of one
        prefill batch split across GPUs (scattered peer-to-peer)."""
        index = (cd or self.cd).index
        parts = list(batch_kv) if isinstance(batch_kv, (list, tuple)) else [batch_kv]
        index.set_request_buffer(parts[0].req_kv)
        index.clear_kv_sources()
        for i, bk in enumerate(parts):
            buf = 0 if i == 0 else index.add_request_buffer(bk.req_kv)
            for r in range(len(bk.keys)):
                h0, h1 = host_last_hash(bk.keys[r], bk.weights[r])
                index.set_kv_source(h0, h1, int(bk.row0[r]), buf)

    def finish_insert(self, batch_kv: "BatchKV | None" = None, cd: "CacheDevice | None" = None):
        """Flush the coalesced index updates + KV scatter, then drop sources."""
        index = (cd or self.cd).index
        with torch.cuda.device(index.device):
            index.flush()
        index.clear_kv_sources()

    def insert_batch(self, reqs, now: float, batch_kv: "BatchKV | None" = None,
                     cd: "CacheDevice | None" = None) -> list[int]:
        """insert_prefix of every request of a prefill batch (engine.py:653-656);
        the KV scatter into the pool rides on the flush."""
        cd = cd or self.cd
        bk = batch_kv or self._last
        self.prepare_insert(bk, cd)
        out = []
        for r in range(len(reqs)):
            seq = KeySeq(bk.keys[r], bk.weights[r], cd.cache.codec)
            out.append(cd.cache.insert_prefix(seq, seq.weights, now))
        return out

    @property
    def _req_kv(self):
        return self._last.req_kv if self._last is not None else None

    def release_batch_kv(self, cd: "CacheDevice | None" = None):
        self.finish_insert(cd=cd)
        self._last = None


@dataclass
class BatchKV:
    """A prefill batch's request KV buffer [L, 2, rows, kv_dim] and the keys
    needed to scatter it into the pool at insert time."""
    req_kv: torch.Tensor
    keys: tuple
    weights: tuple
    row0: np.ndarray
    rids: list = field(default_factory=list)


class CacheDevice:
    """Device state of one GpuUnifiedCache (one modality group): the GPU
    prefix index with its paged KV pool, and the image slabs."""

    def __init__(self, hp: "HotPath", cache: GpuUnifiedCache, pool=None):
        dec = hp.shape.decoder
        self.cache = cache
        self.index = dataplane.DeviceIndex(cache, n_layers=dec.kv_layers, kv_dim=dec.kv_dim,
                                           device=hp.device, pool=pool)
        self.slabs: dict[str, torch.Tensor] = {}
        cache.listeners.append(self._on_image_event)
        cache.device_state = self

    def _on_image_event(self, kind, content_hash, ok, evicted):
        # pool evictions drop the pool's reference only; requests in flight
        # keep theirs through the tensors they captured
        for h in evicted:
            self.slabs.pop(h, None)


def host_last_hash(keys: np.ndarray, w: np.ndarray) -> tuple[int, int]:
    """Block hash of the last symbol (host restatement in libemm)."""
    n = len(keys)
    k = np.ascontiguousarray(keys, np.uint64)
    ww = np.ascontiguousarray(w, np.int64)
    h0 = np.empty(max(n, 1), np.uint64)
    h1 = np.empty(max(n, 1), np.uint64)
    check(lib.emm_prefix_hashes_host(k.ctypes.data, ww.ctypes.data, n, h0.ctypes.data,
                                     h1.ctypes.data))
    return int(h0[n - 1]), int(h1[n - 1])


class HotPathSet:
    """The hot path on every GPU of one box: one HotPath per logical GPU
    (instance i -> GPU i mod n), weights replicated once per
    physical device.  `devices` may repeat a physical GPU (e.g. [0, 0]) to
    exercise the multi-GPU code paths — job splitting, peer gathers, KV
    hand-offs, multi-buffer scatters — on a one-GPU box; logical GPUs that
    share a physical one run their sub-jobs back to back on its stream."""

    def __init__(self, shape: ModelShape, budget_tokens: int, image_fraction: float = 0.25,
                 devices=None, seed: int = 0):
        if devices is None:
            devices = list(range(torch.cuda.device_count()))
        self.shape = shape
        self.paths: list[HotPath] = []
        shared: dict[int, tuple] = {}
        for d in devices:
            dev = torch.device("cuda", int(d))
            hp = HotPath(shape, budget_tokens, image_fraction, device=dev, seed=seed,
                         weights=shared.get(dev.index), own_cache=False)
            shared.setdefault(dev.index, (hp.Wv, hp.Wd))
            self.paths.append(hp)
        phys = sorted(shared)
        if len(phys) > 1:
            import ctypes
            from . import _lib
            _lib.declare_more({"emm_enable_peer_access": (ctypes.c_int, [ctypes.c_int,
                                                                         ctypes.c_int])})
            for a in phys:
                for b in phys:
                    if a != b:
                        check(lib.emm_enable_peer_access(a, b))

    def __len__(self):
        return len(self.paths)

    def __getitem__(self, i) -> HotPath:
        return self.paths[i]

    @property
    def codec(self):
        return self.paths[0].codec


def split_balanced(costs, n: int) -> list[list[int]]:
    """Longest-processing-time split of items with `costs` over n workers;
    each worker's item indices stay in their original order."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0] * n
    out: list[list[int]] = [[] for _ in range(n)]
    for i in order:
        w = min(range(n), key=lambda k: (load[k], k))
        load[w] += costs[i]
        out[w].append(i)
    return [sorted(x) for x in out]
