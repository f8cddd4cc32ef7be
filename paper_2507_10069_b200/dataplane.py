"""Device data plane of the unified cache: K1 block hashes / pixel digests,
the GPU prefix index (K2, block tables) and paged KV row copies (K3/K6).

All work runs in libemm.so kernels on the current torch stream; torch only
allocates the buffers.  The host control plane (GpuUnifiedCache) stays the
authority for decisions; `DeviceIndex` mirrors it (dataplane.cu).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .ops import _stream, h2d

EMM_E_OOM = 4  # include/emm.h

vp, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64
P = C.POINTER

_lib.declare_more({
    "emm_block_hash": (C.c_int, [vp, vp, vp, i64, vp, vp, vp, vp]),
    "emm_pixel_digest_scratch_bytes": (i64, [vp, i64]),
    "emm_pixel_digest": (C.c_int, [vp, vp, vp, vp, vp, i64, vp, vp, vp]),
    "emm_index_attach": (C.c_int, [vp, C.c_int, i64, i64, i64, P(vp)]),
    "emm_index_set_stream": (C.c_int, [vp, vp]),
    "emm_index_set_kv_source": (C.c_int, [vp, u64, u64, i64]),
    "emm_index_set_kv_source_buf": (C.c_int, [vp, u64, u64, C.c_int, i64]),
    "emm_index_add_request_buffer": (C.c_int, [vp, vp, i64, C.POINTER(C.c_int)]),
    "emm_index_clear_kv_sources": (C.c_int, [vp]),
    "emm_index_set_kv_geometry": (C.c_int, [vp, vp, i64, vp, i64, i64, i64]),
    "emm_index_flush": (C.c_int, [vp, vp]),
    "emm_index_match": (C.c_int, [vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp]),
    "emm_index_info": (C.c_int, [vp, P(i64)]),
    "emm_index_tok_slots_host": (C.c_int, [vp, i64, i64, vp]),
    "emm_kv_copy_rows": (C.c_int, [vp, i64, vp, vp, i64, vp, i64, i64, i64, vp]),
    "emm_kv_copy_planes_ce": (C.c_int, [vp, i64, vp, i64, i64, i64, i64, vp]),
    "emm_kv_checksum": (C.c_int, [vp, i64, vp, i64, i64, i64, vp, vp]),
})


def _dev_i64(a, device):
    return h2d(a, device, np.int64)


class SeqBatch:
    """CSR batch of unified sequences (keys, weights) resident on the device."""

    def __init__(self, key_list, weight_list, device="cuda"):
        lens = [len(k) for k in key_list]
        off = np.zeros(len(lens) + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        keys = np.concatenate(key_list).astype(np.uint64) if lens else np.zeros(0, np.uint64)
        w = np.concatenate(weight_list).astype(np.int64) if lens else np.zeros(0, np.int64)
        self.n = len(lens)
        self.off_host = off
        self.keys = h2d(keys.view(np.int64), device)
        self.weights = h2d(w, device)
        self.off = h2d(off, device)
        total = int(off[-1])
        self.h0 = torch.empty(max(total, 1), dtype=torch.int64, device=device)
        self.h1 = torch.empty(max(total, 1), dtype=torch.int64, device=device)
        self.cumw = torch.empty(max(total, 1), dtype=torch.int64, device=device)

    def hash(self):
        """K1: per-symbol prefix (block) hashes and KV-token ends."""
        check(lib.emm_block_hash(self.keys.data_ptr(), self.weights.data_ptr(),
                                 self.off.data_ptr(), self.n, self.h0.data_ptr(),
                                 self.h1.data_ptr(), self.cumw.data_ptr(), _stream()))
        return self


def block_hash(key_list, weight_list, device="cuda") -> SeqBatch:
    return SeqBatch(key_list, weight_list, device).hash()


def pixel_digests(images: list[torch.Tensor]) -> torch.Tensor:
    """K1: 122-bit content digests of uint8 device images -> int64 [n, 2]
    (packs the images 16-byte aligned into one buffer, one launch pair)."""
    dev = images[0].device
    sizes = np.array([int(t.numel()) for t in images], np.int64)
    starts = np.zeros(len(images), np.int64)
    if len(images) > 1:
        starts[1:] = np.cumsum((sizes[:-1] + 15) // 16 * 16)
    total = int(starts[-1] + sizes[-1]) if len(images) else 0
    buf = torch.empty(max(total, 16), dtype=torch.uint8, device=dev)
    for i, t in enumerate(images):
        buf[starts[i]:starts[i] + sizes[i]].copy_(t.reshape(-1))
    return pixel_digest_ranges(buf, starts, sizes)


def pixel_digest_ranges(buf: torch.Tensor, starts: np.ndarray, sizes: np.ndarray) -> torch.Tensor:
    """Digest of byte ranges [starts[i], starts[i]+sizes[i]) of `buf`."""
    n = len(starts)
    dev = buf.device
    st_h = np.ascontiguousarray(starts, dtype=np.int64)
    ln_h = np.ascontiguousarray(sizes, dtype=np.int64)
    st_d, ln_d = _dev_i64(st_h, dev), _dev_i64(ln_h, dev)
    scratch = torch.empty(int(lib.emm_pixel_digest_scratch_bytes(ln_h.ctypes.data, n)),
                          dtype=torch.uint8, device=dev)
    out = torch.empty(n, 2, dtype=torch.int64, device=dev)
    check(lib.emm_pixel_digest(buf.data_ptr(), st_d.data_ptr(), ln_d.data_ptr(), st_h.ctypes.data,
                               ln_h.ctypes.data, n, scratch.data_ptr(), out.data_ptr(),
                               _stream()))
    out._emm_keepalive = (st_d, ln_d, scratch)
    return out


def kv_copy_rows(src: torch.Tensor, src_rows, dst: torch.Tensor, dst_rows, n_rows: int):
    """K3/K6: for every layer and K/V half, dst[l,h,dst_rows[i]] = src[l,h,src_rows[i]].

    src/dst: [L, 2, rows, row_elems] (any dtype, contiguous rows);
    *_rows: int32 device tensors or None (identity)."""
    assert src.dim() == 4 and dst.dim() == 4 and src.shape[0] == dst.shape[0]
    assert src.shape[1] == 2 and dst.shape[1] == 2 and src.shape[3] == dst.shape[3]
    row_bytes = src.shape[3] * src.element_size()
    from .ops import TIMER
    TIMER.wrap("kv_gather", 2.0 * n_rows * row_bytes * 2 * src.shape[0],
               lambda: check(lib.emm_kv_copy_rows(
                   src.data_ptr(), src.stride(1) * src.element_size(),
                   None if src_rows is None else src_rows.data_ptr(), dst.data_ptr(),
                   dst.stride(1) * dst.element_size(),
                   None if dst_rows is None else dst_rows.data_ptr(), n_rows, row_bytes,
                   src.shape[0], _stream())))


def kv_copy_planes_ce(src: torch.Tensor, dst: torch.Tensor, n_rows: int):
    """K6 on the copy engines: dst[l, h, :n_rows] = src[l, h, :n_rows] for every
    layer / K-V plane as one strided DMA on the current stream (peer-to-peer
    when the tensors live on different GPUs).  src/dst: [L, 2, rows, row_elems]
    with contiguous rows inside each plane."""
    assert src.dim() == 4 and dst.dim() == 4 and src.shape[0] == dst.shape[0]
    assert src.shape[1] == 2 and dst.shape[1] == 2 and src.shape[3] == dst.shape[3]
    assert src.stride(3) == 1 and dst.stride(3) == 1
    assert src.stride(2) == src.shape[3] and dst.stride(2) == dst.shape[3]
    assert src.stride(0) == 2 * src.stride(1) and dst.stride(0) == 2 * dst.stride(1)
    row_bytes = src.shape[3] * src.element_size()
    from .ops import TIMER
    TIMER.wrap("kv_copy_ce", 2.0 * n_rows * row_bytes * 2 * src.shape[0],
               lambda: check(lib.emm_kv_copy_planes_ce(
                   src.data_ptr(), src.stride(1) * src.element_size(), dst.data_ptr(),
                   dst.stride(1) * dst.element_size(), n_rows, row_bytes, src.shape[0],
                   _stream())))


def kv_checksum(planes: torch.Tensor, rows, n_rows: int) -> torch.Tensor:
    """K6 verification: a device uint64 (as int64 [1]) =
    sum over (layer, K/V) planes p and rows i < n_rows of XXH64(row bytes,
    seed p << 32 | i), the row planes[l, h, rows[i]] (rows: int32 device tensor
    or None = identity).  Both sides of an exact copy give the same value."""
    assert planes.dim() == 4 and planes.shape[1] == 2 and planes.stride(3) == 1
    assert planes.stride(0) == 2 * planes.stride(1), "planes must be evenly strided"
    out = torch.empty(1, dtype=torch.int64, device=planes.device)
    check(lib.emm_kv_checksum(planes.data_ptr(), planes.stride(1) * planes.element_size(),
                              None if rows is None else rows.data_ptr(), int(n_rows),
                              planes.shape[3] * planes.element_size(), planes.shape[0],
                              out.data_ptr(), _stream()))
    return out


def kv_move(src: torch.Tensor, dst: torch.Tensor, n_rows: int, transport: str = "kernel"):
    """K6 transport switch: "kernel" = SM-driven row copy (peer loads/stores),
    "copy_engine" = one strided DMA on the copy engines."""
    if transport == "copy_engine":
        kv_copy_planes_ce(src, dst, n_rows)
    elif transport == "kernel":
        kv_copy_rows(src, None, dst, None, n_rows)
    else:
        raise ValueError(f"unknown K6 transport {transport!r}")


class DeviceIndex:
    """GPU mirror of a GpuUnifiedCache's prefix tree plus its paged KV pool.

    pool: [n_layers, 2, n_slots, kv_dim] bf16; slots are handed out by the
    index as the host tree inserts nodes and returned when it evicts them.
    """

    def __init__(self, cache, n_layers: int, kv_dim: int, device="cuda", n_slots=None,
                 dtype=torch.bfloat16, alloc_pool: bool = True, pool: torch.Tensor | None = None):
        cap = cache.prefixes.capacity
        n_slots = n_slots if n_slots is not None else max(cap, 1)
        self.cache = cache
        self.device = torch.device(device)
        self.n_layers, self.kv_dim, self.n_slots = n_layers, kv_dim, n_slots
        h = C.c_void_p()
        check(lib.emm_index_attach(cache._h, self.device.index or 0, max(cap, 1),
                                   4 * max(cap, 1) + 4096, n_slots, C.byref(h)))
        self._h = h
        cache.device = self
        if pool is not None:
            assert pool.shape == (n_layers, 2, n_slots, kv_dim) and pool.dtype == dtype
            self.pool = pool  # reuse the HBM of a previous index (fresh cache, same pool)
        else:
            self.pool = (torch.empty(n_layers, 2, n_slots, kv_dim, dtype=dtype,
                                     device=self.device) if alloc_pool else None)
        self._req = None
        self._extra = []
        self.set_stream()

    def set_stream(self, stream=None):
        s = stream if stream is not None else _stream()
        check(lib.emm_index_set_stream(self._h, s))

    def set_request_buffer(self, req_kv: torch.Tensor):
        """Register the batch's request KV buffer [L, 2, rows, kv_dim] as the
        scatter source for subsequent insert_prefix calls."""
        assert self.pool is not None
        assert req_kv.shape[0] == self.n_layers and req_kv.shape[3] == self.kv_dim
        self._req = req_kv
        self._extra = []
        es = req_kv.element_size()
        check(lib.emm_index_set_kv_geometry(
            self._h, self.pool.data_ptr(), self.pool.stride(1) * es, req_kv.data_ptr(),
            req_kv.stride(1) * es, self.kv_dim * es, self.n_layers))

    def add_request_buffer(self, req_kv: torch.Tensor) -> int:
        """Register one more request KV buffer (a sub-batch prefilled on
        another GPU; the scatter reads it peer-to-peer).  Returns its id."""
        assert self._req is not None, "set_request_buffer first"
        assert req_kv.shape[0] == self.n_layers and req_kv.shape[3] == self.kv_dim
        assert req_kv.stride(2) == self.kv_dim and req_kv.dtype == self._req.dtype
        b = C.c_int()
        check(lib.emm_index_add_request_buffer(self._h, req_kv.data_ptr(),
                                               req_kv.stride(1) * req_kv.element_size(),
                                               C.byref(b)))
        self._extra.append(req_kv)
        return b.value

    def set_kv_source(self, h0_last: int, h1_last: int, row0: int, buffer: int = 0):
        if buffer == 0:
            check(lib.emm_index_set_kv_source(self._h, h0_last & (2**64 - 1),
                                              h1_last & (2**64 - 1), int(row0)))
        else:
            check(lib.emm_index_set_kv_source_buf(self._h, h0_last & (2**64 - 1),
                                                  h1_last & (2**64 - 1), int(buffer), int(row0)))

    def clear_kv_sources(self):
        check(lib.emm_index_clear_kv_sources(self._h))

    def flush(self):
        with torch.cuda.device(self.device):
            rc = lib.emm_index_flush(self._h, _stream())
            if rc == EMM_E_OOM:
                # the staging buffer is cudaMalloc'ed outside torch's caching
                # allocator: hand torch's cached blocks back and retry once
                torch.cuda.empty_cache()
                rc = lib.emm_index_flush(self._h, _stream())
            check(rc)

    def info(self) -> dict:
        out = (C.c_int64 * 6)()
        check(lib.emm_index_info(self._h, out))
        return {"live_symbols": out[0], "tombstones": out[1], "table_capacity": out[2],
                "free_slots": out[3], "device_error": out[4], "free_virtual": out[5]}

    def match(self, batch: SeqBatch, want_kv) -> dict:
        """K2 over a hashed SeqBatch: matched symbols / KV and block tables."""
        dev = self.device
        want = np.ascontiguousarray(want_kv, dtype=np.int64)
        bt_off = np.zeros(batch.n + 1, np.int64)
        np.cumsum(want, out=bt_off[1:])
        want_d = _dev_i64(want, dev)
        bt_off_d = _dev_i64(bt_off, dev)
        matched_sym = torch.empty(batch.n, dtype=torch.int64, device=dev)
        matched_kv = torch.empty(batch.n, dtype=torch.int64, device=dev)
        sym_v = torch.empty_like(batch.h0)
        bt = torch.empty(max(int(bt_off[-1]), 1), dtype=torch.int32, device=dev)
        check(lib.emm_index_match(self._h, batch.h0.data_ptr(), batch.h1.data_ptr(),
                                  batch.cumw.data_ptr(), batch.off.data_ptr(), batch.n,
                                  want_d.data_ptr(), bt_off_d.data_ptr(),
                                  matched_sym.data_ptr(), matched_kv.data_ptr(),
                                  sym_v.data_ptr(), bt.data_ptr(), _stream()))
        return {"matched_sym": matched_sym, "matched_kv": matched_kv, "bt": bt,
                "bt_off": bt_off, "_keep": (want_d, bt_off_d, sym_v)}
