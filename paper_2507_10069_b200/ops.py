"""torch-tensor front end of the device entry points in libemm.so.

PyTorch provides device memory and streams only; every op here launches one
of our sm_100a kernels through the C ABI.  There is no fallback: calling an
op on a non-CUDA tensor raises.
"""
from __future__ import annotations

import ctypes as C
import functools
import os

import torch

from . import _lib
from ._lib import check, lib

# NVTX ranges around the hot path's stages (scope ncu / nsys
# captures to encode / prefill / decode step / migration), EMM_NVTX=1 at
# import time; otherwise the decorator returns the function unchanged.
NVTX = os.environ.get("EMM_NVTX", "") == "1"


def nvtx_stage(name: str):
    def deco(fn):
        if not NVTX:
            return fn

        @functools.wraps(fn)
        def wrapped(*a, **k):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*a, **k)
            finally:
                torch.cuda.nvtx.range_pop()
        return wrapped
    return deco

vp, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64

_lib.declare_more({
    "emm_launch_count": (C.c_uint64, []),
    "emm_device_sm_count": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "emm_gemm_bf16": (C.c_int, [vp, i64, vp, i64, vp, i64, i64, i64, i64, vp, vp, i64, C.c_int,
                                vp]),
    "emm_gemm_bf16_ex": (C.c_int, [vp, i64, vp, i64, vp, i64, i64, i64, i64, vp, vp]),
    "emm_row_sumsq_bf16": (C.c_int, [vp, i64, i64, i64, vp, vp]),
})

EPI_NONE, EPI_GELU_TANH, EPI_QUICK_GELU, EPI_GELU_ERF, EPI_GLU_SILU, EPI_QKV_ROPE = 0, 1, 2, 3, 4, 5


class GemmEpilogue(C.Structure):
    """emm_gemm_epilogue (include/emm.h)."""
    _fields_ = [("kind", C.c_int), ("bias", vp), ("residual", vp), ("ldr", i64),
                ("row_ss_in", vp), ("rms_eps", C.c_float), ("rms_dim", i64),
                ("row_ss_out", vp), ("q_out", vp), ("ld_q", i64), ("k_out", vp), ("v_out", vp),
                ("ld_kv", i64), ("kv_row", vp), ("pos", vp), ("rope_cs", vp), ("hq", C.c_int),
                ("hkv", C.c_int), ("hd", C.c_int), ("pos_h", vp), ("pos_w", vp),
                ("mrope_t", C.c_int), ("mrope_h", C.c_int), ("row_ss_zero", vp),
                ("rope2_cs", vp), ("rope2_cols", C.c_int), ("rope2_hd", C.c_int)]


def _stream(t: torch.Tensor | None = None):
    return torch.cuda.current_stream().cuda_stream


def h2d(a, device, dtype=None) -> torch.Tensor:
    """Asynchronous host->device copy of a small numpy array through pinned
    memory (torch's caching host allocator keeps the block alive until the
    copy has run).  A pageable copy would block the host until the stream
    drains, leaving the GPU idle while the next batch is prepared."""
    import numpy as np
    arr = np.ascontiguousarray(a, dtype=dtype)
    return torch.from_numpy(arr).pin_memory().to(device, non_blocking=True)


def _req_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("emm ops need CUDA tensors (no CPU fallback)")


def _ptr(t):
    return None if t is None else t.data_ptr()


def launch_count() -> int:
    return int(lib.emm_launch_count())


class KernelTimer:
    """Optional live timing of selected kernel classes with CUDA events on
    the launching stream (bench.py roofline).  Off by default."""

    def __init__(self):
        self.enabled = False
        self.records: dict[str, list] = {}
        self.trace = None  # optional [(kind, start ev, end ev, host s, host t0)]

    def start(self, trace: bool = False):
        self.enabled = True
        self.records = {}
        self.trace = [] if trace else None

    def stop(self):
        self.enabled = False

    def wrap(self, kind: str, work: float, fn, nbytes: float = 0.0):
        """work: algorithmic FLOPs (or bytes for copy kernels); nbytes:
        algorithmic DRAM bytes of compute kernels (their HBM roofline)."""
        if not self.enabled:
            return fn()
        import time
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        h0 = time.perf_counter()
        out = fn()
        h1 = time.perf_counter()
        e.record()
        self.records.setdefault(kind, []).append((s, e, work, nbytes))
        if self.trace is not None:
            self.trace.append((kind, s, e, h1 - h0, h0))
        return out

    def summary(self) -> dict:
        torch.cuda.synchronize()
        out = {}
        for kind, recs in self.records.items():
            ts = sorted(r[0].elapsed_time(r[1]) for r in recs)
            work = sum(r[2] for r in recs)
            nbytes = sum(r[3] for r in recs)
            out[kind] = {"launches": len(recs), "ms": sum(ts), "work": work, "bytes": nbytes,
                         "ms_min": ts[0], "ms_p50": ts[len(ts) // 2], "ms_max": ts[-1]}
        return out


TIMER = KernelTimer()


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None,
         bias: torch.Tensor | None = None, residual: torch.Tensor | None = None,
         epi: int = EPI_NONE) -> torch.Tensor:
    """out[M,N] = epi(a[M,K] @ b[N,K]^T + bias) (+ residual) on tcgen05.

    For EPI_GLU_SILU, b holds gate/up rows interleaved in blocks of 128
    (see interleave_glu) and out is [M, N/2]."""
    _req_cuda(a, b, bias, residual)
    assert a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    assert a.dim() == 2 and b.dim() == 2 and a.shape[1] == b.shape[1]
    assert a.stride(1) == 1 and b.stride(1) == 1
    M, K = a.shape
    N = b.shape[0]
    n_out = N // 2 if epi == EPI_GLU_SILU else N
    if out is None:
        out = torch.empty(M, n_out, device=a.device, dtype=torch.bfloat16)
    assert out.shape == (M, n_out) and out.stride(1) == 1
    if residual is not None:
        assert residual.shape == (M, n_out) and residual.stride(1) == 1
    TIMER.wrap("gemm", 2.0 * M * N * K, lambda: check(lib.emm_gemm_bf16(
        a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), out.data_ptr(), out.stride(0), M, N,
        K, _ptr(bias), _ptr(residual), residual.stride(0) if residual is not None else 0, epi,
        _stream())))
    return out


def gemm_ex(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None, *,
            epi: int = EPI_NONE, bias=None, residual=None, row_ss_in=None, rms_dim: int = 0,
            rms_eps: float = 1e-5, row_ss_out=None, qkv: dict | None = None,
            row_ss_zero=None, rope2: dict | None = None) -> torch.Tensor:
    """GEMM with the extended epilogue: folded RMSNorm row scale
    (row_ss_in), row sum-of-squares output (row_ss_out), zeroing of the next
    sum-of-squares buffer (row_ss_zero), and the fused QKV
    split + RoPE + KV-cache write (epi=EPI_QKV_ROPE, qkv=dict(q_out, k_out,
    v_out, kv_row, pos, rope_cs, hq, hkv, hd[, pos_h, pos_w, mrope=(t, h, w)])
    — with pos_h / pos_w the rotation is Qwen2-VL's multimodal RoPE)."""
    _req_cuda(a, b, bias, residual, row_ss_in, row_ss_out)
    M, K = a.shape
    N = b.shape[0]
    if epi == EPI_QKV_ROPE:
        out_ptr, ldc = None, 0
    else:
        n_out = N // 2 if epi == EPI_GLU_SILU else N
        if out is None:
            out = torch.empty(M, n_out, device=a.device, dtype=torch.bfloat16)
        out_ptr, ldc = out.data_ptr(), out.stride(0)
    e = GemmEpilogue()
    e.kind = epi
    e.bias = _ptr(bias)
    e.residual = _ptr(residual)
    e.ldr = residual.stride(0) if residual is not None else 0
    e.row_ss_in = _ptr(row_ss_in)
    e.rms_eps = rms_eps
    e.rms_dim = rms_dim
    e.row_ss_out = _ptr(row_ss_out)
    e.row_ss_zero = _ptr(row_ss_zero)
    if rope2 is not None:   # dict(cs, cols, hd, pos_h, pos_w): see include/emm.h
        _req_cuda(rope2["cs"], rope2["pos_h"], rope2["pos_w"])
        e.rope2_cs = rope2["cs"].data_ptr()
        e.rope2_cols, e.rope2_hd = int(rope2["cols"]), int(rope2["hd"])
        e.pos_h, e.pos_w = rope2["pos_h"].data_ptr(), rope2["pos_w"].data_ptr()
    if qkv is not None:
        e.q_out = qkv["q_out"].data_ptr()
        e.ld_q = qkv["q_out"].stride(0)
        e.k_out = qkv["k_out"].data_ptr()
        e.v_out = qkv["v_out"].data_ptr()
        e.ld_kv = qkv["k_out"].stride(0)
        e.kv_row = qkv["kv_row"].data_ptr()
        e.pos = _ptr(qkv.get("pos"))
        e.rope_cs = _ptr(qkv.get("rope_cs"))
        e.hq, e.hkv, e.hd = qkv["hq"], qkv["hkv"], qkv["hd"]
        if qkv.get("pos_h") is not None:
            _req_cuda(qkv["pos_h"], qkv["pos_w"])
            e.pos_h, e.pos_w = qkv["pos_h"].data_ptr(), qkv["pos_w"].data_ptr()
            e.mrope_t, e.mrope_h = int(qkv["mrope"][0]), int(qkv["mrope"][1])
    TIMER.wrap("gemm", 2.0 * M * N * K, lambda: check(lib.emm_gemm_bf16_ex(
        a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), out_ptr, ldc, M, N, K,
        C.byref(e), _stream())))
    return out


def row_sumsq(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """fp32 per-row sum of squares of a bf16 matrix (folded-RMSNorm input)."""
    _req_cuda(x)
    if out is None:
        out = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    check(lib.emm_row_sumsq_bf16(x.data_ptr(), x.stride(0), x.shape[0], x.shape[1],
                                 out.data_ptr(), _stream()))
    return out


def rope_table(max_pos: int, hd: int, theta: float, device="cuda") -> torch.Tensor:
    """(cos, sin) of pos * theta^(-2i/hd), computed in float64 -> fp32 pairs."""
    import numpy as np
    inv = theta ** (-np.arange(0, hd // 2, dtype=np.float64) * 2.0 / hd)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    cs = np.stack([np.cos(ang), np.sin(ang)], -1).astype(np.float32)
    return torch.from_numpy(cs).to(device)


def interleave_glu(w_gate: torch.Tensor, w_up: torch.Tensor, block: int = 128) -> torch.Tensor:
    """[I,K] gate and up -> [2I,K] with rows [g0..g127, u0..u127, g128..] so the
    GLU epilogue finds gate and up of the same feature in one 256-wide tile."""
    inter, k = w_gate.shape
    assert inter % block == 0, "intermediate size must be a multiple of 128"
    g = w_gate.reshape(inter // block, block, k)
    u = w_up.reshape(inter // block, block, k)
    return torch.stack([g, u], dim=1).reshape(2 * inter, k).contiguous()


def interleave_glu_bias(b_gate: torch.Tensor, b_up: torch.Tensor, block: int = 128):
    inter = b_gate.shape[0]
    return torch.stack([b_gate.reshape(-1, block), b_up.reshape(-1, block)], 1).reshape(2 * inter)


_lib.declare_more({
    "emm_attention_bf16": (C.c_int, [vp, i64, vp, vp, i64, vp, i64, i64, i64, C.c_int, C.c_int,
                                     C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, C.c_float,
                                     C.c_int, C.c_int, vp]),
})


DEFAULT_TILE_ROWS = 256
HEAD_MAJOR_DEFAULT = "tile"  # EMM_ATT_ORDER: tile | head (work-item order)


def pack_windows(seq_start, windows, rows: int = 128):
    """Greedy packing of consecutive whole windows of each sequence into
    groups of <= `rows` rows (AttnMeta.window_packed).  Returns the groups'
    absolute start rows and lengths and the per-row visible key range
    [lo, hi) relative to the row's group, indexed by absolute row."""
    import numpy as np
    wl = [np.asarray(w, np.int64) for w in windows]
    assert all((w <= rows).all() and (w > 0).all() for w in wl), "window longer than a tile"
    g_start, g_len, w_group, w_abs = [], [], [], []
    for s, w in enumerate(wl):
        cur, cur_len = int(seq_start[s]), 0
        pos = cur
        for x in w.tolist():
            if cur_len + x > rows:
                g_start.append(cur)
                g_len.append(cur_len)
                cur, cur_len = cur + cur_len, 0
            w_group.append(len(g_start))
            w_abs.append(pos)
            pos += x
            cur_len += x
        if cur_len:
            g_start.append(cur)
            g_len.append(cur_len)
    g_start = np.asarray(g_start, np.int64)
    g_len = np.asarray(g_len, np.int64)
    w_all = np.concatenate(wl) if wl else np.zeros(0, np.int64)
    w_abs = np.asarray(w_abs, np.int64)
    lo_w = w_abs - g_start[np.asarray(w_group, np.int64)]  # window start within its group
    rows_abs = np.repeat(w_abs, w_all) + (np.arange(int(w_all.sum())) -
                                          np.repeat(np.cumsum(w_all) - w_all, w_all))
    rb = np.zeros((int(rows_abs.max()) + 1 if len(rows_abs) else 0, 2), np.int64)
    rb[rows_abs, 0] = np.repeat(lo_w, w_all)
    rb[rows_abs, 1] = rb[rows_abs, 0] + np.repeat(w_all, w_all)
    return g_start, g_len, rb


class AttnMeta:
    """Varlen batch description shared by every layer of one forward pass.

    Sequence s has q_len[s] queries at rows q_start[s].. of the Q buffer and
    kv_len[s] keys at rows kv_start[s].. of the K/V buffers; with causal=True
    the queries are the LAST q_len positions of the KV sequence (uncached
    suffix after a cached prefix).  `windows` (optional, per sequence a list
    of segment lengths tiling it, q == kv): each row sees only its own
    segment (Qwen2.5-VL windowed vision attention).  Work items are
    `tile_rows` queries (256: a pair of 128-query tiles sharing every K/V
    block; 128: one tile with S double-buffered in TMEM) with the range of
    128-key blocks any of their rows can see; ordered longest-first."""

    def __init__(self, q_start, q_len, kv_start, kv_len, n_q_heads, causal, device="cuda",
                 windows=None, tile_rows: int | None = None):
        import os
        import numpy as np
        q_start, q_len = np.asarray(q_start, np.int64), np.asarray(q_len, np.int64)
        kv_start, kv_len = np.asarray(kv_start, np.int64), np.asarray(kv_len, np.int64)
        assert (q_len >= 0).all() and (kv_len >= 0).all()
        assert not causal or (kv_len >= q_len).all(), "causal queries are the last KV positions"
        bounds = None
        if windows is not None:
            bounds = np.zeros((int(q_len.sum()) if len(q_len) else 0, 2), np.int64)
            for s, segs in enumerate(windows):
                segs = np.asarray(segs, np.int64)
                assert q_len[s] == kv_len[s] == segs.sum(), "windows must tile the sequence"
                lo = np.repeat(np.concatenate([[0], np.cumsum(segs)[:-1]]), segs)
                r0 = int(q_start[s])
                bounds[r0:r0 + len(lo), 0] = lo
                bounds[r0:r0 + len(lo), 1] = lo + np.repeat(segs, segs)
        if tile_rows is None:
            tile_rows = int(os.environ.get("EMM_ATT_TILE_ROWS", DEFAULT_TILE_ROWS))
        assert tile_rows in (128, 256)
        self.tile_rows = tile_rows
        tpi = tile_rows // 128  # 128-query tiles per work item
        items, work = [], []
        for s in range(len(q_len)):
            ql, kl = int(q_len[s]), int(kv_len[s])
            nt = (ql + 127) // 128
            for t in range(0, nt, tpi):
                last_q = min(ql, (t + tpi) * 128) - 1
                if bounds is not None:
                    r0 = int(q_start[s])
                    b0 = int(bounds[r0 + t * 128, 0]) // 128
                    b1 = (int(bounds[r0 + last_q, 1]) + 127) // 128
                elif causal:
                    b0, b1 = 0, min((kl - ql + last_q) // 128 + 1, (kl + 127) // 128)
                else:
                    b0, b1 = 0, (kl + 127) // 128
                items.append((s, t, b0, b1))
                work.append(b1 - b0)
        order = np.argsort(-np.asarray(work, np.int64), kind="stable") if items else []
        if os.environ.get("EMM_ATT_ORDER", HEAD_MAJOR_DEFAULT) == "head":
            # longest first; among items of equal length, head-major, so the
            # CTAs in flight share one head's K/V in L2 (one ViT head's K/V
            # is 9.5 MB, all 16 heads' 152 MB exceed the 126 MB L2)
            wk = np.asarray(work, np.int64)
            tiles = []
            for w in (np.unique(wk)[::-1] if items else []):
                run = [i for i in order if wk[i] == w]
                tiles += [(items[i][0], h, items[i][1], items[i][2], items[i][3])
                          for h in range(n_q_heads) for i in run]
        else:
            tiles = [(items[i][0], h, items[i][1], items[i][2], items[i][3])
                     for i in order for h in range(n_q_heads)]
        arr = np.asarray(tiles, np.int32).reshape(-1, 5)
        self.n_tiles = arr.shape[0]
        self.work_blocks = int(np.sum(work)) * n_q_heads if work else 0
        i32t = lambda a: h2d(a, device, np.int32)
        self.tiles = i32t(arr.reshape(-1)) if self.n_tiles else torch.zeros(5, dtype=torch.int32,
                                                                              device=device)
        self.q_start, self.q_len = i32t(q_start), i32t(q_len)
        self.kv_start, self.kv_len = i32t(kv_start), i32t(kv_len)
        self.row_bounds = i32t(bounds.reshape(-1)) if bounds is not None else None
        self.causal = bool(causal)
        self.n_q_heads = n_q_heads
        self.q_len_host, self.kv_len_host = q_len, kv_len
        self.windows = windows

    @classmethod
    def window_packed(cls, seq_start, windows, n_q_heads, device="cuda", rows: int = 128):
        """Windowed (block-diagonal) attention with every window <= `rows`
        tokens: consecutive whole windows of one sequence are packed
        greedily into groups of <= `rows` rows, and each group becomes its
        own varlen sequence of ONE 128-query tile against ONE 128-key block
        (single-tile kernel, tile_rows=128; per-row bounds keep the windows
        apart inside a group).  Interior Qwen windows of 8x8 patches pack two
        per tile, so a 128x128 score tile is 50 % useful instead of the 25 %
        of a 256-row item spanning two key blocks, and a single key block
        per item never rescales O.  Same results as the `windows=` form."""
        import numpy as np
        g_start, g_len, rb = pack_windows(seq_start, windows, rows)
        wl = [np.asarray(w, np.int64) for w in windows]
        self = cls.__new__(cls)
        self.tile_rows = 128
        n_g = len(g_len)
        arr = np.zeros((n_g, n_q_heads, 5), np.int32)
        arr[:, :, 0] = np.arange(n_g, dtype=np.int32)[:, None]
        arr[:, :, 1] = np.arange(n_q_heads, dtype=np.int32)[None, :]
        arr[:, :, 4] = 1
        self.n_tiles = n_g * n_q_heads
        self.work_blocks = self.n_tiles
        i32t = lambda a: h2d(a, device, np.int32)
        self.tiles = (i32t(arr.reshape(-1)) if self.n_tiles
                      else torch.zeros(5, dtype=torch.int32, device=device))
        # the kernel reads row_bounds[q_start[seq] + row]: absolute rows
        self.q_start = self.kv_start = i32t(g_start)
        self.q_len = self.kv_len = i32t(g_len)
        self.row_bounds = i32t(rb.reshape(-1))
        self.causal = False
        self.n_q_heads = n_q_heads
        self.q_len_host = self.kv_len_host = g_len
        self.windows = wl
        return self

    def flops(self, head_dim: int) -> float:
        """Algorithmic FLOPs (QK^T + PV) of the valid (unmasked) entries."""
        import numpy as np
        tot = 0.0
        if self.windows is not None:
            tot = float(sum(float(np.sum(np.asarray(w, np.float64) ** 2)) for w in self.windows))
        else:
            for ql, kl in zip(self.q_len_host, self.kv_len_host):
                ql, kl = int(ql), int(kl)
                tot += ql * (kl - ql) + ql * (ql + 1) / 2 if self.causal else ql * kl
        return 4.0 * head_dim * self.n_q_heads * tot


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, meta: AttnMeta,
              n_kv_heads: int, head_dim: int, out: torch.Tensor | None = None,
              scale: float | None = None, label: str = "attention") -> torch.Tensor:
    """Varlen (GQA) flash attention on tcgen05.

    q: [Tq, n_q_heads*head_dim] (row pitch = q.stride(0)); k, v: [Tk, n_kv*hd]."""
    _req_cuda(q, k, v)
    assert q.dtype == k.dtype == v.dtype == torch.bfloat16
    assert k.stride(0) == v.stride(0) and q.stride(1) == 1 and k.stride(1) == 1
    if out is None:
        out = torch.empty(q.shape[0], meta.n_q_heads * head_dim, device=q.device,
                          dtype=torch.bfloat16)
    if scale is None:
        scale = head_dim ** -0.5
    # algorithmic bytes: q and out rows once, k / v rows once per query tile
    # group is the kernel's re-read pattern; count them once (lower bound)
    nb = 0.0
    if TIMER.enabled:
        nb = 2.0 * (q.shape[0] * q.shape[1] * 2 + k.shape[0] * k.shape[1] * 2)
    TIMER.wrap(label, meta.flops(head_dim) if TIMER.enabled else 0.0,
               lambda: check(lib.emm_attention_bf16(
                   q.data_ptr(), q.stride(0), k.data_ptr(), v.data_ptr(), k.stride(0),
                   out.data_ptr(), out.stride(0), q.shape[0], k.shape[0], meta.n_q_heads,
                   n_kv_heads, head_dim, meta.tiles.data_ptr(), meta.n_tiles,
                   meta.q_start.data_ptr(), meta.q_len.data_ptr(), meta.kv_start.data_ptr(),
                   meta.kv_len.data_ptr(), _ptr(meta.row_bounds), float(scale),
                   int(meta.causal), meta.tile_rows, _stream())), nbytes=nb)
    return out


_lib.declare_more({
    "emm_decode_attention_workspace": (i64, [i64, C.c_int, C.c_int, C.c_int, i64]),
    "emm_decode_attention_bf16": (C.c_int, [vp, i64, vp, vp, i64, vp, vp, vp, i64, C.c_int,
                                            C.c_int, C.c_int, i64, vp, i64, vp, i64, C.c_float,
                                            vp]),
})


_lib.declare_more({"emm_embed_rows": (C.c_int, [vp, i64, vp, vp, i64, i64, i64, vp])})


def embed_rows(table: torch.Tensor, ids: torch.Tensor, out: torch.Tensor | None = None):
    """out[i] = table[ids[i]] (int32 ids on the device)."""
    _req_cuda(table, ids)
    assert ids.dtype == torch.int32 and table.stride(1) == 1
    if out is None:
        out = torch.empty(ids.shape[0], table.shape[1], device=table.device, dtype=table.dtype)
    es = table.element_size()
    check(lib.emm_embed_rows(table.data_ptr(), table.stride(0) * es, ids.data_ptr(),
                             out.data_ptr(), out.stride(0) * es, ids.shape[0],
                             table.shape[1] * es, _stream()))
    return out


_lib.declare_more({"emm_decode_advance": (C.c_int, [vp, vp, vp, vp, vp, vp, i64, vp])})


def decode_advance(bt, bt_off, kv_len, next_pos, slot, pos):
    """Device-side decode step advance (see include/emm.h)."""
    _req_cuda(bt, bt_off, kv_len, next_pos, slot, pos)
    check(lib.emm_decode_advance(bt.data_ptr(), bt_off.data_ptr(), kv_len.data_ptr(),
                                 next_pos.data_ptr(), slot.data_ptr(), pos.data_ptr(),
                                 kv_len.shape[0], _stream()))


def decode_attention(q: torch.Tensor, k_plane: torch.Tensor, v_plane: torch.Tensor,
                     bt: torch.Tensor, bt_off: torch.Tensor, kv_len: torch.Tensor,
                     n_kv_heads: int, head_dim: int, max_kv_len: int,
                     out: torch.Tensor | None = None, scale: float | None = None,
                     label: str = "attention_decode") -> torch.Tensor:
    """Paged GQA decode attention (one query token per request).

    q: [n_req, hq*hd]; k_plane / v_plane: [slots, hkv*hd] (one layer of the
    arena); bt int32 slots, bt_off int64 [n_req + 1], kv_len int32 [n_req]."""
    _req_cuda(q, k_plane, v_plane, bt, bt_off, kv_len)
    assert q.dtype == k_plane.dtype == v_plane.dtype == torch.bfloat16
    assert bt.dtype == torch.int32 and bt_off.dtype == torch.int64 and kv_len.dtype == torch.int32
    assert k_plane.stride(0) == v_plane.stride(0) and q.stride(1) == 1
    n = q.shape[0]
    hq = q.shape[1] // head_dim
    if out is None:
        out = torch.empty(n, hq * head_dim, device=q.device, dtype=torch.bfloat16)
    if scale is None:
        scale = head_dim ** -0.5
    wsb = int(lib.emm_decode_attention_workspace(n, hq, n_kv_heads, head_dim, max_kv_len))
    ws = torch.empty(max(wsb // 4, 1), device=q.device, dtype=torch.float32)
    work = 4.0 * head_dim * hq * float(max_kv_len) * n if TIMER.enabled else 0.0
    TIMER.wrap(label, work, lambda: check(lib.emm_decode_attention_bf16(
        q.data_ptr(), q.stride(0), k_plane.data_ptr(), v_plane.data_ptr(), k_plane.stride(0),
        bt.data_ptr(), bt_off.data_ptr(), kv_len.data_ptr(), n, hq, n_kv_heads, head_dim,
        int(max_kv_len), out.data_ptr(), out.stride(0), ws.data_ptr(), wsb, float(scale),
        _stream())))
    return out


_lib.declare_more({
    "emm_norm_bf16": (C.c_int, [vp, i64, vp, vp, vp, vp, i64, i64, i64, C.c_float, C.c_int,
                                vp]),
    "emm_rope_split_bf16": (C.c_int, [vp, i64, i64, C.c_int, C.c_int, C.c_int, vp, C.c_float,
                                      C.c_int, vp, i64, vp, vp, vp, i64, vp]),
    "emm_gather_rows": (C.c_int, [vp, vp, i64, i64, i64, vp]),
    "emm_patchify": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.POINTER(C.c_float), C.POINTER(C.c_float), vp, vp]),
    "emm_vit_embed": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, i64, C.c_int, C.c_int, vp]),
    "emm_argmax_rows": (C.c_int, [vp, i64, i64, i64, vp, vp]),
    "emm_argmax_workspace_keys": (i64, [i64, i64]),
    "emm_argmax_rows_ws": (C.c_int, [vp, i64, i64, i64, vp, vp, vp]),
})


def norm(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor | None = None, eps: float = 1e-5,
         out: torch.Tensor | None = None, rows: torch.Tensor | None = None) -> torch.Tensor:
    """RMSNorm (b is None) or LayerNorm over the last dim; optional row gather."""
    _req_cuda(x, w, b)
    T = x.shape[0] if rows is None else rows.shape[0]
    D = x.shape[1]
    if out is None:
        out = torch.empty(T, D, device=x.device, dtype=torch.bfloat16)
    check(lib.emm_norm_bf16(x.data_ptr(), x.stride(0), _ptr(rows), w.data_ptr(), _ptr(b),
                            out.data_ptr(), out.stride(0), T, D, float(eps), int(b is not None),
                            _stream()))
    return out


def rope_split(qkv: torch.Tensor, hq: int, hkv: int, hd: int, q_out: torch.Tensor,
               k_out: torch.Tensor, v_out: torch.Tensor, kv_row: torch.Tensor,
               pos: torch.Tensor | None = None, theta: float = 10000.0):
    """Split fused QKV rows; RoPE (rotate-half) on q and k when pos is given;
    q -> q_out[t], k/v -> k_out/v_out[kv_row[t]]."""
    _req_cuda(qkv, q_out, k_out, v_out, kv_row, pos)
    assert k_out.stride(0) == v_out.stride(0)
    check(lib.emm_rope_split_bf16(qkv.data_ptr(), qkv.stride(0), qkv.shape[0], hq, hkv, hd,
                                  _ptr(pos), float(theta), int(pos is not None),
                                  q_out.data_ptr(), q_out.stride(0), k_out.data_ptr(),
                                  v_out.data_ptr(), kv_row.data_ptr(), k_out.stride(0),
                                  _stream()))


def gather_rows(src_ptrs: torch.Tensor, out: torch.Tensor):
    """out[i, :] = bytes at src_ptrs[i] (int64 device addresses)."""
    _req_cuda(src_ptrs, out)
    check(lib.emm_gather_rows(src_ptrs.data_ptr(), out.data_ptr(),
                              out.stride(0) * out.element_size(), out.shape[0],
                              out.shape[1] * out.element_size(), _stream()))


def patchify(pix: torch.Tensor, pix_off: torch.Tensor, gh: torch.Tensor, gw: torch.Tensor,
             patch_off: torch.Tensor, max_patches: int, patch: int, k_pad: int, mean, std,
             out: torch.Tensor):
    _req_cuda(pix, pix_off, gh, gw, patch_off, out)
    m = (C.c_float * 3)(*mean)
    s = (C.c_float * 3)(*std)
    check(lib.emm_patchify(pix.data_ptr(), pix_off.data_ptr(), gh.data_ptr(), gw.data_ptr(),
                           patch_off.data_ptr(), gh.shape[0], max_patches, patch, k_pad, m, s,
                           out.data_ptr(), _stream()))


def vit_embed(patch_out: torch.Tensor, cls: torch.Tensor | None, pos: torch.Tensor,
              tok_off: torch.Tensor, patch_off: torch.Tensor, out: torch.Tensor):
    """ViT token rows: [CLS] + patch embeddings of each image, plus learned
    absolute position embeddings (tok_off/patch_off: int64 device CSR)."""
    _req_cuda(patch_out, cls, pos, out, tok_off, patch_off)
    check(lib.emm_vit_embed(patch_out.data_ptr(), _ptr(cls), pos.data_ptr(), out.data_ptr(),
                            tok_off.data_ptr(), patch_off.data_ptr(), patch_off.shape[0],
                            out.shape[0], int(cls is not None), patch_out.shape[1], _stream()))


_lib.declare_more({
    "emm_patchify_rows": (C.c_int, [vp, vp, vp, vp, vp, i64, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_float), C.POINTER(C.c_float), vp, vp]),
    "emm_rope2d_bf16": (C.c_int, [vp, i64, i64, C.c_int, C.c_int, vp, vp, C.c_float, vp]),
})


def patchify_rows(pix: torch.Tensor, pix_off: torch.Tensor, gw: torch.Tensor,
                  row_img: torch.Tensor, row_patch: torch.Tensor, patch: int, temporal: int,
                  k_pad: int, mean, std, out: torch.Tensor):
    """Qwen2.5-VL patch rows in the caller's (window) order: out[r] = patch
    row_patch[r] of image row_img[r], columns (c, t, ky, kx)."""
    _req_cuda(pix, pix_off, gw, row_img, row_patch, out)
    m = (C.c_float * 3)(*mean)
    s = (C.c_float * 3)(*std)
    check(lib.emm_patchify_rows(pix.data_ptr(), pix_off.data_ptr(), gw.data_ptr(),
                                row_img.data_ptr(), row_patch.data_ptr(), out.shape[0], patch,
                                temporal, k_pad, m, s, out.data_ptr(), _stream()))


def rope2d_(x: torch.Tensor, n_heads: int, hd: int, pos_h: torch.Tensor, pos_w: torch.Tensor,
            theta: float = 10000.0):
    """In-place 2-D RoPE of the first n_heads heads of every row of x."""
    _req_cuda(x, pos_h, pos_w)
    assert x.stride(1) == 1
    check(lib.emm_rope2d_bf16(x.data_ptr(), x.stride(0), x.shape[0], n_heads, hd,
                              pos_h.data_ptr(), pos_w.data_ptr(), float(theta), _stream()))


ARGMAX_CHUNK = 8192  # emm.h EMM_ARGMAX_CHUNK


def argmax_rows(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    _req_cuda(x)
    if out is None:
        out = torch.empty(x.shape[0], dtype=torch.int32, device=x.device)
    T, V = x.shape[0], x.shape[1]
    if V > ARGMAX_CHUNK and T <= 65535:
        # vocabulary split over CTAs; scratch from the caching allocator
        # (graph-capture safe)
        ws = torch.empty(int(lib.emm_argmax_workspace_keys(T, V)), dtype=torch.int64,
                         device=x.device)
        check(lib.emm_argmax_rows_ws(x.data_ptr(), x.stride(0), T, V, out.data_ptr(),
                                     ws.data_ptr(), _stream()))
    else:
        check(lib.emm_argmax_rows(x.data_ptr(), x.stride(0), T, V, out.data_ptr(), _stream()))
    return out
