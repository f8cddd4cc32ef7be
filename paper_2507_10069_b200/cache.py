"""Drop-in replacements for mmsim.cache (pkg/src/mmsim/cache.py:1-406).

`GpuUnifiedCache` is duck-type compatible with `mmsim.cache.UnifiedCache`
(same constructor, same six methods, same `stats` / `images` / `prefixes`
attributes) and is what `paper_2507_10069_b200.engine.install()` binds into
the unchanged reference scheduler.  `ImagePool` and `PrefixTree` mirror the
reference classes for the ported unit tests.

Every decision is made by the C++ control plane in libemm.so
(csrc/host_cache.cpp, a bit-exact restatement); this module only converts
symbols to injective uint64 keys (keys.py) and marshals arguments.  The
device data plane (block hashes, GPU hash-table match, block tables, paged
KV pool) is attached with `attach_device(...)` (dataplane.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Hashable, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib
from .keys import KeyCodec, _seqcodec

if _seqcodec is None:
    raise ImportError("paper_2507_10069_b200._seqcodec is not built (build.py)")


def _fp(fn) -> int:
    return C.cast(fn, C.c_void_p).value


# the CPython binding calls the same C-ABI entry points ctypes resolved
_seqcodec.bind(_fp(lib.emm_cache_match_prefix), _fp(lib.emm_cache_match_prefix_lazy),
               _fp(lib.emm_cache_insert_prefix),
               _fp(lib.emm_cache_release), _fp(lib.emm_cache_image_lookup),
               _fp(lib.emm_cache_image_insert))

try:  # reuse the reference's exception types when the reference is importable
    from mmsim.cache import ReleaseWithoutMatch as _RefRelease  # type: ignore
    from mmsim.core import MmsimError as _RefBase  # type: ignore
except Exception:  # pragma: no cover - the GPU box has no reference
    _RefBase = Exception
    _RefRelease = None

if _RefRelease is not None:
    class ReleaseWithoutMatch(_RefRelease):  # type: ignore[misc,valid-type]
        """A handle was released twice or never issued by this tree (cache.py:18-19)."""
else:
    class ReleaseWithoutMatch(_RefBase):  # type: ignore[no-redef]
        """A handle was released twice or never issued by this tree (cache.py:18-19)."""

DEFAULT_CODEC = KeyCodec()

_u64p = C.POINTER(C.c_uint64)


def _check(code: int) -> None:
    if code == _lib.EMM_E_RELEASE_WITHOUT_MATCH:
        raise ReleaseWithoutMatch(lib.emm_last_error().decode())
    check(code)


def _as_arrays(codec: KeyCodec, tokens, weights):
    pre = getattr(tokens, "emm_keys", None)
    prew = getattr(weights, "emm_array", None)
    if pre is not None and (prew is not None or weights is None):
        keys = pre
        w = prew if prew is not None else np.ones(keys.shape[0], dtype=np.int64)
        if w.shape[0] != keys.shape[0]:  # zip() semantics of the reference loops
            n = min(w.shape[0], keys.shape[0])
            keys, w = keys[:n], w[:n]
        return keys, w
    return codec.keys_weights(tokens, weights)


# ------------------------------------------------------------------ image pool

class ImagePool:
    """LRU pool of encoded image tokens keyed by content hash (cache.py:31-74)."""

    def __init__(self, capacity_tokens: int = 0, _handle=None, _owner=None):
        if _handle is None:
            h = C.c_void_p()
            check(lib.emm_pool_create(int(capacity_tokens), C.byref(h)))
            self._h = h
            self._own = True
        else:
            self._h = _handle
            self._own = False
        self._owner = _owner

    def __del__(self):
        if getattr(self, "_own", False) and self._h:
            lib.emm_pool_destroy(self._h)
            self._h = None

    def _info(self):
        out = (C.c_int64 * 4)()
        check(lib.emm_pool_info(self._h, out))
        return out

    @property
    def capacity(self) -> int:
        return self._info()[2]

    @property
    def total_tokens(self) -> int:
        return self._info()[0]

    @property
    def evictions(self) -> int:
        return self._info()[1]

    def __len__(self) -> int:
        return self._info()[3]

    def lookup(self, content_hash: str, now: float) -> int | None:
        out = C.c_int64()
        check(lib.emm_pool_lookup(self._h, content_hash.encode(), float(now), C.byref(out)))
        return None if out.value < 0 else out.value

    def insert(self, content_hash: str, token_count: int, now: float,
               bytes_estimate: int = 0) -> bool:
        ok = C.c_int32()
        check(lib.emm_pool_insert(self._h, content_hash.encode(), int(token_count), float(now),
                                  int(bytes_estimate), C.byref(ok)))
        return bool(ok.value)

    def take_evicted(self) -> list[str]:
        need = C.c_int64()
        check(lib.emm_pool_take_evicted(self._h, None, 0, C.byref(need)))
        if need.value == 0:
            return []
        buf = C.create_string_buffer(need.value)
        check(lib.emm_pool_take_evicted(self._h, buf, need.value, C.byref(need)))
        return buf.raw[: need.value].decode().split("\n")[:-1]


# ----------------------------------------------------------------- prefix tree

class MatchHandle(_seqcodec.Handle):
    """Pin on the matched path; release exactly once (cache.py:93-103).
    Fields `_id`, `_tree`, `released` live in the C base type, so the cache
    core creates handles without running Python code."""

    __slots__ = ()

    @property
    def entries(self) -> list:
        n = C.c_int64()
        check(lib.emm_tree_handle_entries(self._tree._h, self._id, C.byref(n)))
        return [None] * max(0, n.value)


@dataclass
class NodeView:
    """Read-only snapshot of a tree node (cache.py:79-90)."""
    node_id: int
    span: tuple
    weights: tuple
    user_count: int
    last_used: float
    children: dict = field(default_factory=dict)

    @property
    def kv_tokens(self) -> int:
        return sum(self.weights)


class PrefixTree:
    """Span-compressed radix tree over weighted symbols (cache.py:105-336)."""

    def __init__(self, capacity_tokens: int = 0, _handle=None, _owner=None,
                 codec: KeyCodec | None = None):
        if _handle is None:
            h = C.c_void_p()
            check(lib.emm_tree_create(int(capacity_tokens), C.byref(h)))
            self._h = h
            self._own = True
        else:
            self._h = _handle
            self._own = False
        self._owner = _owner
        self.codec = codec or DEFAULT_CODEC

    def __del__(self):
        if getattr(self, "_own", False) and self._h:
            lib.emm_tree_destroy(self._h)
            self._h = None

    def _info(self):
        out = (C.c_int64 * 8)()
        check(lib.emm_tree_info(self._h, out))
        return out

    capacity = property(lambda self: self._info()[0])
    total_tokens = property(lambda self: self._info()[1])
    evictions = property(lambda self: self._info()[2])
    increments = property(lambda self: self._info()[3])
    decrements = property(lambda self: self._info()[4])
    live_handle_count = property(lambda self: self._info()[5])

    def match_prefix(self, tokens: Sequence[Hashable], weights: Sequence[int] | None = None,
                     now: float = 0.0):
        keys, w = _as_arrays(self.codec, tokens, weights)
        matched = C.c_int64()
        hid = C.c_uint64()
        check(lib.emm_tree_match(self._h, keys.ctypes.data, w.ctypes.data, keys.shape[0],
                                 float(now), C.byref(matched), C.byref(hid)))
        return matched.value, MatchHandle(hid.value, self)

    def release(self, handle: MatchHandle) -> None:
        if not isinstance(handle, MatchHandle) or handle._tree is not self or handle.released:
            raise ReleaseWithoutMatch("handle already released or unknown")
        _check(lib.emm_tree_release(self._h, handle._id))
        handle.released = True

    def insert_prefix(self, tokens, weights=None, now: float = 0.0) -> int:
        keys, w = _as_arrays(self.codec, tokens, weights)
        added = C.c_int64()
        check(lib.emm_tree_insert(self._h, keys.ctypes.data, w.ctypes.data, keys.shape[0],
                                  float(now), C.byref(added)))
        return added.value

    def evict(self, needed_tokens: int, now: float = 0.0) -> int:
        freed = C.c_int64()
        check(lib.emm_tree_evict(self._h, int(needed_tokens), float(now), C.byref(freed)))
        return freed.value

    @property
    def eviction_log(self) -> list[tuple[int, int, float]]:
        n = self._info()[6]
        if n == 0:
            return []
        ids = np.empty(n, dtype=np.int64)
        kvs = np.empty(n, dtype=np.int64)
        lu = np.empty(n, dtype=np.float64)
        check(lib.emm_tree_eviction_log(self._h, 0, n, ids.ctypes.data, kvs.ctypes.data,
                                        lu.ctypes.data))
        return [(int(a), int(b), float(c)) for a, b, c in zip(ids, kvs, lu)]

    def _snapshot(self):
        nn, ns = C.c_int64(), C.c_int64()
        check(lib.emm_tree_nodes(self._h, 0, 0, C.byref(nn), C.byref(ns), None, None, None,
                                 None, None, None, None, None))
        n, s = nn.value, ns.value
        ids = np.empty(n, np.int64)
        par = np.empty(n, np.int64)
        kvs = np.empty(n, np.int64)
        ucs = np.empty(n, np.int64)
        lu = np.empty(n, np.float64)
        off = np.empty(n + 1, np.int64)
        sk = np.empty(max(s, 1), np.uint64)
        sw = np.empty(max(s, 1), np.int64)
        check(lib.emm_tree_nodes(self._h, n, s, C.byref(nn), C.byref(ns), ids.ctypes.data,
                                 par.ctypes.data, kvs.ctypes.data, ucs.ctypes.data,
                                 lu.ctypes.data, off.ctypes.data, sk.ctypes.data,
                                 sw.ctypes.data))
        root = NodeView(0, (), (), 0, 0.0)
        by_id = {0: root}
        views = []
        for i in range(n):
            span = tuple(self.codec.symbol(k) for k in sk[off[i]:off[i + 1]])
            v = NodeView(int(ids[i]), span, tuple(int(x) for x in sw[off[i]:off[i + 1]]),
                         int(ucs[i]), float(lu[i]))
            by_id[v.node_id] = v
            views.append((v, int(par[i])))
        for v, p in views:
            by_id[p].children[v.span[0]] = v
        return root, [v for v, _ in views]

    @property
    def root(self) -> NodeView:
        return self._snapshot()[0]

    def iter_nodes(self):
        return iter(self._snapshot()[1])

    def cached_sequences(self) -> list[tuple[tuple, int]]:
        """All root-to-node sequences with their cumulative KV length (cache.py:312-324)."""
        root, _ = self._snapshot()
        out = []

        def walk(node, prefix, kv):
            for child in node.children.values():
                seq = prefix + child.span
                total = kv + child.kv_tokens
                out.append((seq, total))
                walk(child, seq, total)
        walk(root, (), 0)
        return out


# ------------------------------------------------------------- unified cache

@dataclass
class CacheStats:
    """Counters of cache.py:341-360, read from the C++ façade."""
    image_hits: int = 0
    image_misses: int = 0
    image_tokens_saved: int = 0
    prefix_lookups: int = 0
    prefix_hits: int = 0
    prefix_tokens_saved: int = 0
    evictions: int = 0

    def as_dict(self) -> dict:
        return dict(self.__dict__)


class GpuUnifiedCache(_seqcodec.Core):
    """Image pool plus prefix tree behind one budget split (cache.py:363-406).

    Constructor and methods match mmsim.cache.UnifiedCache exactly; the
    device data plane is attached separately (attach_device) so the same
    object drops into the reference scheduler unchanged.  match_prefix,
    insert_prefix, release and image_lookup are C methods of the base type
    (csrc/py/seqcodec.c); the rest is Python.
    """

    def __init__(self, budget_tokens: int, image_fraction: float = 0.2,
                 codec: KeyCodec | None = None):
        h = C.c_void_p()
        check(lib.emm_cache_create(int(budget_tokens), float(image_fraction), C.byref(h)))
        self._h = h
        self._hv = h.value  # plain int for the CPython binding
        self.codec = codec or DEFAULT_CODEC
        ph, th = C.c_void_p(), C.c_void_p()
        check(lib.emm_cache_parts(h, C.byref(ph), C.byref(th)))
        self.images = ImagePool(_handle=ph, _owner=self)
        self.prefixes = PrefixTree(_handle=th, _owner=self, codec=self.codec)
        self.device = None  # DeviceIndex when the data plane is attached
        self.listeners: list = []
        self._core_bind(self._hv, self.codec._img_key, self.prefixes, MatchHandle,
                        ReleaseWithoutMatch)

    def __del__(self):
        if getattr(self, "_h", None):
            self._core_unbind()
            self.device = None
            lib.emm_cache_destroy(self._h)
            self._h = None

    def _raise(self, rc: int) -> None:
        _check(rc)

    @property
    def stats(self) -> CacheStats:
        s = self._stats_raw()
        return CacheStats(*[int(x) for x in s[:6]], evictions=0)

    def _stats_raw(self):
        out = (C.c_int64 * 9)()
        check(lib.emm_cache_stats(self._h, out))
        return out

    def image_insert(self, content_hash: str, token_count: int, now: float,
                     bytes_estimate: int = 0) -> bool:
        rc, ok = _seqcodec.image_insert(self._hv, content_hash, token_count, now,
                                        bytes_estimate)
        if rc:
            check(rc)
        if self.listeners:
            evicted = self.images.take_evicted()
            for fn in self.listeners:
                fn("image_insert", content_hash, bool(ok), evicted)
        return bool(ok)

    # match_prefix / insert_prefix / release / image_lookup: C methods of
    # _seqcodec.Core; these take the sequences the C walk leaves to the codec
    def _match_slow(self, tokens: Sequence[Hashable], weights: Sequence[int], now: float):
        keys, w = _as_arrays(self.codec, tokens, weights)
        matched = C.c_int64()
        hid = C.c_uint64()
        check(lib.emm_cache_match_prefix(self._h, keys.ctypes.data, w.ctypes.data,
                                         keys.shape[0], float(now), C.byref(matched),
                                         C.byref(hid)))
        return matched.value, MatchHandle(hid.value, self.prefixes)

    def _insert_slow(self, tokens: Sequence[Hashable], weights: Sequence[int],
                     now: float) -> int:
        keys, w = _as_arrays(self.codec, tokens, weights)
        added = C.c_int64()
        check(lib.emm_cache_insert_prefix(self._h, keys.ctypes.data, w.ctypes.data,
                                          keys.shape[0], float(now), C.byref(added)))
        return added.value

    def snapshot_stats(self) -> dict:
        s = self._stats_raw()
        return {
            "image_hits": int(s[0]), "image_misses": int(s[1]),
            "image_tokens_saved": int(s[2]), "prefix_lookups": int(s[3]),
            "prefix_hits": int(s[4]), "prefix_tokens_saved": int(s[5]),
            "evictions": int(s[6]), "image_pool_tokens": int(s[7]),
            "prefix_pool_tokens": int(s[8]),
        }


# name-compatible alias for code written against mmsim.cache
UnifiedCache = GpuUnifiedCache
