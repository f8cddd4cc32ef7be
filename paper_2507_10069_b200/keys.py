"""Injective 64-bit keys for unified-sequence symbols.

The reference's prefix tree is keyed by arbitrary hashables; the engine emits
("img", content_hash), ("pfx", prefix_id, i) and ("txt", request_id, i)
(pkg/src/mmsim/engine.py:448-461).  Request-unique text symbols must never
match across requests, so keys are *encodings*, not hashes of token ids:

  bits 63..62  tag   0 = generic (interned), 1 = pfx, 2 = txt, 3 = img
  pfx / txt    (id << 32) | i          id < 2^30, i < 2^32
  img          62 bits of the 128-bit content hash (collision-checked)
  generic      interned ordinal (Python equality semantics preserved)

The KeyCodec owns the reverse maps so introspection (cached_sequences,
iter_nodes) can return the original symbols.
"""
from __future__ import annotations

import hashlib

import numpy as np

try:
    from . import _seqcodec  # built next to libemm.so (build.py)
except ImportError:  # pragma: no cover
    _seqcodec = None

TAG_GENERIC, TAG_PFX, TAG_TXT, TAG_IMG = 0, 1, 2, 3
_MASK62 = (1 << 62) - 1
_TAG_PFX = TAG_PFX << 62
_TAG_TXT = TAG_TXT << 62
_TAG_IMG = TAG_IMG << 62


class KeyCollision(RuntimeError):
    pass


class KeyCodec:
    def __init__(self):
        self._img_key: dict[str, int] = {}
        self._img_of: dict[int, str] = {}
        self._gen_key: dict = {}
        self._gen_of: list = []

    # -- images ----------------------------------------------------------
    def image_key(self, content_hash: str) -> int:
        k = self._img_key.get(content_hash)
        if k is not None:
            return k
        try:
            v = int(content_hash[:16], 16) if len(content_hash) >= 16 else None
        except ValueError:
            v = None
        if v is None:
            v = int.from_bytes(hashlib.md5(content_hash.encode()).digest()[:8], "big")
        k = _TAG_IMG | (v & _MASK62)
        other = self._img_of.get(k)
        if other is not None and other != content_hash:
            raise KeyCollision(f"image keys collide: {other!r} vs {content_hash!r}")
        self._img_key[content_hash] = k
        self._img_of[k] = content_hash
        return k

    # -- generic symbols --------------------------------------------------
    def _generic(self, sym) -> int:
        k = self._gen_key.get(sym)
        if k is None:
            k = len(self._gen_of)
            if k > _MASK62:
                raise KeyCollision("generic key space exhausted")
            self._gen_key[sym] = k
            self._gen_of.append(sym)
        return k

    def key(self, sym) -> int:
        if type(sym) is tuple and len(sym) >= 2:
            tag = sym[0]
            if tag == "img" and len(sym) == 2 and isinstance(sym[1], str):
                return self.image_key(sym[1])
            if (len(sym) == 3 and (tag == "txt" or tag == "pfx")
                    and type(sym[1]) is int and type(sym[2]) is int
                    and 0 <= sym[1] < (1 << 30) and 0 <= sym[2] < (1 << 32)):
                return (_TAG_TXT if tag == "txt" else _TAG_PFX) | (sym[1] << 32) | sym[2]
        return self._generic(sym)

    def keys(self, tokens) -> np.ndarray:
        """Encode a token sequence; fast path for engine-built sequences."""
        pre = getattr(tokens, "emm_keys", None)
        if pre is not None:
            return pre
        return self.keys_weights(tokens, None)[0]

    def keys_weights(self, tokens, weights) -> tuple[np.ndarray, np.ndarray]:
        """Keys and int64 weights of (tokens, weights), zip()-truncated like
        the reference loops (cache.py:121-156).  Engine-built lists
        (engine.py:448-461) are walked in C (_seqcodec); symbols it cannot
        encode (generic hashables, first sight of an image, non-int weights)
        go through `key` one at a time and the walk resumes after them."""
        n = len(tokens) if weights is None else min(len(tokens), len(weights))
        keys = np.empty(n, dtype=np.uint64)
        w = np.empty(n, dtype=np.int64)
        if _seqcodec is None:  # pragma: no cover - built with libemm.so
            raise ImportError("paper_2507_10069_b200._seqcodec is not built")
        start = 0
        img = self._img_key
        while True:
            r = _seqcodec.encode(tokens, weights, img, keys, w, start)
            if r >= 0:
                return keys, w
            i = -r - 1
            keys[i] = self.key(tokens[i])
            w[i] = 1 if weights is None else np.asarray(weights[i], dtype=np.int64)
            start = i + 1

    def symbol(self, key: int):
        key = int(key)
        tag = key >> 62
        if tag == TAG_IMG:
            return ("img", self._img_of[key])
        if tag == TAG_TXT or tag == TAG_PFX:
            return ("txt" if tag == TAG_TXT else "pfx", (key >> 32) & ((1 << 30) - 1),
                    key & 0xFFFFFFFF)
        return self._gen_of[key]


def request_keys(codec: KeyCodec, req) -> tuple[np.ndarray, np.ndarray]:
    """Vectorised keys/weights of Engine.unified_sequence(req)
    (pkg/src/mmsim/engine.py:448-461) for a reference `Request`.  Ids outside
    the packed range (KeyCodec.key: id < 2^30, position < 2^32) go through
    the per-symbol codec, so the result always equals codec.keys() of the
    reference's symbols."""
    n_img = len(req.images)
    prefix_len = req.prefix_len if req.prefix_id is not None else 0
    n_txt = req.text_input_len - prefix_len
    if not (_packable(req.prefix_id, prefix_len) and _packable(req.id, n_txt)):
        syms = [("img", img.content_hash) for img in req.images]
        syms += [("pfx", req.prefix_id, i) for i in range(prefix_len)]
        syms += [("txt", req.id, i) for i in range(max(0, n_txt))]
        wts = [img.token_count for img in req.images] + [1] * (len(syms) - n_img)
        return codec.keys_weights(syms, wts)
    keys = np.empty(n_img + prefix_len + max(0, n_txt), dtype=np.uint64)
    weights = np.ones(keys.shape[0], dtype=np.int64)
    for i, img in enumerate(req.images):
        keys[i] = codec.image_key(img.content_hash)
        weights[i] = img.token_count
    if prefix_len:
        keys[n_img:n_img + prefix_len] = (np.uint64(_TAG_PFX | (req.prefix_id << 32))
                                          + np.arange(prefix_len, dtype=np.uint64))
    if n_txt > 0:
        keys[n_img + prefix_len:] = (np.uint64(_TAG_TXT | (req.id << 32))
                                     + np.arange(n_txt, dtype=np.uint64))
    return keys, weights


def _packable(ident, count) -> bool:
    if count <= 0:
        return True
    return type(ident) is int and 0 <= ident < (1 << 30) and count <= (1 << 32)


class WeightSeq(list):
    """Weights list carrying its int64 array."""

    __slots__ = ("emm_array",)


class SymbolSeq(list):
    """A unified sequence (the reference's list of symbols, engine.py:448-461)
    carrying its precomputed keys / weights so the cache boundary skips the
    per-symbol encoding.  It IS the reference's list, so it is
    interchangeable with what Engine.unified_sequence returns."""

    __slots__ = ("emm_keys", "weights")

    def __init__(self, keys: np.ndarray, weights: np.ndarray, symbols):
        super().__init__(symbols)
        self.emm_keys = np.ascontiguousarray(keys, dtype=np.uint64)
        if len(self) != self.emm_keys.shape[0]:
            raise ValueError("symbols and keys differ in length")
        ws = WeightSeq(weights.tolist())
        ws.emm_array = np.ascontiguousarray(weights, dtype=np.int64)
        self.weights = ws


class KeySeq:
    """Keys-only sequence for the repo's own driver (no symbol list is ever
    built on the hot path).  Iterating or indexing decodes the symbols through
    the codec on demand, so handing one to reference code sees the same
    symbols as Engine.unified_sequence would produce."""

    __slots__ = ("emm_keys", "weights", "_codec")

    def __init__(self, keys: np.ndarray, weights: np.ndarray, codec: KeyCodec):
        self.emm_keys = np.ascontiguousarray(keys, dtype=np.uint64)
        self._codec = codec
        self.weights = _KeyWeights(np.ascontiguousarray(weights, dtype=np.int64))

    def __len__(self):
        return int(self.emm_keys.shape[0])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._codec.symbol(k) for k in self.emm_keys[i]]
        return self._codec.symbol(self.emm_keys[i])

    def __iter__(self):
        return (self._codec.symbol(k) for k in self.emm_keys)


class _KeyWeights:
    __slots__ = ("emm_array",)

    def __init__(self, arr):
        self.emm_array = arr

    def __len__(self):
        return int(self.emm_array.shape[0])

    def __getitem__(self, i):
        v = self.emm_array[i]
        return v.tolist()

    def __iter__(self):
        return iter(self.emm_array.tolist())
