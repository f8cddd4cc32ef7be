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

TAG_GENERIC, TAG_PFX, TAG_TXT, TAG_IMG = 0, 1, 2, 3
_MASK62 = (1 << 62) - 1
_TAG_PFX = TAG_PFX << 62
_TAG_TXT = TAG_TXT << 62
_TAG_IMG = TAG_IMG << 62


class KeyCollision(RuntimeError):
    pass


_MEMO_MAX = 1 << 22


class KeyCodec:
    def __init__(self):
        self._img_key: dict[str, int] = {}
        self._img_of: dict[int, str] = {}
        self._gen_key: dict = {}
        self._gen_of: list = []
        self._memo: dict = {}  # symbol -> key (bounded; keys are deterministic)

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
        memo = self._memo
        try:
            return np.fromiter(map(memo.__getitem__, tokens), dtype=np.uint64, count=len(tokens))
        except KeyError:
            pass
        if len(memo) > _MEMO_MAX:
            memo.clear()
        key = self.key
        for t in tokens:
            if t not in memo:
                memo[t] = key(t)
        return np.fromiter(map(memo.__getitem__, tokens), dtype=np.uint64, count=len(tokens))

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
    (pkg/src/mmsim/engine.py:448-461) for a reference `Request`."""
    n_img = len(req.images)
    prefix_len = req.prefix_len if req.prefix_id is not None else 0
    n_txt = req.text_input_len - prefix_len
    keys = np.empty(n_img + prefix_len + n_txt, dtype=np.uint64)
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


class WeightSeq(list):
    """Weights list carrying its int64 array."""

    __slots__ = ("emm_array",)


class SymbolSeq(list):
    """A unified sequence carrying its precomputed keys / weights so the cache
    boundary skips per-symbol encoding.  Iterating yields the reference's
    symbols (built lazily from the keys), so it is interchangeable with the
    list Engine.unified_sequence returns (engine.py:448-461)."""

    __slots__ = ("emm_keys", "weights")

    def __init__(self, keys: np.ndarray, weights: np.ndarray, symbols=None):
        super().__init__(symbols if symbols is not None else ())
        self.emm_keys = np.ascontiguousarray(keys, dtype=np.uint64)
        ws = WeightSeq(weights.tolist() if symbols is not None else ())
        ws.emm_array = np.ascontiguousarray(weights, dtype=np.int64)
        self.weights = ws

    def __len__(self):
        return int(self.emm_keys.shape[0])
