"""Host boundary: symbol -> key encoding (keys.py, csrc/py/seqcodec.c) and the
lazy match entry point (emm_cache_match_prefix_lazy) agree with the Python
codec and with the reference cache (pkg/src/mmsim/cache.py:121-156, 363-406)."""
import random

import numpy as np
import pytest

from conftest import have_mmsim
from paper_2507_10069_b200.cache import GpuUnifiedCache
from paper_2507_10069_b200.keys import KeyCodec, KeySeq, request_keys
from paper_2507_10069_b200.workload import ImageInput, Request


def _slow_keys(codec, toks, weights):
    n = len(toks) if weights is None else min(len(toks), len(weights))
    k = np.array([codec.key(t) for t in toks[:n]], dtype=np.uint64)
    w = (np.ones(n, np.int64) if weights is None
         else np.asarray(list(weights)[:n], dtype=np.int64))
    return k, w


def test_keys_weights_matches_per_symbol_codec():
    rng = random.Random(5)
    codec = KeyCodec()
    for trial in range(200):
        toks, wts = [], []
        for _ in range(rng.randint(0, 60)):
            r = rng.random()
            if r < 0.1:
                toks.append(("img", f"{rng.randint(0, 7):x}" * 32))
                wts.append(rng.randint(1, 7000))
            elif r < 0.4:
                toks.append(("pfx", rng.randint(0, 5), rng.randint(0, 100)))
                wts.append(1)
            elif r < 0.85:
                toks.append(("txt", rng.randint(0, 1 << 31), rng.randint(0, 1 << 33)))
                wts.append(1)
            elif r < 0.9:
                toks.append(rng.choice(["a", "b", 3, (1, 2), ("txt", True, 1)]))
                wts.append(rng.choice([1, 2.0, np.int64(3)]))
            else:
                toks.append(("txt", -1, 0))
                wts.append(1)
        if trial % 3 == 0 and toks:
            wts = wts[: rng.randint(0, len(wts))]  # zip() truncation
        weights = None if trial % 7 == 0 else wts
        got = codec.keys_weights(toks, weights)
        want = _slow_keys(codec, toks, weights)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_request_keys_out_of_range_ids_fall_back():
    codec = KeyCodec()
    img = ImageInput("f" * 32, 64, (0, 0))
    for rid, pid in [(5, 7), ((1 << 30) + 3, 7), (5, (1 << 31)), ((1 << 40), (1 << 33))]:
        req = Request(rid, 0.0, "multimodal", 20, (img,), 4, prefix_id=pid, prefix_len=6)
        syms = [("img", img.content_hash)] + [("pfx", pid, i) for i in range(6)] + \
               [("txt", rid, i) for i in range(14)]
        w = [64] + [1] * 20
        k, ww = request_keys(codec, req)
        k2, w2 = codec.keys_weights(syms, w)
        assert np.array_equal(k, k2) and np.array_equal(ww, w2)
        assert len(set(k.tolist())) == len(k)
        assert list(KeySeq(k, ww, codec)) == syms


def test_keyseq_iterates_symbols():
    codec = KeyCodec()
    req = Request(9, 0.0, "multimodal", 12, (ImageInput("a" * 32, 10, (0, 0)),), 4,
                  prefix_id=2, prefix_len=3)
    k, w = request_keys(codec, req)
    s = KeySeq(k, w, codec)
    syms = list(s)
    assert len(syms) == len(s) == 13
    assert syms[0] == ("img", "a" * 32) and syms[1] == ("pfx", 2, 0) and syms[-1] == ("txt", 9, 8)
    assert list(s.weights) == [10] + [1] * 12 and s[4] == ("txt", 9, 0)


def _seqs(rng, n_req):
    out = []
    for rid in range(n_req):
        toks, wts = [], []
        for _ in range(rng.randint(0, 2)):
            toks.append(("img", f"{rng.randint(0, 3):x}" * 32))
            wts.append(rng.choice([576, 6516]))
        pid = rng.randint(0, 3)
        plen = rng.choice([0, 5, 31, 32, 33, 127, 128, 129, 600])
        toks += [("pfx", pid, i) for i in range(plen)]
        wts += [1] * plen
        ntxt = rng.choice([0, 1, 40, 300, 2000])
        toks += [("txt", rid, i) for i in range(ntxt)]
        wts += [1] * ntxt
        out.append((toks, wts))
    return out


@pytest.mark.skipif(not have_mmsim(), reason="reference not importable")
def test_lazy_match_equals_reference():
    from mmsim.cache import UnifiedCache as Ref
    rng = random.Random(11)
    seqs = _seqs(rng, 160)
    for budget in (600_000, 3_000):
        ref, emm = Ref(budget, 0.25), GpuUnifiedCache(budget, 0.25)
        emk = GpuUnifiedCache(budget, 0.25)
        now = 0.0
        for toks, wts in seqs:
            now += 1.0
            a, ha = ref.match_prefix(toks, wts, now)
            b, hb = emm.match_prefix(toks, wts, now)
            k, w = emk.codec.keys_weights(toks, wts)
            ks = KeySeq(k, w, emk.codec)
            c, hc = emk.match_prefix(ks, ks.weights, now)
            assert a == b == c
            if rng.random() < 0.7:
                x = ref.insert_prefix(toks, wts, now)
                assert emm.insert_prefix(toks, wts, now) == x
                assert emk.insert_prefix(ks, ks.weights, now) == x
            ref.release(ha)
            emm.release(hb)
            emk.release(hc)
        assert ref.snapshot_stats() == emm.snapshot_stats() == emk.snapshot_stats()


def test_cache_methods_accept_the_reference_keywords():
    """The C methods take positional or keyword arguments under the
    reference's parameter names (cache.py:372-406)."""
    from paper_2507_10069_b200.cache import GpuUnifiedCache, ReleaseWithoutMatch
    c = GpuUnifiedCache(1000, 0.2)
    seq = [("pfx", 3, 0), ("pfx", 3, 1), ("txt", 7, 0)]
    assert c.insert_prefix(tokens=seq, weights=[1, 1, 1], now=0.0) == 3
    m, h = c.match_prefix(seq, [1, 1, 1], now=1.0)
    assert m == 3 and not h.released
    c.release(handle=h)
    assert h.released
    with pytest.raises(ReleaseWithoutMatch):
        c.release(h)
    assert c.image_lookup(content_hash="f" * 32, now=2.0) is None
    with pytest.raises(TypeError):
        c.match_prefix(seq, [1, 1, 1])
    with pytest.raises(TypeError):
        c.match_prefix(seq, [1, 1, 1], 1.0, now=2.0)


def test_c_core_differential_against_reference_mixed_symbols():
    """Randomised differential run of the C cache core against the reference
    UnifiedCache on symbol lists that exercise every branch of the C walk:
    ("txt" | "pfx", id, i) runs sharing (and not sharing) the id object,
    images seen for the first time, plain strings / ints / other tuples
    (the Python codec path), ids and offsets outside the packed ranges, and
    keyword / positional calls mixed."""
    import random
    mmsim_cache = pytest.importorskip("mmsim.cache")
    from paper_2507_10069_b200.cache import GpuUnifiedCache
    rng = random.Random(11)
    ours, ref = GpuUnifiedCache(3000, 0.2), mmsim_cache.UnifiedCache(3000, 0.2)
    pool = [("img", "%032x" % rng.getrandbits(128)) for _ in range(6)]

    def seq():
        syms, w = [], []
        for _ in range(rng.randint(1, 4)):
            kind = rng.random()
            if kind < 0.35:
                tag, rid = rng.choice(["txt", "pfx"]), rng.choice([1, 2, 3, 2**31, 7])
                start = rng.choice([0, 0, 5, 2**33])
                syms += [(tag, rid, start + i) for i in range(rng.randint(1, 40))]
            elif kind < 0.55:
                syms.append(rng.choice(pool))
            elif kind < 0.75:
                syms.append(rng.choice(["a", "b", "c", 17, ("x", 1), ("txt", "s", 1)]))
            else:
                tag = "".join(["t", "x", "t"])          # equal, not the interned object
                syms += [(tag, 9, i) for i in range(rng.randint(1, 10))]
        for s in syms:
            w.append(rng.choice([1, 1, 1, 64]) if isinstance(s, tuple) and s[0] == "img" else 1)
        return syms, w

    handles = []
    for step in range(400):
        now = float(step)
        syms, w = seq()
        if rng.random() < 0.5:
            assert ours.insert_prefix(syms, w, now) == ref.insert_prefix(syms, w, now)
        m1, h1 = ours.match_prefix(syms, w, now=now)
        m2, h2 = ref.match_prefix(syms, w, now)
        assert m1 == m2, (step, syms[:4])
        handles.append((h1, h2))
        if handles and rng.random() < 0.6:
            a, b = handles.pop(rng.randrange(len(handles)))
            ours.release(a)
            ref.release(b)
    s1, s2 = ours.snapshot_stats(), ref.snapshot_stats() if hasattr(ref, "snapshot_stats") else None
    if s2 is not None:
        assert s1 == s2


def test_precomputed_keys_any_8_byte_buffer():
    """The ndarray fast path (data pointer read directly) and the buffer
    protocol fallback (non-ndarray or non-contiguous keys) decide alike."""
    import array
    codec = KeyCodec()
    toks = [("txt", 7, i) for i in range(40)]
    k, w = codec.keys_weights(toks, [1] * 40)
    base = GpuUnifiedCache(10_000, 0.2, codec=codec)
    assert base.insert_prefix(KeySeq(k, w, codec), KeySeq(k, w, codec).weights, 0.0) == 40
    variants = {
        "ndarray": (k, w),
        "array.array": (array.array("Q", k.tolist()), array.array("q", w.tolist())),
        "strided": (np.repeat(k, 2)[::2], np.repeat(w, 2)[::2]),
    }
    for name, (kk, ww) in variants.items():
        seq = KeySeq(np.asarray(k), np.asarray(w), codec)
        seq.emm_keys = kk
        seq.weights.emm_array = ww
        try:
            m, h = base.match_prefix(seq, seq.weights, 1.0)
        except (TypeError, BufferError, ValueError):
            assert name == "strided", name  # non-contiguous: refused, never misread
            continue
        assert m == 40, name
        base.release(h)
