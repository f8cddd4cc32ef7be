"""Cache-path CPU leg — TEST / BASELINE INFRASTRUCTURE ONLY.

SURVEY.md §8d CPU leg 1 / BASELINE.md §4.1: the reference engine's recorded
cache calls on a canonical trace (tests/golden/calllogs/*.json.gz, written by
oracle/gen_golden.py from the UNCHANGED reference engine, with its retries)
replayed through a cache class, timed in µs per request, every result
checked against the recorded one.  Arms:

  reference  mmsim.cache.UnifiedCache (pkg/src/mmsim/cache.py:363-406), the
             symbol lists exactly as Engine.unified_sequence builds them
  symbols    GpuUnifiedCache fed the same symbol lists (what install() binds)
  keys       GpuUnifiedCache fed precomputed uint64 keys (what B200Engine
             and the GPU driver pass)
"""
from __future__ import annotations

import gzip
import json
import os
import time

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                      "golden", "calllogs")


def load(name: str) -> dict:
    with gzip.open(os.path.join(GOLDEN, f"{name}.json.gz"), "rt") as fh:
        return json.load(fh)


def decode_segments(segs):
    """Run-length segments of gen_golden.encode_tokens -> (symbols, weights)."""
    toks, wts = [], []
    for s in segs:
        kind = s[0]
        if kind == "i":
            toks.append(("img", s[1]))
            wts.append(s[2])
        elif kind in ("p", "t"):
            tag = "pfx" if kind == "p" else "txt"
            toks.extend((tag, s[1], s[2] + i) for i in range(s[3]))
            wts.extend([1] * s[3])
        else:
            toks.append(s[1] if not isinstance(s[1], list) else tuple(s[1]))
            wts.append(s[2])
    return toks, wts


def materialise(log: dict, codec=None) -> list:
    """Decode every call's symbols once (outside the timed region); with a
    codec, precompute keys (keys.KeySeq) as the product's callers do."""
    out = []
    for clog in log["caches"]:
        calls = []
        for call in clog["calls"]:
            op = call[0]
            if op in ("mp", "ip"):
                toks, wts = decode_segments(call[1])
                if codec is not None:
                    from paper_2507_10069_b200.keys import KeySeq
                    k, w = codec.keys_weights(toks, wts)
                    toks = KeySeq(k, w, codec)
                    wts = toks.weights
                calls.append((op, toks, wts) + tuple(call[2:]))
            else:
                calls.append(tuple(call))
        out.append((clog["budget_tokens"], clog["image_fraction"], calls))
    return out


def replay_timed(make_cache, mats) -> float:
    """Seconds spent inside the cache calls; raises on the first result
    that differs from the recorded one."""
    total = 0.0
    pc = time.perf_counter
    for budget, frac, calls in mats:
        cache = make_cache(budget, frac)
        handles = {}
        t0 = pc()
        for call in calls:
            op = call[0]
            if op == "il":
                got, want = cache.image_lookup(call[1], call[2]), call[3]
            elif op == "ii":
                got, want = cache.image_insert(call[1], call[2], call[3], call[4]), call[5]
            elif op == "mp":
                got, h = cache.match_prefix(call[1], call[2], call[3])
                want = call[4]
                handles[call[5]] = h
            elif op == "ip":
                got, want = cache.insert_prefix(call[1], call[2], call[3]), call[4]
            else:
                cache.release(handles.pop(call[1]))
                continue
            if got != want:
                raise AssertionError(f"cache replay mismatch: {op} got {got} want {want}")
        total += pc() - t0
    return total


def leg(name: str = "c3_elastic8", arms=("reference",), repeats: int = 3) -> dict:
    """µs per request (best of `repeats`) of each arm on one golden run."""
    log = load(name)
    n_req = len(log["requests"]) if "requests" in log else sum(
        1 for c in log["caches"] for x in c["calls"] if x[0] == "ip")
    n_calls = sum(len(c["calls"]) for c in log["caches"])
    res = {"calllog": name, "trace": log.get("trace"), "policy": log.get("policy"),
           "instances": log.get("n_instances"), "requests": n_req, "cache_calls": n_calls,
           "cores": 1, "unit": "us/request"}
    syms = None
    for arm in arms:
        if arm == "reference":
            from mmsim.cache import UnifiedCache
            syms = syms or materialise(log)
            t = min(replay_timed(UnifiedCache, syms) for _ in range(repeats))
        elif arm == "symbols":
            from paper_2507_10069_b200.cache import GpuUnifiedCache
            syms = syms or materialise(log)
            t = min(replay_timed(GpuUnifiedCache, syms) for _ in range(repeats))
        elif arm == "keys":
            from paper_2507_10069_b200.cache import GpuUnifiedCache
            from paper_2507_10069_b200.keys import KeyCodec
            codec = KeyCodec()
            pre = materialise(log, codec)
            t = min(replay_timed(lambda b, f: GpuUnifiedCache(b, f, codec=codec), pre)
                    for _ in range(repeats))
        else:
            raise ValueError(arm)
        res[f"{arm}_us_per_request"] = 1e6 * t / n_req
    if "reference_us_per_request" in res:
        for arm in ("symbols", "keys"):
            if f"{arm}_us_per_request" in res:
                res[f"speedup_{arm}"] = (res["reference_us_per_request"]
                                         / res[f"{arm}_us_per_request"])
    return res
