"""Request routing and prefill batching — pure Python, no native code, so
the CPU reference arm of bench.py can form exactly the GPU driver's batches
without loading libemm.so.

* form_batches: arrival order, <= max_tokens input tokens per batch (the
  reference's per-instance cap, RunConfig.max_batch_tokens_per_instance,
  pkg/src/mmsim/engine.py:80; budgeted on total_input_len like dispatch,
  engine.py:1057-1060).
* route / route_balanced / shard: cache-affine request routing over ranks
  (requests are independent units).
"""
from __future__ import annotations


def affinity_key(req) -> str:
    """The request's first unified-sequence symbol (engine.py:448-461): its
    first image, else its shared system prefix, else its own text — requests
    with equal keys can share a cached prefix."""
    if req.images:
        return "img:" + req.images[0].content_hash
    if req.prefix_id is not None and req.prefix_len > 0:
        return f"pfx:{req.prefix_id}"
    return f"txt:{req.id}"


def route(req, world: int) -> int:
    """Stateless cache-affine routing: hash of the affinity key mod world.
    Deterministic across processes."""
    import hashlib
    key = affinity_key(req)
    return int.from_bytes(hashlib.blake2b(key.encode(), digest_size=8).digest(), "big") % world


def route_balanced(reqs, world: int) -> list[int]:
    """Online cache-affine routing with load balance: in arrival order, a
    request whose affinity key was seen goes to that key's rank (its cached
    prefix lives there); a new key goes to the rank with the fewest input
    tokens routed so far.  Uses only past requests, deterministic, so every
    rank computes the same assignment without communication."""
    owner: dict[str, int] = {}
    load = [0] * world
    out = []
    for r in sorted(reqs, key=lambda r: (r.arrival_time, r.id)):
        k = affinity_key(r)
        g = owner.get(k)
        if g is None:
            g = min(range(world), key=lambda i: (load[i], i))
            owner[k] = g
        load[g] += r.total_input_len
        out.append((r.id, g))
    by_id = dict(out)
    return [by_id[r.id] for r in reqs]


def shard(reqs, rank: int, world: int, balanced: bool = False):
    """This rank's requests (arrival order preserved) under `route`, or
    under `route_balanced` when balanced=True."""
    if balanced:
        ranks = route_balanced(reqs, world)
        return [r for r, g in zip(reqs, ranks) if g == rank]
    return [r for r in reqs if route(r, world) == rank]


def form_batches(reqs, max_tokens: int):
    out, cur, tok = [], [], 0
    for r in reqs:
        n = r.total_input_len
        if cur and tok + n > max_tokens:
            out.append(cur)
            cur, tok = [], 0
        cur.append(r)
        tok += n
    if cur:
        out.append(cur)
    return out
