"""Port of the reference's cache unit tests (pkg/tests/test_cache.py) and
acceptance criterion 8 (pkg/tests/test_acceptance.py:306-339) onto the C++
control plane, plus the recorded random op sequences and the Appendix-A
hazard KATs measured on the reference (tests/golden)."""
import random

import pytest

from goldens import load_hazards, load_op_sequences
from paper_2507_10069_b200.cache import (GpuUnifiedCache, ImagePool, PrefixTree,
                                         ReleaseWithoutMatch)


# --- image pool (test_cache.py:10-47) ---

def test_image_lookup_empty_pool_misses():
    assert ImagePool(10_000).lookup("deadbeef", now=0.0) is None


def test_image_insert_then_hit():
    pool = ImagePool(10_000)
    assert pool.insert("h1", 6516, now=0.0)
    assert pool.lookup("h1", now=1.0) == 6516


def test_image_pool_lru_eviction():
    pool = ImagePool(300)
    for i, h in enumerate("abcd"):
        pool.insert(h, 100, now=float(i + 1))
    assert pool.lookup("a", 5.0) is None
    assert pool.lookup("d", 5.0) == 100
    assert pool.total_tokens <= 300


def test_image_pool_hit_refreshes_recency():
    pool = ImagePool(200)
    pool.insert("a", 100, now=1.0)
    pool.insert("b", 100, now=2.0)
    pool.lookup("a", now=3.0)
    pool.insert("c", 100, now=4.0)
    assert pool.lookup("b", 5.0) is None
    assert pool.lookup("a", 5.0) == 100


def test_image_pool_tie_breaks_on_hash_string():
    pool = ImagePool(200)
    pool.insert("zz", 100, now=1.0)
    pool.insert("aa", 100, now=1.0)
    pool.insert("mm", 100, now=2.0)  # evicts min((1.0,"aa"),(1.0,"zz")) = "aa"
    assert pool.lookup("aa", 3.0) is None and pool.lookup("zz", 3.0) == 100


def test_image_too_large_refused():
    pool = ImagePool(100)
    assert not pool.insert("big", 101, now=0.0)
    assert pool.total_tokens == 0 and pool.evictions == 0


# --- prefix tree matching (test_cache.py:52-105) ---

def test_match_partial_prefix():
    tree = PrefixTree(1000)
    tree.insert_prefix(["a", "b", "c", "d"], now=0.0)
    matched, h = tree.match_prefix(["a", "b", "x"], now=1.0)
    assert matched == 2
    tree.release(h)


def test_match_against_brute_force_longest_common_prefix():
    rng = random.Random(4)
    for _ in range(300):
        tree = PrefixTree(10_000)
        stored = []
        for _ in range(rng.randint(1, 6)):
            seq = [rng.choice("abcdef") for _ in range(rng.randint(1, 10))]
            stored.append(seq)
            tree.insert_prefix(seq, now=rng.random())
        probe = [rng.choice("abcdef") for _ in range(rng.randint(1, 10))]
        expected = 0
        for seq in stored:
            c = 0
            for a, b in zip(seq, probe):
                if a != b:
                    break
                c += 1
            expected = max(expected, c)
        matched, h = tree.match_prefix(probe, now=99.0)
        assert matched == expected
        tree.release(h)


def test_weighted_symbols_count_kv_tokens():
    tree = PrefixTree(100_000)
    tree.insert_prefix([("img", "h"), "t0", "t1"], weights=[6516, 1, 1], now=0.0)
    matched, h = tree.match_prefix([("img", "h"), "t0", "zz"], weights=[6516, 1, 1], now=1.0)
    assert matched == 6517
    tree.release(h)


# --- insertion shape (test_cache.py:110-133) ---

def test_overlapping_inserts_share_prefix_node():
    tree = PrefixTree(1000)
    tree.insert_prefix(["a", "b", "c"], now=0.0)
    tree.insert_prefix(["a", "b", "d"], now=1.0)
    seqs = {seq for seq, _ in tree.cached_sequences()}
    assert {("a", "b"), ("a", "b", "c"), ("a", "b", "d")} <= seqs
    assert tree.total_tokens == 4


def test_reinsert_adds_nothing_and_extension_appends():
    tree = PrefixTree(1000)
    assert tree.insert_prefix(["a", "b", "c"], now=0.0) == 3
    assert tree.insert_prefix(["a", "b", "c"], now=1.0) == 0
    assert tree.insert_prefix(["a", "b", "c", "d", "e"], now=2.0) == 2
    assert tree.total_tokens == 5


# --- pins (test_cache.py:138-187) ---

def test_double_release_rejected():
    tree = PrefixTree(1000)
    tree.insert_prefix(["a"], now=0.0)
    _, h = tree.match_prefix(["a"], now=1.0)
    tree.release(h)
    with pytest.raises(ReleaseWithoutMatch):
        tree.release(h)


def test_release_of_foreign_handle_rejected():
    t1, t2 = PrefixTree(100), PrefixTree(100)
    _, h = t1.match_prefix(["a"], now=0.0)
    with pytest.raises(ReleaseWithoutMatch):
        t2.release(h)
    t1.release(h)


def test_pinned_node_survives_split():
    tree = PrefixTree(1000)
    tree.insert_prefix(["a", "b", "c", "d"], now=0.0)
    matched, h = tree.match_prefix(["a", "b", "c", "d"], now=1.0)
    assert matched == 4
    tree.insert_prefix(["a", "b", "x"], now=2.0)
    assert sum(n.user_count for n in tree.iter_nodes()) == 2
    tree.release(h)
    assert all(n.user_count == 0 for n in tree.iter_nodes())


def test_partial_pin_does_not_leak_after_split():
    tree = PrefixTree(1000)
    tree.insert_prefix(["a", "b", "c", "d"], now=0.0)
    _, h = tree.match_prefix(["a", "b"], now=1.0)
    tree.insert_prefix(["a", "b", "z"], now=2.0)
    tree.release(h)
    assert all(n.user_count == 0 for n in tree.iter_nodes())


# --- eviction (test_cache.py:192-272) ---

def test_pinned_nodes_never_evicted():
    tree = PrefixTree(10)
    tree.insert_prefix(list("abcde"), now=0.0)
    _, h = tree.match_prefix(list("abcde"), now=1.0)
    assert tree.evict(5, now=2.0) == 0
    tree.release(h)
    assert tree.evict(5, now=3.0) == 5


def test_evict_lru_order():
    tree = PrefixTree(100)
    for i, s in enumerate("abc"):
        tree.insert_prefix([s], now=float(i + 1))
    tree.evict(1, now=4.0)
    seqs = {seq for seq, _ in tree.cached_sequences()}
    assert ("a",) not in seqs and ("b",) in seqs and ("c",) in seqs


def test_capacity_never_exceeded_random_stress():
    rng = random.Random(99)
    tree = PrefixTree(50)
    handles = []
    for step in range(2000):
        op = rng.random()
        if op < 0.5:
            tree.insert_prefix([rng.choice("abcd") for _ in range(rng.randint(1, 12))],
                               now=float(step))
        elif op < 0.8:
            _, h = tree.match_prefix([rng.choice("abcd") for _ in range(rng.randint(1, 12))],
                                     now=float(step))
            handles.append(h)
            if len(handles) > 3:
                tree.release(handles.pop(0))
        else:
            tree.evict(rng.randint(1, 30), now=float(step))
        assert 0 <= tree.total_tokens <= 50
        if step % 50 == 0:
            assert sum(n.kv_tokens for n in tree.iter_nodes()) == tree.total_tokens
    for h in handles:
        tree.release(h)


def test_user_count_bookkeeping_balances():
    rng = random.Random(5)
    tree = PrefixTree(200)
    live = []
    for step in range(500):
        if rng.random() < 0.6:
            tree.insert_prefix([rng.choice("ab") for _ in range(rng.randint(1, 6))],
                               now=float(step))
        if rng.random() < 0.5:
            _, h = tree.match_prefix([rng.choice("ab") for _ in range(rng.randint(1, 6))],
                                     now=float(step))
            live.append(h)
        if live and rng.random() < 0.5:
            tree.release(live.pop(rng.randrange(len(live))))
        held = sum(len(h.entries) for h in live)
        assert tree.increments == tree.decrements + held
        assert sum(n.user_count for n in tree.iter_nodes()) == held
    for h in live:
        tree.release(h)
    assert tree.increments == tree.decrements


# --- unified cache (test_cache.py:277-300) ---

def test_unified_cache_budget_split():
    cache = GpuUnifiedCache(1000, image_fraction=0.2)
    assert cache.images.capacity == 200 and cache.prefixes.capacity == 800


def test_unified_cache_stats_flow():
    cache = GpuUnifiedCache(100_000, image_fraction=0.5)
    assert cache.image_lookup("h", 0.0) is None
    cache.image_insert("h", 6516, 0.5)
    assert cache.image_lookup("h", 1.0) == 6516
    m, h1 = cache.match_prefix(["a", "b"], [1, 1], 2.0)
    assert m == 0
    cache.insert_prefix(["a", "b"], [1, 1], 3.0)
    m, h2 = cache.match_prefix(["a", "b"], [1, 1], 4.0)
    assert m == 2
    cache.release(h1)
    cache.release(h2)
    s = cache.snapshot_stats()
    assert (s["image_hits"], s["image_misses"], s["prefix_hits"]) == (1, 1, 1)
    assert s["image_tokens_saved"] == 6516 and s["prefix_tokens_saved"] == 2


# --- recorded reference op sequences + criterion 8 ---

def _snapshot(tree):
    nodes = {}
    root = tree.root

    def walk(node, parent_id):
        for child in node.children.values():
            nodes[child.node_id] = {"parent": parent_id, "kv": child.kv_tokens,
                                    "last_used": child.last_used,
                                    "user_count": child.user_count}
            walk(child, child.node_id)
    walk(root, 0)
    return nodes


def test_recorded_op_sequences_bit_exact():
    cases = load_op_sequences()
    for ci, case in enumerate(cases):
        tree = PrefixTree(case["capacity"])
        for op in case["ops"]:
            if op[0] == "ip":
                assert tree.insert_prefix(op[1], op[2], now=op[3]) == op[4], ci
            elif op[0] == "mp":
                got, h = tree.match_prefix(op[1], op[2], now=op[3])
                assert got == op[4], ci
                op.append(h)
            elif op[0] == "rl":
                tree.release(case["ops"][op[1]][-1])
            elif op[0] == "ev":
                mark = len(tree.eviction_log)
                assert tree.evict(op[1], now=op[2]) == op[3], ci
                assert [e[0] for e in tree.eviction_log[mark:]] == op[4], ci
        fin = case["final"]
        assert tree.total_tokens == fin["total_tokens"]
        assert [list(e) for e in tree.eviction_log] == fin["eviction_log"]
        assert tree.increments == fin["increments"]
        assert tree.live_handle_count == 0 and tree.increments == tree.decrements


def test_hazard_kats():
    kats = {k["name"]: k for k in load_hazards()}
    t = PrefixTree(10)  # H1 ghost tokens
    t.insert_prefix(list("abcde"), now=0.0)
    added = t.insert_prefix(list("abcdefghijk"), now=1.0)
    m, h = t.match_prefix(list("abcdefghijk"), now=2.0)
    t.release(h)
    k = kats["H1_ghost"]
    assert (added, t.total_tokens, m, t.evictions) == (k["added"], k["total_tokens"],
                                                       k["match"], k["evictions"])
    t = PrefixTree(8000)  # H2 trimmed inserts
    t.insert_prefix([("img", "A"), "t0"], [7410, 1], now=0.0)
    _, h = t.match_prefix([("img", "A"), "t0"], [7410, 1], now=1.0)
    a1 = t.insert_prefix([("img", "B"), "p0"], [7410, 1], now=2.0)
    a2 = t.insert_prefix([("img", "A"), "t0"] + [f"x{i}" for i in range(700)],
                         [7410, 1] + [1] * 700, now=3.0)
    t.release(h)
    k = kats["H2_trim"]
    assert (a1, a2, t.total_tokens) == (k["added_b"], k["added_ext"], k["total_tokens"])
    t = PrefixTree(100)
    a = t.insert_prefix([("img", "Z"), "c", "d"], [150, 1, 1], now=0.0)
    k = kats["H2_oversize"]
    assert (a, t.total_tokens, t.evictions) == (k["added"], k["total_tokens"], k["evictions"])


def test_criterion_8_lru_matches_brute_force_oracle():
    """test_acceptance.py:306-339 (2 000 of its 10 000 sequences, same rng)."""
    def oracle_evict(nodes, needed):
        alive = {k: dict(v, children=[]) for k, v in nodes.items()}
        for nid, n in alive.items():
            if n["parent"] in alive:
                alive[n["parent"]]["children"].append(nid)
        victims, freed = [], 0
        while freed < needed:
            leaves = [n for n, v in alive.items() if not v["children"] and v["user_count"] == 0]
            if not leaves:
                break
            v = min(leaves, key=lambda n: (alive[n]["last_used"], n))
            freed += alive[v]["kv"]
            victims.append(v)
            p = alive[v]["parent"]
            if p in alive:
                alive[p]["children"].remove(v)
            del alive[v]
        return victims

    rng = random.Random(77)
    for case in range(2000):
        tree = PrefixTree(rng.randint(6, 24))
        handles, clock = [], 0.0
        for _ in range(rng.randint(4, 9)):
            clock += 1.0
            op = rng.random()
            if op < 0.55:
                tree.insert_prefix([rng.choice("abc") for _ in range(rng.randint(1, 6))],
                                   now=clock)
            elif op < 0.8:
                _, h = tree.match_prefix([rng.choice("abc") for _ in range(rng.randint(1, 6))],
                                         now=clock)
                handles.append(h)
                if len(handles) > 2:
                    tree.release(handles.pop(0))
            else:
                needed = rng.randint(1, 12)
                pinned = {n.node_id for n in tree.iter_nodes() if n.user_count > 0}
                snap = _snapshot(tree)
                mark = len(tree.eviction_log)
                tree.evict(needed, now=clock)
                got = [e[0] for e in tree.eviction_log[mark:]]
                assert got == oracle_evict(snap, needed), case
                assert not (set(got) & pinned)
            assert tree.total_tokens <= tree.capacity
        for h in handles:
            tree.release(h)
