"""Golden-fixture generator — TEST INFRASTRUCTURE, runs only in the build
container where the read-only reference lives at /root/reference.

It imports the reference simulator `mmsim` (pure Python) and records, for the
canonical traces of SURVEY.md §8(d) (configs C1..C5 of BASELINE.json):

* the trace itself as JSON lines (reference `write_trace`,
  pkg/src/mmsim/core.py:277-281) -> tests/golden/traces/<cfg>.jsonl;
* the engine's complete cache call log per modality-group cache: every
  image_lookup / image_insert / match_prefix / insert_prefix / release with its
  `now` and its result (pkg/src/mmsim/cache.py:372-399, call sites
  pkg/src/mmsim/engine.py:470,492,545,552,593,656) plus the final
  snapshot_stats and eviction_log -> tests/golden/calllogs/<run>.json;
* per-request reference records (cached_prefix_tokens, encode/prefill
  computed tokens, modelled TTFT) (engine.py:206-225, metrics.py:20-35);
* criterion-8-style random op sequences with the reference PrefixTree's
  eviction victims (pkg/tests/test_acceptance.py:306-339).

Nothing under tests/ reads /root/reference: the GPU box only sees the JSON
written here.  Re-run with `python oracle/gen_golden.py` (about a minute).
"""
from __future__ import annotations

import dataclasses
import gzip
import hashlib
import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "..", "tests", "golden")


def _import_mmsim():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import mmsim  # noqa: F401
    from mmsim import cache, engine, experiments, metrics, workload, core
    return cache, engine, experiments, metrics, workload, core


def encode_tokens(tokens, weights):
    """Run-length encode a unified sequence (engine.py:448-461) as segments.

    ["i", hash, w]            one image symbol ("img", hash) of weight w
    ["p", pid, start, count]  ("pfx", pid, start..start+count-1), weight 1
    ["t", rid, start, count]  ("txt", rid, start..start+count-1), weight 1
    ["g", json-able, w]       any other hashable (unit tests)
    """
    segs = []
    for tok, w in zip(tokens, weights):
        if isinstance(tok, tuple) and tok and tok[0] == "img":
            segs.append(["i", tok[1], int(w)])
            continue
        if (isinstance(tok, tuple) and len(tok) == 3 and tok[0] in ("pfx", "txt")
                and int(w) == 1):
            tag = "p" if tok[0] == "pfx" else "t"
            if (segs and segs[-1][0] == tag and segs[-1][1] == tok[1]
                    and segs[-1][2] + segs[-1][3] == tok[2]):
                segs[-1][3] += 1
            else:
                segs.append([tag, tok[1], tok[2], 1])
            continue
        segs.append(["g", tok, int(w)])
    return segs


def make_recorder(cache_mod, log):
    base = cache_mod.UnifiedCache

    class RecordingCache(base):
        def __init__(self, budget_tokens, image_fraction=0.2):
            super().__init__(budget_tokens, image_fraction)
            self.cache_index = len(log["caches"])
            self.calls = []
            self._next_hid = 0
            log["caches"].append({"budget_tokens": budget_tokens,
                                  "image_fraction": image_fraction,
                                  "calls": self.calls})

        def image_lookup(self, content_hash, now):
            r = super().image_lookup(content_hash, now)
            self.calls.append(["il", content_hash, now, r])
            return r

        def image_insert(self, content_hash, token_count, now, bytes_estimate=0):
            r = super().image_insert(content_hash, token_count, now, bytes_estimate)
            self.calls.append(["ii", content_hash, token_count, now, bytes_estimate, r])
            return r

        def match_prefix(self, tokens, weights, now):
            matched, handle = super().match_prefix(tokens, weights, now)
            hid = self._next_hid
            self._next_hid += 1
            handle._golden_hid = hid  # id() can be reused after GC
            self.calls.append(["mp", encode_tokens(tokens, weights), now, matched, hid])
            return matched, handle

        def insert_prefix(self, tokens, weights, now):
            r = super().insert_prefix(tokens, weights, now)
            self.calls.append(["ip", encode_tokens(tokens, weights), now, r])
            return r

        def release(self, handle):
            hid = handle._golden_hid
            super().release(handle)
            self.calls.append(["rl", hid])

        def finish(self):
            log_entry = log["caches"][self.cache_index]
            log_entry["final_stats"] = self.snapshot_stats()
            log_entry["eviction_log"] = [list(e) for e in self.prefixes.eviction_log]
            log_entry["prefix_total_tokens"] = self.prefixes.total_tokens
            log_entry["image_total_tokens"] = self.images.total_tokens
            log_entry["n_nodes"] = sum(1 for _ in self.prefixes.iter_nodes())

    return RecordingCache


def traces(workload, experiments):
    share = experiments.resolve_dataset_profile("sharegpt4o-like")
    visual = experiments.resolve_dataset_profile("visualwebinstruct-like")
    rep = dataclasses.replace
    out = {}
    out["c1"] = workload.generate(share, 1.0, 200.0, seed=1)[:64]
    out["c2"] = workload.generate(
        rep(share, name="llava-1img", images_per_request={1: 1.0},
            image_token_choices={576: 1.0}, image_pixels={576: (336, 336)}),
        2.0, 120.0, seed=1)
    out["c3"] = workload.generate(
        rep(share, duplicate_image_rate=0.5, duplicate_prefix_rate=0.5), 1.5, 120.0,
        seed=1, bursts=[workload.BurstSpec(40, 30, 3, "multimodal")])
    out["c4"] = workload.generate(
        rep(visual, name="long-multi", images_per_request={2: 0.5, 4: 0.5},
            image_token_choices={6516: 1.0}, image_pixels={6516: (904, 904)},
            multimodal_fraction=0.6), 0.8, 120.0, seed=1)
    out["c5"] = workload.generate(share, 3.0, 90.0, seed=11)
    return out


# run name -> (trace, policy, n_instances, overrides)
RUNS = {
    "c1_elastic8": ("c1", "elastic", 8, {}),
    "c1_elastic8_tight": ("c1", "elastic", 8, {"cache_budget_tokens": 40_000}),
    "c1_coupled1": ("c1", "coupled", 1, {"cache_enabled": True}),
    "c2_coupled1": ("c2", "coupled", 1, {"cache_enabled": True,
                                          "cache_budget_tokens": 200_000}),
    "c2_elastic2": ("c2", "elastic", 2, {"cache_budget_tokens": 200_000}),
    "c3_coupled1": ("c3", "coupled", 1, {"cache_enabled": True}),
    "c3_elastic2": ("c3", "elastic", 2, {}),
    "c3_elastic4": ("c3", "elastic", 4, {}),
    "c3_elastic8": ("c3", "elastic", 8, {}),
    "c3_elastic8_tight": ("c3", "elastic", 8, {"cache_budget_tokens": 60_000}),
    "c4_elastic8": ("c4", "elastic", 8, {}),
    "c5_elastic8": ("c5", "elastic", 8, {}),
}


def record_runs(cache_mod, engine, experiments, metrics, core, trs, only=None):
    cost = experiments.resolve_cost_profile("default")
    os.makedirs(os.path.join(GOLDEN, "calllogs"), exist_ok=True)
    summary = {}
    for name, (tr_name, policy, n, overrides) in RUNS.items():
        if only and name not in only:
            continue
        log = {"run": name, "trace": tr_name, "policy": policy, "n_instances": n,
               "overrides": overrides, "caches": []}
        rec_cls = make_recorder(cache_mod, log)
        saved = engine.UnifiedCache
        engine.UnifiedCache = rec_cls
        try:
            cfg = engine.config_for_policy(policy, engine.RunConfig(n_instances=n),
                                           **overrides)
            trace = [dataclasses.replace(r) for r in trs[tr_name]]
            eng = engine.Engine(trace, policy, cost, cfg, seed=0)
            res = eng.run()
            for c in eng.caches.values():
                c.finish()
        finally:
            engine.UnifiedCache = saved
        recs = sorted(res.records, key=lambda r: r.id)
        ttft = metrics.summarize([r.ttft for r in recs])
        log["config"] = {"cache_budget_tokens": cfg.cache_budget_tokens,
                         "cache_image_fraction": cfg.cache_image_fraction,
                         "cache_enabled": cfg.cache_enabled,
                         "kv_bytes_per_token": cost.kv_bytes_per_token}
        log["requests"] = [
            {"id": r.id, "cached_prefix_tokens": r.cached_prefix_tokens,
             "encode_computed_tokens": r.encode_computed_tokens,
             "prefill_computed_tokens": r.prefill_computed_tokens,
             "input_len": r.input_len, "ttft": r.ttft} for r in recs]
        log["ttft"] = ttft
        log["counters"] = res.counters
        log["cache_stats"] = res.cache_stats
        blob = json.dumps(log, sort_keys=True, separators=(",", ":"))
        path = os.path.join(GOLDEN, "calllogs", f"{name}.json.gz")
        with gzip.open(path, "wt", encoding="utf-8", compresslevel=9) as fh:
            fh.write(blob)
        n_calls = sum(len(c["calls"]) for c in log["caches"])
        summary[name] = {"calls": n_calls, "sha256": hashlib.sha256(blob.encode()).hexdigest()[:16],
                         "ttft_p50": ttft["p50"], "ttft_p99": ttft["p99"],
                         "cached": sum(r.cached_prefix_tokens for r in recs),
                         "input": sum(r.input_len for r in recs)}
        print(name, summary[name], flush=True)
    return summary


def tree_snapshot(tree):
    nodes = {}

    def walk(node, parent_id):
        for child in node.children.values():
            nodes[child.node_id] = {"parent": parent_id, "kv": child.kv_tokens,
                                    "last_used": child.last_used,
                                    "user_count": child.user_count}
            walk(child, child.node_id)
    walk(tree.root, 0)
    return nodes


def record_op_sequences(cache_mod, n_cases=3000, seed=77):
    """Criterion-8-style random op sequences (test_acceptance.py:306-339),
    extended with weighted symbols, with every result recorded."""
    rng = random.Random(seed)
    cases = []
    for _ in range(n_cases):
        cap = rng.randint(6, 40)
        tree = cache_mod.PrefixTree(cap)
        ops = []
        handles = []
        clock = 0.0
        for _ in range(rng.randint(4, 14)):
            clock += rng.choice([0.0, 0.5, 1.0])
            op = rng.random()
            if op < 0.5:
                n = rng.randint(1, 8)
                seq = [rng.choice("abcd") for _ in range(n)]
                wts = [rng.choice([1, 1, 1, 2, 5, 9]) for _ in range(n)]
                added = tree.insert_prefix(seq, wts, now=clock)
                ops.append(["ip", seq, wts, clock, added])
            elif op < 0.8:
                n = rng.randint(1, 8)
                seq = [rng.choice("abcd") for _ in range(n)]
                wts = [rng.choice([1, 1, 1, 2, 5, 9]) for _ in range(n)]
                matched, h = tree.match_prefix(seq, wts, now=clock)
                handles.append((len(ops), h))
                ops.append(["mp", seq, wts, clock, matched])
                if len(handles) > 2:
                    idx, hh = handles.pop(0)
                    tree.release(hh)
                    ops.append(["rl", idx])
            else:
                needed = rng.randint(1, 20)
                mark = len(tree.eviction_log)
                freed = tree.evict(needed, now=clock)
                ops.append(["ev", needed, clock, freed,
                            [e[0] for e in tree.eviction_log[mark:]]])
        state = {"total_tokens": tree.total_tokens,
                 "eviction_log": [list(e) for e in tree.eviction_log],
                 "nodes": tree_snapshot(tree),
                 "increments": tree.increments, "decrements": tree.decrements}
        for idx, h in handles:
            tree.release(h)
            ops.append(["rl", idx])
        cases.append({"capacity": cap, "ops": ops, "final": state})
    path = os.path.join(GOLDEN, "op_sequences.json.gz")
    with gzip.open(path, "wt", encoding="utf-8", compresslevel=9) as fh:
        json.dump(cases, fh, sort_keys=True, separators=(",", ":"))
    print("op_sequences", len(cases))


def record_ghost_kats(cache_mod):
    """Appendix-A hazards H1/H2 measured on the reference."""
    out = []
    t = cache_mod.PrefixTree(10)
    t.insert_prefix(list("abcde"), now=0.0)
    added = t.insert_prefix(list("abcdefghijk"), now=1.0)
    m, h = t.match_prefix(list("abcdefghijk"), now=2.0)
    t.release(h)
    out.append({"name": "H1_ghost", "added": added, "total_tokens": t.total_tokens,
                "match": m, "evictions": t.evictions})
    t = cache_mod.PrefixTree(8000)
    t.insert_prefix([("img", "A"), "t0"], [7410, 1], now=0.0)
    _, h = t.match_prefix([("img", "A"), "t0"], [7410, 1], now=1.0)
    a1 = t.insert_prefix([("img", "B"), "p0"], [7410, 1], now=2.0)
    a2 = t.insert_prefix([("img", "A"), "t0"] + [f"x{i}" for i in range(700)],
                         [7410, 1] + [1] * 700, now=3.0)
    t.release(h)
    out.append({"name": "H2_trim", "added_b": a1, "added_ext": a2,
                "total_tokens": t.total_tokens})
    t = cache_mod.PrefixTree(100)
    a = t.insert_prefix([("img", "Z"), "c", "d"], [150, 1, 1], now=0.0)
    out.append({"name": "H2_oversize", "added": a, "total_tokens": t.total_tokens,
                "evictions": t.evictions})
    with open(os.path.join(GOLDEN, "hazard_kats.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("hazards", out)


def main():
    cache_mod, engine, experiments, metrics, workload, core = _import_mmsim()
    trs = traces(workload, experiments)
    os.makedirs(os.path.join(GOLDEN, "traces"), exist_ok=True)
    for name, tr in trs.items():
        core.write_trace(os.path.join(GOLDEN, "traces", f"{name}.jsonl"), tr)
        print("trace", name, len(tr), sum(r.total_input_len for r in tr))
    only = set(sys.argv[1:]) or None
    summary = record_runs(cache_mod, engine, experiments, metrics, core, trs, only)
    if not only:
        record_op_sequences(cache_mod)
        record_ghost_kats(cache_mod)
        with open(os.path.join(GOLDEN, "calllogs", "SUMMARY.json"), "w") as fh:
            json.dump(summary, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
