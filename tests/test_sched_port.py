"""Scheduler host loop in C++  vs the reference's Python:
LoadEstimator (balancer.py:115-164), assign_idle_instances
(balancer.py:67-84), place_reservations (partition.py:169-184) and
allocate_prefill (partition.py:187-290) fuzzed on random inputs — every
result, float and decision record equal — then the golden engine runs
replayed with all four installed next to the C++ cache."""
import dataclasses
import random
import time

import pytest

from conftest import have_mmsim

pytestmark = pytest.mark.skipif(not have_mmsim(), reason="reference scheduler not importable")


def _profile(rng):
    from mmsim import experiments
    base = experiments.resolve_cost_profile("default")
    if rng.random() < 0.5:
        return base
    return dataclasses.replace(
        base, prefill_rate=rng.uniform(500, 50000), parallel_alpha=rng.uniform(0, 0.9),
        migration_bandwidth=rng.uniform(1e3, 1e6), decode_base=rng.uniform(1e-3, 0.1),
        decode_batch_coeff=rng.uniform(0, 1e-3), decode_kv_coeff=rng.uniform(0, 1e-3),
        encode_rate=rng.uniform(100, 20000), decode_batch_threshold=rng.randint(1, 64))


def test_load_estimator_matches_reference():
    from mmsim import balancer as bal
    from paper_2507_10069_b200 import sched
    rng = random.Random(1)
    for case in range(60):
        prof = _profile(rng)
        window = rng.choice([60.0, 30.0, 7.5, rng.uniform(1, 100)])
        bucket = rng.choice([5.0, 2.5, rng.uniform(0.1, 10)])
        ref, ours = bal.LoadEstimator(prof, window, bucket), sched.LoadEstimator(prof, window,
                                                                                bucket)
        now = rng.uniform(0, 5)
        for _ in range(300):
            op = rng.random()
            if op < 0.5:
                args = (rng.randint(0, 20000), rng.choice([0, rng.randint(1, 30000)]),
                        rng.randint(0, 2000))
                assert ours.service_seconds(*args) == ref.service_seconds(*args)
                ref.observe(now, *args)
                ours.observe(now, *args)
            elif op < 0.75:
                assert ours.avg_required(now) == ref.avg_required(now), case
            else:
                assert ours.peak_required(now) == ref.peak_required(now), case
            # bucket-boundary times hit CPython's float floor division
            now += rng.choice([0.0, bucket, rng.expovariate(2.0), rng.uniform(0, window)])
        assert len(ours) == len(ref._events)


def test_assign_idle_instances_matches_reference():
    from mmsim import balancer as bal
    from paper_2507_10069_b200 import sched
    rng = random.Random(2)
    for _ in range(500):
        groups = rng.sample(range(10), rng.randint(0, 5))
        avg = {g: rng.choice([0, rng.randint(1, 40)]) for g in groups}
        busy = {g: rng.randint(0, 8) for g in groups if rng.random() < 0.8}
        idle = list(range(rng.randint(0, 12)))
        assert sched.assign_idle_instances(avg, busy, idle) == \
            bal.assign_idle_instances(avg, busy, idle)


def _specs(part, rng, n):
    out = []
    for i in range(n):
        inp = rng.randint(1, 8000)
        out.append(part.PrefillRequestSpec(request_id=100 + i, kv_need=inp + rng.randint(0, 500),
                                           input_len=inp, prefill_tokens=rng.randint(1, inp)))
    return out


def test_place_reservations_matches_reference():
    from mmsim import partition as part
    from paper_2507_10069_b200 import sched
    rng = random.Random(3)
    for _ in range(500):
        reqs = _specs(part, rng, rng.randint(0, 8))
        head = {rng.randint(0, 15): rng.choice([0, rng.randint(0, 20000)])
                for _ in range(rng.randint(0, 6))}
        assert sched.place_reservations(reqs, head) == part.place_reservations(reqs, head)


def _alloc_tuple(a):
    return (list(a.instance_ids), a.placements if a.placements is None else dict(a.placements),
            list(a.preempted), list(a.forced_preempted), list(a.dropped), list(a.decisions))


def test_allocate_prefill_matches_reference():
    from mmsim import partition as part
    from paper_2507_10069_b200 import sched
    rng = random.Random(4)
    kinds = {"forced": 0, "opportunistic": 0, "dropped": 0}
    for case in range(1500):
        prof = _profile(rng)
        reqs = _specs(part, rng, rng.randint(0, 6))
        ids = rng.sample(range(16), rng.randint(0, 12))
        n_idle = rng.randint(0, len(ids))
        idle = [part.InstanceSlot(i, rng.choice([0, rng.randint(0, 30000)])) for i in ids[:n_idle]]
        victims = []
        for i in ids[n_idle:]:
            cap = rng.randint(1000, 40000)
            used = rng.randint(0, cap)
            victims.append(part.DecodeVictim(i, cap - used, used, cap, rng.random() < 0.85))
        outs = tuple(rng.randint(1, 2000) for _ in range(rng.randint(0, 10)))
        batch = part.DecodeBatchView(outs, sum(outs) // 2, rng.randint(0, 200000),
                                     rng.randint(1, len(victims) + 2))
        extra = None
        if rng.random() < 0.5:
            extra = [part.InstanceSlot(rng.randint(0, 20), rng.randint(0, 20000))
                     for _ in range(rng.randint(0, 3))]
        w = rng.choice([0.0, 1.0, rng.uniform(0, 20)])
        mx = rng.choice([None, None, rng.randint(0, 8)])
        ref = part.allocate_prefill(prof, reqs, idle, victims, batch, w, mx, extra)
        ours = sched.allocate_prefill(prof, reqs, idle, victims, batch, w, mx, extra)
        assert _alloc_tuple(ours) == _alloc_tuple(ref), case
        kinds["forced"] += bool(ref.forced_preempted)
        kinds["opportunistic"] += len(ref.preempted) > len(ref.forced_preempted)
        kinds["dropped"] += bool(ref.dropped)
    assert all(v >= 20 for v in kinds.values()), kinds   # every branch exercised


RUNS = ["c1_elastic8", "c1_elastic8_tight", "c3_elastic8_tight", "c5_elastic8"]


@pytest.mark.parametrize("name", RUNS)
def test_golden_runs_with_native_scheduler(name):
    """The unchanged reference engine with the C++ cache AND the C++
    scheduler loop installed reproduces the reference's recorded run."""
    import mmsim.balancer as bal
    import mmsim.engine as E
    import mmsim.partition as part
    from mmsim import experiments, workload
    from paper_2507_10069_b200 import sched
    from paper_2507_10069_b200.cache import GpuUnifiedCache
    from goldens import load_calllog, recording_cache_class, trace_path
    gold = load_calllog(name)
    cost = experiments.resolve_cost_profile("default")
    trace = workload.load_trace(trace_path(gold["trace"]))
    cfg = E.config_for_policy(gold["policy"], E.RunConfig(n_instances=gold["n_instances"]),
                              **gold["overrides"])

    def run_once():
        t0 = time.perf_counter()
        res = E.Engine([dataclasses.replace(r) for r in trace], gold["policy"], cost, cfg,
                       seed=0).run()
        return res, time.perf_counter() - t0

    _, t_ref = run_once()
    log = []
    prev_cache = E.UnifiedCache
    E.UnifiedCache = recording_cache_class(GpuUnifiedCache, log)
    prev = sched.install(part, bal)
    try:
        res, t_native = run_once()
    finally:
        sched.uninstall(prev)
        E.UnifiedCache = prev_cache
    for got, want in zip(log, gold["caches"]):
        assert got["calls"] == want["calls"], name
    recs = {r.id: r for r in res.records}
    for w in gold["requests"]:
        r = recs[w["id"]]
        assert r.cached_prefix_tokens == w["cached_prefix_tokens"]
        assert r.prefill_computed_tokens == w["prefill_computed_tokens"]
        assert r.ttft == w["ttft"]
    assert res.cache_stats == gold["cache_stats"]
    assert res.counters == gold["counters"]
    print(f"{name}: reference engine {t_ref:.2f} s, with C++ cache + scheduler loop "
          f"{t_native:.2f} s")
