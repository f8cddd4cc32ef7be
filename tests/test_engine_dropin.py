"""Drop-in boundary: the UNCHANGED reference scheduler (mmsim.engine) runs on
GpuUnifiedCache (install()) and on B200Engine (control plane only), and
every cache call, per-request result and statistic equals the reference's
own recorded run (tests/golden/calllogs)."""
import dataclasses

import pytest

from conftest import have_mmsim
from goldens import load_calllog, recording_cache_class, trace_path

pytestmark = pytest.mark.skipif(not have_mmsim(), reason="reference scheduler not importable")

RUNS = ["c1_elastic8", "c1_elastic8_tight", "c1_coupled1", "c3_elastic8_tight", "c5_elastic8"]


def _run(name, engine_factory):
    import mmsim.engine as E
    from mmsim import experiments, workload
    from paper_2507_10069_b200.cache import GpuUnifiedCache
    gold = load_calllog(name)
    cost = experiments.resolve_cost_profile("default")
    trace = workload.load_trace(trace_path(gold["trace"]))
    cfg = E.config_for_policy(gold["policy"], E.RunConfig(n_instances=gold["n_instances"]),
                              **gold["overrides"])
    log = []
    prev = E.UnifiedCache
    E.UnifiedCache = recording_cache_class(GpuUnifiedCache, log)
    try:
        res = engine_factory(E, [dataclasses.replace(r) for r in trace], gold["policy"], cost,
                             cfg).run()
    finally:
        E.UnifiedCache = prev
    assert len(log) == len(gold["caches"])
    for got, want in zip(log, gold["caches"]):
        assert got["calls"] == want["calls"], name
        assert got["cache"].snapshot_stats() == want["final_stats"]
    recs = {r.id: r for r in res.records}
    for w in gold["requests"]:
        r = recs[w["id"]]
        assert r.cached_prefix_tokens == w["cached_prefix_tokens"]
        assert r.prefill_computed_tokens == w["prefill_computed_tokens"]
        assert r.encode_computed_tokens == w["encode_computed_tokens"]
        assert r.ttft == pytest.approx(w["ttft"], abs=0, rel=0)
    assert res.cache_stats == gold["cache_stats"]
    assert res.counters == gold["counters"]


@pytest.mark.parametrize("name", RUNS)
def test_reference_engine_on_gpu_unified_cache(name):
    _run(name, lambda E, tr, pol, cost, cfg: E.Engine(tr, pol, cost, cfg, seed=0))


@pytest.mark.parametrize("name", ["c1_elastic8", "c1_coupled1"])
def test_b200_engine_control_plane_only(name):
    from paper_2507_10069_b200.engine import B200Engine
    _run(name, lambda E, tr, pol, cost, cfg: B200Engine(tr, pol, cost, cfg, seed=0,
                                                         hotpath=None))
