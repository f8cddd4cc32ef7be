"""Bit-exact cache decisions: every call the reference engine made on the
canonical traces (C1..C5, several policies / budgets), replayed through the
C++ control plane, must return exactly what mmsim.cache returned, and the
final stats / eviction logs must be identical.  Fixtures: tests/golden/calllogs
(oracle/gen_golden.py)."""
import os

import pytest

from goldens import calllog_names, load_calllog, replay
from paper_2507_10069_b200.cache import GpuUnifiedCache

SMALL = [n for n in calllog_names() if n not in ("c2_elastic2", "c3_elastic2", "c3_elastic4")]
BIG = ["c2_elastic2", "c3_elastic2", "c3_elastic4"]


def _check_run(name):
    log = load_calllog(name)
    assert log["caches"], name
    for ci, clog in enumerate(log["caches"]):
        cache = GpuUnifiedCache(clog["budget_tokens"], clog["image_fraction"])
        bad = replay(clog, cache)
        assert not bad, f"{name} cache {ci}: first mismatches {bad[:5]}"
        stats = cache.snapshot_stats()
        assert stats == clog["final_stats"], (name, ci, stats, clog["final_stats"])
        got_log = [list(e) for e in cache.prefixes.eviction_log]
        assert got_log == clog["eviction_log"], (name, ci)
        assert cache.prefixes.total_tokens == clog["prefix_total_tokens"]
        assert cache.images.total_tokens == clog["image_total_tokens"]
        assert sum(1 for _ in cache.prefixes.iter_nodes()) == clog["n_nodes"]
        assert cache.prefixes.live_handle_count == 0


@pytest.mark.parametrize("name", SMALL)
def test_replay_bit_exact(name):
    _check_run(name)


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("EMM_SLOW_TESTS"), reason="set EMM_SLOW_TESTS=1")
@pytest.mark.parametrize("name", BIG)
def test_replay_bit_exact_retry_heavy(name):
    # hundreds of thousands of scheduler-retry lookups
    _check_run(name)
