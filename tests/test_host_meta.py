"""Host-side attention work descriptions (no GPU): the packed-window groups
of AttnMeta.window_packed must cover every row exactly once with whole
windows, fit one 128-row tile, and give each row the same visible keys as
the one-sequence-per-image `windows=` form."""
import numpy as np
import pytest

from paper_2507_10069_b200.encoder import window_plan
from paper_2507_10069_b200.ops import pack_windows


def _cases():
    yield [0], [[64] * 9 + [32, 16, 64]]
    yield [0, 2300], [[64, 64, 48, 16, 64, 40, 24] * 7, [128, 8, 120, 64, 100, 64]]
    for gh, gw in [(84, 88), (36, 52), (10, 14), (2, 2)]:
        p = window_plan(gh, gw, 2, 112 // 14)
        yield [7], [p["window_lens"]]


@pytest.mark.parametrize("case", list(_cases()))
def test_pack_windows(case):
    starts, wins = case
    g_start, g_len, rb = pack_windows(starts, wins, 128)
    assert (g_len > 0).all() and (g_len <= 128).all()
    covered = np.zeros(len(rb), np.int64)
    for s, n in zip(g_start, g_len):
        covered[s:s + n] += 1
    for st, w in zip(starts, wins):
        n = int(np.sum(w))
        assert (covered[st:st + n] == 1).all()
        # expected absolute window of every row
        lo_abs = np.repeat(st + np.cumsum(w) - w, w)
        hi_abs = lo_abs + np.repeat(w, w)
        rows = np.arange(st, st + n)
        grp = np.searchsorted(g_start, rows, side="right") - 1
        assert (rb[rows, 0] + g_start[grp] == lo_abs).all()
        assert (rb[rows, 1] + g_start[grp] == hi_abs).all()
        # windows are whole inside their group
        assert (rb[rows, 0] >= 0).all() and (rb[rows, 1] <= g_len[grp]).all()


def test_pack_windows_qwen_interior_pairs():
    """Interior 8x8-patch windows (64 rows) pack two per tile."""
    p = window_plan(84, 88, 2, 8)
    g_start, g_len, _ = pack_windows([0], [p["window_lens"]], 128)
    assert np.mean(g_len == 128) > 0.8


def test_split_balanced():
    from paper_2507_10069_b200.pipeline import split_balanced
    costs = [7410, 6516, 6516, 1036, 2304, 50, 7410]
    parts = split_balanced(costs, 3)
    assert sorted(i for p in parts for i in p) == list(range(len(costs)))
    assert all(p == sorted(p) for p in parts)
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(costs)
    assert split_balanced([5], 4) == [[0], [], [], []]
    assert split_balanced([], 2) == [[], []]


def test_decode_arena_slots_cpu():
    """Token-granular arena bookkeeping (paged decode KV): allocations are
    disjoint, release returns them, exhaustion raises."""
    from paper_2507_10069_b200 import shapes
    from paper_2507_10069_b200.decode import DecodeArena
    a = DecodeArena(shapes.TINY, 100, device="cpu")
    x, y = a.alloc(30), a.alloc(50)
    assert len(set(x.tolist()) | set(y.tolist())) == 80 and a.free_slots == 20
    a.release(x)
    z = a.alloc(40)
    assert not set(z.tolist()) & set(y.tolist()) and a.free_slots == 10
    with pytest.raises(MemoryError):
        a.alloc(11)
    a.release(y)
    a.release(z)
    assert a.free_slots == 100 and sorted(a.alloc(100).tolist()) == list(range(100))
