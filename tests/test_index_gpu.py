"""End-to-end data-plane parity (K1 + K2 + block tables + KV scatter/gather).

The reference engine's recorded cache call logs are replayed through a
GpuUnifiedCache with a DeviceIndex attached.  Every insert carries KV rows
whose bytes are a function of (block hash of the symbol, token offset), so a
gathered row is only correct if hashing, publish/erase, virtual->slot maps,
the scatter and the block table all are.  At every match the device result
(matched symbols / KV tokens) must equal the reference's recorded result and
the gathered prefix KV must equal the expected bytes exactly.
"""
import numpy as np
import pytest
import torch

from goldens import decode_segments, load_calllog
from oracle import hashes

pytestmark = pytest.mark.gpu

L, KV_DIM = 2, 8  # 16-byte rows, int16 payload (exact integers)


def _expected_rows(keys, w, n_tokens):
    """[L, 2, n_tokens, KV_DIM] int16 payload for the first n_tokens KV tokens."""
    h0, _ = hashes.prefix_hashes(keys, w)
    sym = np.repeat(np.arange(len(keys)), w)[:n_tokens]
    starts = np.concatenate([[0], np.cumsum(w)[:-1]])
    off = np.arange(n_tokens, dtype=np.uint64) - starts[sym].astype(np.uint64)
    base = h0[sym] * np.uint64(0x9E3779B97F4A7C15) + off * np.uint64(0xBF58476D1CE4E5B9)
    lh = np.arange(L * 2, dtype=np.uint64).reshape(L, 2, 1, 1)
    e = np.arange(KV_DIM, dtype=np.uint64).reshape(1, 1, 1, KV_DIM)
    x = base.reshape(1, 1, -1, 1) + lh * np.uint64(0x94D049BB133111EB) + e * np.uint64(1315423911)
    x ^= x >> np.uint64(29)
    x *= np.uint64(0xD6E8FEB86659FD93)
    x ^= x >> np.uint64(32)
    return (x & np.uint64(0x7FFF)).astype(np.int16)


@pytest.mark.parametrize("name", ["c1_elastic8", "c1_elastic8_tight", "c3_elastic8_tight"])
def test_replay_with_device_index(name):
    from paper_2507_10069_b200.cache import GpuUnifiedCache
    from paper_2507_10069_b200 import dataplane
    log = load_calllog(name)
    checked = 0
    for clog in log["caches"]:
        cache = GpuUnifiedCache(clog["budget_tokens"], clog["image_fraction"])
        ix = dataplane.DeviceIndex(cache, n_layers=L, kv_dim=KV_DIM, dtype=torch.int16)
        ix.pool.zero_()
        handles = {}
        for call in clog["calls"]:
            op = call[0]
            if op == "il":
                assert cache.image_lookup(call[1], call[2]) == call[3]
            elif op == "ii":
                assert cache.image_insert(call[1], call[2], call[3], call[4]) == call[5]
            elif op == "ip":
                toks, wts = decode_segments(call[1])
                keys = cache.codec.keys(toks)
                w = np.asarray(wts, np.int64)
                total = int(w.sum())
                req = torch.from_numpy(_expected_rows(keys, w, total)).cuda()
                ix.set_request_buffer(req)
                h0, h1 = hashes.prefix_hashes(keys, w)
                ix.set_kv_source(int(h0[-1]), int(h1[-1]), 0)
                assert cache.insert_prefix(toks, wts, call[2]) == call[3]
                ix.clear_kv_sources()
                torch.cuda.synchronize()
                del req
            elif op == "mp":
                toks, wts = decode_segments(call[1])
                got, handle = cache.match_prefix(toks, wts, call[2])
                assert got == call[3]
                handles[call[4]] = handle
                keys = cache.codec.keys(toks)
                w = np.asarray(wts, np.int64)
                b = dataplane.block_hash([keys], [w])
                res = ix.match(b, [got])
                torch.cuda.synchronize()
                assert int(res["matched_kv"][0]) == got
                if got:
                    bt = res["bt"][:got].long()
                    gathered = ix.pool[:, :, bt, :].cpu().numpy()
                    assert np.array_equal(gathered, _expected_rows(keys, w, got))
                checked += 1
            elif op == "rl":
                cache.release(handles.pop(call[1]))
        info = ix.info()
        assert info["device_error"] == 0
        assert cache.snapshot_stats() == clog["final_stats"]
        # every reachable symbol is published, every slot accounted for
        n_syms = sum(len(n.span) for n in cache.prefixes.iter_nodes())
        assert info["live_symbols"] == n_syms
        assert info["free_slots"] == ix.n_slots - cache.prefixes.total_tokens
    assert checked > 10


def test_kv_copy_rows_matches_torch():
    from paper_2507_10069_b200 import dataplane
    g = torch.Generator(device="cuda").manual_seed(1)
    for row_elems, n_layers, n in [(8, 1, 1), (64, 2, 1000), (512, 3, 777), (4096, 2, 300),
                                   (8192, 1, 50)]:
        src = torch.randint(-30000, 30000, (n_layers, 2, 2000, row_elems), generator=g,
                            device="cuda", dtype=torch.int16)
        dst = torch.zeros(n_layers, 2, 3000, row_elems, device="cuda", dtype=torch.int16)
        si = torch.randperm(2000, device="cuda", generator=g)[:n].int()
        di = torch.randperm(3000, device="cuda", generator=g)[:n].int()
        dataplane.kv_copy_rows(src, si, dst, di, n)
        torch.cuda.synchronize()
        ref = torch.zeros_like(dst)
        ref[:, :, di.long()] = src[:, :, si.long()]
        assert torch.equal(dst, ref), (row_elems, n_layers, n)
