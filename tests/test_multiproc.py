"""N>1 host path on CPU (gloo, world_size 2): bench.py's workload at N=2
(the C3 recipe at 2x load, sharded by cache-affine load-balanced routing)
covers every request exactly once with balanced token loads, each rank runs
its own control-plane cache on its shard, and the bench's max / sum
reductions, TTFT gather and barrier work.  (The GPU data plane is per rank; there is no data-path
collective.)"""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from goldens import trace_path


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_2507_10069_b200.cache import GpuUnifiedCache
    from paper_2507_10069_b200.driver import form_batches, shard
    from paper_2507_10069_b200.keys import KeySeq, request_keys
    from paper_2507_10069_b200.workload import read_trace
    import bench
    reqs = read_trace(trace_path("c3").replace("c3.jsonl", f"c3_x{world}.jsonl.gz"))
    mine, info = bench.load_workload("c3", rank, world)
    assert info["trace"] == f"c3_x{world}"
    assert [r.id for r in mine] == [r.id for r in shard(reqs, rank, world, balanced=True)]
    cache = GpuUnifiedCache(600_000, 0.25)
    cached = 0
    for bi, batch in enumerate(form_batches(mine, 16384)):
        hs, seqs = [], []
        for r in batch:
            k, w = request_keys(cache.codec, r)
            s = KeySeq(k, w, cache.codec)
            m, h = cache.match_prefix(s, s.weights, float(bi))
            cached += min(m, r.total_input_len - 1)
            hs.append(h)
            seqs.append(s)
        for s in seqs:
            cache.insert_prefix(s, s.weights, float(bi))
        for h in hs:
            cache.release(h)
    ids = torch.tensor([r.id for r in mine] + [-1] * (len(reqs) - len(mine)))
    gathered = [torch.zeros_like(ids) for _ in range(world)]
    dist.all_gather(gathered, ids)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        all_ids = sorted(int(x) for g in gathered for x in g.tolist() if x >= 0)
        out.put((all_ids, [r.id for r in reqs], float(t.item())))
    c = torch.tensor([cached])
    dist.all_reduce(c)
    load = torch.tensor([float(sum(r.total_input_len for r in mine))], dtype=torch.float64)
    loads = [torch.zeros_like(load) for _ in range(world)]
    dist.all_gather(loads, load)
    parts = [None] * world
    dist.all_gather_object(parts, [float(rank)] * (rank + 1))
    if rank == 0:
        out.put(int(c.item()))
        out.put(([float(x.item()) for x in loads], parts))
    dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    all_ids, want, tmax = q.get(timeout=300)
    cached = q.get(timeout=300)
    loads, parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert all_ids == sorted(want)          # every request exactly once
    assert tmax == 2.0                      # max-over-ranks reduction
    assert cached > 0                       # affinity routing keeps prefix hits
    assert max(loads) / (sum(loads) / 2) < 1.05   # balanced token loads
    assert parts == [[0.0], [1.0, 1.0]]     # TTFT-list gather
