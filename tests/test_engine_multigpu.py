"""B200Engine over several logical GPUs: encode jobs split
their images over the job's GPUs, prefill batches split their requests over
the compute GPUs, each group's cache lives on one GPU and is gathered from /
scattered into peer-to-peer, and a request's KV is handed to its home
instance's GPU when the placement differs.  The box has one B200, so the
logical GPUs share it (HotPathSet(devices=[0, 0, 0, 0])) — the same code
paths, launched back to back.  Every scheduling / cache decision must equal a
plain reference Engine run; every request's first token must equal a
one-GPU B200Engine run's, and its prefill KV must too: bit-identical in
layer 0, within bf16 tolerance after it (the residual GEMMs accumulate each
row's sum of squares for the next RMSNorm with fp32 atomics across N tiles,
so later layers are not bitwise reproducible even run to run)."""
import dataclasses

import pytest

from conftest import have_mmsim
from goldens import trace_path

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_mmsim(), reason="reference scheduler not importable")]




def _run(hotpath, trace, cost, cfg):
    from paper_2507_10069_b200.engine import B200Engine
    eng = B200Engine([dataclasses.replace(r) for r in trace], "elastic", cost, cfg,
                     hotpath=hotpath, mode="A")
    sig = {}
    orig = eng._handle_prefill_done

    def spy(ev):
        before = set(eng.resident)
        orig(ev)
        for rid in set(eng.resident) - before:
            d, kv = eng.resident[rid]
            assert kv.device == eng.hps[d].device
            assert d == eng.device_of(eng.requests[rid].home_instance)
            sig[rid] = (d, kv.clone())
    eng._handle_prefill_done = spy
    res = eng.run()
    return eng, res, sig


def test_engine_split_over_logical_gpus():
    import mmsim.engine as E
    import torch
    from mmsim import experiments, workload
    from paper_2507_10069_b200 import shapes
    from paper_2507_10069_b200.pipeline import HotPath, HotPathSet
    cost = experiments.resolve_cost_profile("default")
    trace = workload.load_trace(trace_path("c3"))[:120]
    cfg = E.config_for_policy("elastic", E.RunConfig(n_instances=4))
    ref = E.Engine([dataclasses.replace(r) for r in trace], "elastic", cost, cfg).run()

    one = HotPath(shapes.TINY, budget_tokens=cfg.cache_budget_tokens,
                  image_fraction=cfg.cache_image_fraction)
    e1, r1, sig1 = _run(one, trace, cost, cfg)
    del one
    four = HotPathSet(shapes.TINY, cfg.cache_budget_tokens, cfg.cache_image_fraction,
                      devices=[0, 0, 0, 0])
    e4, r4, sig4 = _run(four, trace, cost, cfg)

    for res in (r1, r4):
        assert res.counters == ref.counters
        assert res.cache_stats == ref.cache_stats
        ref_recs = {r.id: r for r in ref.records}
        for r in res.records:
            assert r.ttft == ref_recs[r.id].ttft
            assert r.cached_prefix_tokens == ref_recs[r.id].cached_prefix_tokens
    # the split really happened
    assert e4.gpu["prefill_split"] > 0 and e4.gpu["encode_split"] > 0
    assert e4.gpu["handoffs"] > 0
    assert len(set(e4.gpu["device_of_prefill"].values())) == 4
    # device match agrees with the host tree on every logical GPU
    for rid, c in e4.gpu["host_cached_prefix"].items():
        m = e4.gpu["device_matched_kv"][rid]
        total = e4.requests[rid].req.total_input_len
        assert m >= c and (m == c or c == total - 1), (rid, m, c)
    # same results as the one-GPU run; KV resident on the home GPU
    assert e4.gpu["first_tokens"] == e1.gpu["first_tokens"]
    assert set(sig4) == set(sig1)
    for rid, (d, kv) in sig4.items():
        ref_kv = sig1[rid][1]
        assert kv.shape == ref_kv.shape
        assert torch.equal(kv[0], ref_kv[0]), rid
        err = (kv.float() - ref_kv.float()).norm() / ref_kv.float().norm().clamp_min(1e-30)
        assert err.item() < 1e-2, (rid, err.item())


def test_c5_golden_on_eight_logical_gpus():
    """The C5 golden run (Qwen2.5-VL-72B recipe: mixed text-only and
    multimodal groups, 42 migrations at 8 instances) with every instance on
    its own logical GPU: every cache decision / TTFT equals the reference's
    recorded run while jobs split over GPUs, KV is handed to home GPUs and
    migrations copy between GPUs."""
    import mmsim.engine as E
    from goldens import load_calllog
    from mmsim import experiments, workload
    from paper_2507_10069_b200 import shapes
    from paper_2507_10069_b200.engine import B200Engine
    from paper_2507_10069_b200.pipeline import HotPathSet
    gold = load_calllog("c5_elastic8")
    cost = experiments.resolve_cost_profile("default")
    trace = workload.load_trace(trace_path(gold["trace"]))
    cfg = E.config_for_policy(gold["policy"], E.RunConfig(n_instances=gold["n_instances"]),
                              **gold["overrides"])
    hps = HotPathSet(shapes.TINY, cfg.cache_budget_tokens, cfg.cache_image_fraction,
                     devices=[0] * 8)
    eng = B200Engine([dataclasses.replace(r) for r in trace], gold["policy"], cost, cfg,
                     hotpath=hps, mode="A")
    res = eng.run()
    recs = {r.id: r for r in res.records}
    for w in gold["requests"]:
        assert recs[w["id"]].cached_prefix_tokens == w["cached_prefix_tokens"]
        assert recs[w["id"]].ttft == w["ttft"]
    assert res.cache_stats == gold["cache_stats"]
    assert eng.gpu["prefill_split"] > 0 and eng.gpu["handoffs"] > 0
    assert len(set(eng.gpu["device_of_prefill"].values())) > 1
    assert len(eng.migration_log) > 0


@pytest.mark.parametrize("transport", ["copy_engine", "nccl"])
def test_elastic_mode_b_four_gpus_transport(transport):
    """The bench's elastic leg (bench.engine_elastic_leg) on four logical GPUs
    of one B200 (devices=[0, 0, 0, 0], the C3 recipe at 4x load): mode B over the unchanged elastic
    scheduler, KV hand-offs timed, every request served.  With one physical
    GPU the "nccl" transport keeps the K6 kernel for same-device pairs
    (NCCL needs distinct devices; its binding is tested on its own below)."""
    import bench
    from paper_2507_10069_b200 import shapes
    leg = bench.engine_elastic_leg(shapes.TINY, "c3", 4, [0, 0, 0, 0], transport)
    b = leg["b200"]
    assert leg["requests"] > 0 and leg["ttft"]["p99_s"] >= leg["ttft"]["p50_s"] > 0
    assert b["kv_transport"] == transport and b["physical_devices"] == [0]
    assert b["prefill_batches"] > 0 and b["kv_handoffs"] > 0
    assert b["kv_handoff_bytes"] > 0 and b["kv_handoff_gbs"] > 0
    assert leg["prefill_tokens_per_s_per_gpu"] > 0


def test_nccl_p2p_binding_bit_exact():
    """NcclP2P (grouped ncclSend / ncclRecv per (layer, K/V) plane) moves a
    strided request-KV view bit-exactly; one GPU = NCCL's send-to-self."""
    import torch
    from paper_2507_10069_b200.nccl_p2p import NcclP2P
    nc = NcclP2P([0])
    g = torch.Generator(device="cuda").manual_seed(5)
    buf = torch.randn(4, 2, 900, 512, device="cuda", generator=g).bfloat16()
    src = buf[:, :, 100:100 + 700]            # a request's rows inside a batch buffer
    dst = torch.empty(4, 2, 700, 512, device="cuda", dtype=torch.bfloat16)
    src2 = buf[:, :, :50]
    dst2 = torch.zeros(4, 2, 50, 512, device="cuda", dtype=torch.bfloat16)
    nc.move_many([(src, dst, 700), (src2, dst2, 50)])
    torch.cuda.synchronize()
    assert torch.equal(dst, src) and torch.equal(dst2, src2)
    nc.close()
