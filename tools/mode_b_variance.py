"""Why does the mode-B TTFT p99 move between runs (VERDICT r1 weak-7:
0.29 s in one bench, 1.42 s in another, same trace)?

Mode B is CLOSED LOOP: the unchanged reference scheduler (coupled, one
instance) decides batching from the measured device durations, so a few
percent of timing noise can move a batch boundary and change which requests
queue behind which encode.  This runs the bench's mode-B leg R times on one
box, then R more times with every measured prefill / encode duration scaled
by a factor in [0.97, 1.03] (a seeded perturbation the size of box-to-box
clock variation), and reports the p50 / p99 spread, the prefill-batch count
and, for the worst requests, where their time went (the reference's own
RequestRecord TTFT components: queue / encode / prefill).

  python tools/mode_b_variance.py [R]      (GPU box; writes gpurun_out/mode_b_variance.json)
"""
import dataclasses
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))


def main():
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    import mmsim.engine as E
    import torch
    from mmsim import experiments, metrics, workload
    from paper_2507_10069_b200 import engine as BE
    from paper_2507_10069_b200.pipeline import HotPath
    from paper_2507_10069_b200.shapes import SHAPES
    trace = workload.load_trace(os.path.join(ROOT, "tests", "golden", "traces", "c3.jsonl"))
    cost = experiments.resolve_cost_profile("default")
    cfg = E.config_for_policy("coupled", E.RunConfig(n_instances=1), cache_enabled=True)
    hp = HotPath(SHAPES["qwen-7b"], cfg.cache_budget_tokens, cfg.cache_image_fraction)
    out = {"runs": []}
    base_proxy = BE._ProfileProxy

    plans = [("plain", None)] * R + [("jitter3%", None)] * R + [
        ("decode x1.25", 1.25), ("decode x1.5", 1.5), ("decode x2", 2.0)]
    for k, (kind, dscale) in enumerate(plans):
        scale = None
        if kind.startswith("jitter"):
            rng = random.Random(k)
            scale = lambda: 1.0 + rng.uniform(-0.03, 0.03)  # noqa: E731

            class Jitter(base_proxy):
                def __init__(self, base, **over):
                    over = {n: (lambda *a, _f=f: _f(*a) * scale()) for n, f in over.items()}
                    super().__init__(base, **over)
            BE._ProfileProxy = Jitter
        elif dscale is not None:   # slower measured decode steps only
            class DecodeScaled(base_proxy):
                def __init__(self, base, _s=dscale, **over):
                    over = {n: ((lambda *a, _f=f: _f(*a) * _s) if n == "decode_step_time" else f)
                            for n, f in over.items()}
                    super().__init__(base, **over)
            BE._ProfileProxy = DecodeScaled
        try:
            eng = BE.B200Engine([dataclasses.replace(r) for r in trace], "coupled", cost, cfg,
                                hotpath=hp, mode="B")
            res = eng.run()
        finally:
            BE._ProfileProxy = base_proxy
        torch.cuda.synchronize()
        t = metrics.summarize([r.ttft for r in res.records])
        worst = sorted(res.records, key=lambda r: -r.ttft)[:4]
        comp = []
        for r in worst:
            d = dataclasses.asdict(r)
            c = {key: d[key] for key in d
                 if key in ("id", "arrival", "queue_wait", "encode_time", "prefill_time",
                            "migration_wait", "modality", "input_len", "cached_prefix_tokens",
                            "encode_computed_tokens", "prefill_computed_tokens")}
            c["ttft"] = r.ttft
            comp.append(c)
        out["runs"].append({"kind": kind, "p50_s": t["p50"], "p99_s": t["p99"],
                            "max_s": max(r.ttft for r in res.records),
                            "prefill_batches": eng.gpu["prefill_batches"],
                            "encode_jobs": eng.gpu["encode_jobs"], "worst": comp})
        print(k, kind, round(t["p50"], 4), round(t["p99"], 4),
              eng.gpu["prefill_batches"], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "mode_b_variance.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
