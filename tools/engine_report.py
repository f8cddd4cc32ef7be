"""Measured B200 run of the unchanged reference scheduler, reported in the
reference's schema (paper_2507_10069_b200.report) and printed with the
reference's own `mmsim report`.

usage: python tools/engine_report.py --config c3 --policy elastic --instances 8 \
           [--gpus N | --logical K] [--mode B] [--out gpurun_out/report_c3.json]
"""
import argparse
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "mmsim")):
        sys.path.append(p)
        break

SHAPE = {"c1": "tiny", "c2": "llava-7b", "c3": "qwen-7b", "c4": "llama-11b-v", "c5": "qwen-72b"}


def main():
    import torch
    import mmsim.engine as E
    from mmsim import cli, experiments, workload

    from paper_2507_10069_b200 import report
    from paper_2507_10069_b200.pipeline import HotPath, HotPathSet
    from paper_2507_10069_b200.shapes import SHAPES
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--shape", default=None)
    ap.add_argument("--policy", default="elastic")
    ap.add_argument("--instances", type=int, default=8)
    ap.add_argument("--gpus", type=int, default=None, help="physical GPUs (default: all)")
    ap.add_argument("--logical", type=int, default=0,
                    help="K logical GPUs on cuda:0 (multi-GPU code paths on one GPU)")
    ap.add_argument("--mode", default="B")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "report.json"))
    a = ap.parse_args()
    cost = experiments.resolve_cost_profile("default")
    trace = workload.load_trace(os.path.join(ROOT, "tests", "golden", "traces",
                                             f"{a.config}.jsonl"))
    cfg = E.config_for_policy(a.policy, E.RunConfig(n_instances=a.instances))
    shape = SHAPES[a.shape or SHAPE[a.config]]
    if a.logical:
        hp = HotPathSet(shape, cfg.cache_budget_tokens, cfg.cache_image_fraction,
                        devices=[0] * a.logical)
    else:
        n = a.gpus or torch.cuda.device_count()
        hp = (HotPath(shape, cfg.cache_budget_tokens, cfg.cache_image_fraction) if n == 1
              else HotPathSet(shape, cfg.cache_budget_tokens, cfg.cache_image_fraction,
                              devices=list(range(n))))
    res, rep, summary = report.simulate([dataclasses.replace(r) for r in trace], a.policy, cost,
                                        cfg, hotpath=hp, mode=a.mode)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    report.write_report(a.out, rep, summary)
    # the reference's modelled run on the same inputs, for comparison
    ref = E.Engine([dataclasses.replace(r) for r in trace], a.policy, cost, cfg).run()
    from mmsim import metrics
    ref_rep = metrics.aggregate(ref)
    print("== B200 measured run (reference `mmsim report` on the written JSON)")
    cli.cmd_report(argparse.Namespace(input=a.out))
    print("b200:", summary)
    print("== reference modelled run: TTFT mean/p50/p99 "
          f"{ref_rep.aggregates['ttft']['mean']:.4f} / {ref_rep.aggregates['ttft']['p50']:.4f}"
          f" / {ref_rep.aggregates['ttft']['p99']:.4f} s")


if __name__ == "__main__":
    main()
