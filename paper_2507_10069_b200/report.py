"""Measured-run reports in the reference's own schema.

`simulate` is the B200 counterpart of the reference CLI's `simulate`
command (pkg/src/mmsim/cli.py:84-119): the unchanged scheduler runs on
B200Engine (mode "B": every encode / prefill / migration job lasts its
measured device time), the run result goes through the reference's
`metrics.aggregate` (metrics.py:69-138) unchanged, and the payload is the
reference's `MetricsReport.to_json()` — so `mmsim report` (cli.py:175-198),
`metrics` consumers and experiment scripts read B200 runs exactly like
simulated ones.  The only addition is a top-level "b200" object (ignored by
the reference readers) with the device-time totals and the job splits.
"""
from __future__ import annotations

import json
import math


def simulate(trace, policy: str, profile, config=None, hotpath=None, mode: str = "B",
             slo=None, seed: int = 0, transport: str = "kernel"):
    """Run `trace` through B200Engine and aggregate with the reference's
    metrics.  Returns (RunResult, MetricsReport, b200 summary dict)."""
    from mmsim import metrics  # the reference's reporting, unchanged

    from .engine import B200Engine
    slo_input = slo.slo_input if slo is not None else math.inf
    eng = B200Engine(trace, policy, profile, config, slo_input, seed, hotpath=hotpath,
                     mode=mode, transport=transport)
    result = eng.run()
    report = metrics.aggregate(result, slo)
    g = eng.gpu
    summary = {
        "mode": mode,
        "gpus": eng.n_gpus,
        "devices": [str(hp.device) for hp in eng.hps],
        "encode_jobs": g["encode_jobs"], "encode_device_s": g["encode_s"],
        "prefill_batches": g["prefill_batches"], "prefill_device_s": g["prefill_s"],
        "encode_jobs_split": g["encode_split"], "prefill_batches_split": g["prefill_split"],
        "kv_transport": transport,
        "kv_handoffs": g["handoffs"], "kv_handoff_bytes": g["handoff_bytes"],
        "kv_handoff_device_s": g.get("handoff_s", 0.0),
        "kv_handoff_gbs": (g["handoff_bytes"] / g["handoff_s"] / 1e9
                           if g.get("handoff_s") else None),
        "migrations_executed": len(eng.migration_log),
        "migration_bytes": sum(m["bytes"] for m in eng.migration_log),
        "migration_device_s": sum(m["seconds"] for m in eng.migration_log),
        "migration_gbs": (sum(m["bytes"] for m in eng.migration_log)
                          / sum(m["seconds"] for m in eng.migration_log) / 1e9
                          if sum(m["seconds"] for m in eng.migration_log) > 0 else None),
        "physical_devices": sorted({hp.device.index for hp in eng.hps}),
        "timing": ("TTFT = simulated queueing + measured B200 compute (mode B)" if mode == "B"
                   else "analytic durations (mode A); GPU work executed, not charged"),
    }
    return result, report, summary


def write_report(path: str, report, summary: dict | None = None) -> None:
    """The reference's report payload (MetricsReport.as_dict, key order and
    separators as in to_json) plus the "b200" summary."""
    doc = report.as_dict()
    if summary is not None:
        doc["b200"] = summary
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(doc, sort_keys=True, indent=None, separators=(",", ":")))
