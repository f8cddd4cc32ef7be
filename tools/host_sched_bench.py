"""Host time of the UNCHANGED reference engine on the golden traces: pure
Python vs the C++ cache (engine.install) and/or the C++ scheduler loop
(sched.install); best of 3 runs each.  Needs the reference importable
(build container): python tools/host_sched_bench.py c3_elastic8_tight ..."""
import dataclasses
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.append("/root/reference/pkg/src")
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))
import mmsim.balancer as bal  # noqa: E402
import mmsim.engine as E  # noqa: E402
import mmsim.partition as part  # noqa: E402
from mmsim import experiments, workload  # noqa: E402

from goldens import load_calllog, trace_path  # noqa: E402
from paper_2507_10069_b200 import sched  # noqa: E402
from paper_2507_10069_b200.cache import GpuUnifiedCache  # noqa: E402

for name in sys.argv[1:] or ["c1_elastic8", "c3_elastic8_tight", "c5_elastic8"]:
    gold = load_calllog(name)
    cost = experiments.resolve_cost_profile("default")
    trace = workload.load_trace(trace_path(gold["trace"]))
    cfg = E.config_for_policy(gold["policy"], E.RunConfig(n_instances=gold["n_instances"]),
                              **gold["overrides"])

    def run():
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            E.Engine([dataclasses.replace(r) for r in trace], gold["policy"], cost, cfg,
                     seed=0).run()
            best = min(best, time.perf_counter() - t)
        return best

    t_ref = run()
    prev = sched.install(part, bal)
    t_s = run()
    pc = E.UnifiedCache
    E.UnifiedCache = GpuUnifiedCache
    t_sc = run()
    sched.uninstall(prev)
    t_c = run()
    E.UnifiedCache = pc
    print(f"{name}: reference {t_ref:.2f} s | + C++ scheduler loop {t_s:.2f} s | "
          f"+ C++ cache {t_c:.2f} s | both {t_sc:.2f} s ({t_ref / t_sc:.2f}x)", flush=True)
