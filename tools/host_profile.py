"""Host-side cost of one C3 backlog pass (cProfile): where the Python / C++
control-plane time goes while the GPU runs the step.  The pass is GPU-bound
when this total stays well under the device time."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200.driver import TraceDriver  # noqa: E402
from paper_2507_10069_b200.pipeline import HotPath  # noqa: E402
from paper_2507_10069_b200.shapes import SHAPES  # noqa: E402
from paper_2507_10069_b200.workload import read_trace  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
reqs = read_trace(os.path.join(ROOT, "tests", "golden", "traces", "c3.jsonl"))
hp = HotPath(SHAPES["qwen-7b"], budget_tokens=600_000, image_fraction=0.25)
drv = TraceDriver(hp, max_batch_tokens=16384)
hp.stage_pixels({i.content_hash: i for r in reqs for i in r.images}.values())
drv.run_backlog(reqs)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
drv.run_backlog(reqs)
pr.disable()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host returned after {t1 - t0:.2f} s, GPU drained after {t2 - t0:.2f} s")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
