"""Where the device waits on the host: one C3 backlog pass with CUDA events
around every timed launch plus the host time spent inside each launch call;
prints the launches whose device-time bracket is far above the class median,
with the host time inside the call and the previous launch."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402
from paper_2507_10069_b200.driver import TraceDriver  # noqa: E402
from paper_2507_10069_b200.pipeline import HotPath  # noqa: E402
from paper_2507_10069_b200.shapes import SHAPES  # noqa: E402
from paper_2507_10069_b200.workload import read_trace  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
trace = sys.argv[1] if len(sys.argv) > 1 else "c3"
shape = sys.argv[2] if len(sys.argv) > 2 else "qwen-7b"
reqs = read_trace(os.path.join(ROOT, "tests", "golden", "traces", f"{trace}.jsonl"))
hp = HotPath(SHAPES[shape], budget_tokens=600_000, image_fraction=0.25)
drv = TraceDriver(hp, max_batch_tokens=16384)
hp.stage_pixels({i.content_hash: i for r in reqs for i in r.images}.values())
drv.run_backlog(reqs)
torch.cuda.synchronize()
import gc  # noqa: E402
if os.environ.get("NO_GC"):
    gc.disable()
gc_t = []
gc.callbacks.append(lambda phase, info: gc_t.append((phase, time.perf_counter(), info["generation"])))
ops.TIMER.start(trace=True)
s0 = torch.cuda.Event(enable_timing=True)
s0.record()
drv.run_backlog(reqs)
torch.cuda.synchronize()
ops.TIMER.stop()
tr = ops.TIMER.trace
dev = [s.elapsed_time(e) for _, s, e, _, _ in tr]
med = {}
for k in {t[0] for t in tr}:
    med[k] = statistics.median(d for d, t in zip(dev, tr) if t[0] == k)
gaps = [s0.elapsed_time(tr[0][1])] + [tr[i - 1][2].elapsed_time(tr[i][1]) for i in range(1, len(tr))]
print(f"launches {len(tr)}; device time in brackets {sum(dev):.1f} ms; "
      f"device gaps between brackets {sum(gaps):.1f} ms")
ex = sorted(range(len(tr)), key=lambda i: -(dev[i] - med[tr[i][0]]))[:25]
tot_ex = sum(max(0.0, dev[i] - 3 * med[tr[i][0]]) for i in range(len(tr)))
print(f"excess over 3x class median, all launches: {tot_ex:.1f} ms")
pauses = [(gc_t[i + 1][1] - gc_t[i][1]) * 1e3 for i in range(len(gc_t) - 1)
          if gc_t[i][0] == "start" and gc_t[i + 1][0] == "stop"]
print(f"gc collections {len(pauses)}, total {sum(pauses):.1f} ms, max {max(pauses, default=0):.1f} ms")
hic = sorted((t[3] * 1e3 for t in tr), reverse=True)[:10]
print("largest host-in-call (ms):", " ".join(f"{x:.1f}" for x in hic))
for i in ex:
    k, s, e, h, h0 = tr[i]
    prev = tr[i - 1][0] if i else "-"
    dh = (h0 - tr[i - 1][4]) * 1e3 if i else 0.0
    print(f"#{i:6d} {k:22s} dev {dev[i]:8.3f} ms (median {med[k]:.3f}) host-in-call "
          f"{h * 1e3:7.3f} ms  host since prev launch {dh:8.3f} ms  prev {prev}")
