"""Per-launch times of the Qwen2.5-VL vision tower on one C3 image (7410
merged tokens): CUDA events around every launch (ops.TIMER), printed per
kernel class (mean / min / max ms and TF/s), for A/B of attention variants
(EMM_VIT_WINDOW_PACK=0/1, EMM_ATT_TILE_ROWS)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import ops  # noqa: E402
from paper_2507_10069_b200.pipeline import HotPath  # noqa: E402
from paper_2507_10069_b200.shapes import SHAPES  # noqa: E402
from paper_2507_10069_b200.workload import ImageInput  # noqa: E402

tok = int(sys.argv[1]) if len(sys.argv) > 1 else 7410
n_img = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hp = HotPath(SHAPES["qwen-7b"], budget_tokens=100_000)
imgs = [ImageInput(f"{i:032x}", tok, (0, 0)) for i in range(n_img)]
for rep in range(4):
    hp.cd.slabs.clear()
    if rep == 3:
        ops.TIMER.start()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hp.encode(imgs)
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: encode {e0.elapsed_time(e1):.2f} ms device, "
          f"{(time.perf_counter() - t0) * 1e3:.2f} ms host", flush=True)
ops.TIMER.stop()
for kind, recs in ops.TIMER.records.items():
    ts = [r[0].elapsed_time(r[1]) for r in recs]
    w = sum(r[2] for r in recs)
    print(f"{kind:24s} n={len(ts):3d} mean {sum(ts) / len(ts):8.3f} ms min {min(ts):8.3f} "
          f"max {max(ts):8.3f} total {sum(ts):8.2f} ms  {w / (sum(ts) / 1e3) / 1e12:8.1f} TF/s")
    if kind.startswith("attention"):
        print("   first launches:", " ".join(f"{t:.3f}" for t in ts[:8]))
