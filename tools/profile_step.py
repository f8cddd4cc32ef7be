"""One representative C3 batch (Qwen2.5-VL-7B shape) inside an NVTX range
"prof" for ncu (--nvtx --nvtx-include prof/): the first `--warm` batches of the
trace run first (cache and slabs populated), then batch `--batch` runs in the
range: ViT encode of its missed images (32 layers: windowed attention except
layers 7/15/23/31), then the prefix-cached prefill (28 decoder layers) and the
insert scatter.  Kernel order inside the range is deterministic."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200.driver import PassStats, TraceDriver, form_batches  # noqa: E402
from paper_2507_10069_b200.pipeline import HotPath  # noqa: E402
from paper_2507_10069_b200.shapes import SHAPES  # noqa: E402
from paper_2507_10069_b200.workload import read_trace  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--trace", default="c3")
ap.add_argument("--shape", default="qwen-7b")
ap.add_argument("--warm", type=int, default=6)
ap.add_argument("--batch", type=int, default=6)
args = ap.parse_args()
reqs = read_trace(os.path.join(ROOT, "tests", "golden", "traces", f"{args.trace}.jsonl"))
hp = HotPath(SHAPES[args.shape], budget_tokens=600_000, image_fraction=0.25)
drv = TraceDriver(hp, max_batch_tokens=16384)
batches = form_batches(reqs, 16384)
hp.new_cache()
st = PassStats()
for bi in range(args.warm):
    drv.run_batch(batches[bi], float(bi), st)
torch.cuda.synchronize()
b = batches[args.batch]
n_img = len({i.content_hash for r in b for i in r.images if i.content_hash not in hp.slabs})
torch.cuda.nvtx.range_push("prof")
drv.run_batch(b, float(args.batch), st)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(f"batch {args.batch}: {len(b)} requests, {sum(r.total_input_len for r in b)} input tokens, "
      f"{n_img} images to encode", flush=True)
