"""The bench's decode leg step by step: the C3 trace's requests decoded with
continuous batching exactly as bench.py does (driver.run_decode), one record
per step (batch, KV rows read, longest row, ms); summarised per batch bucket
as GB/s and fraction of HBM (decoder weights once per step + KV rows).

  python tools/decode_leg_probe.py [config] [n_requests] > gpurun_out/decode_leg.txt
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_10069_b200.driver import TraceDriver  # noqa: E402
from paper_2507_10069_b200.pipeline import HotPath  # noqa: E402
from paper_2507_10069_b200.shapes import SHAPES  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tr, shape_name, budget, frac, _ = bench.CONFIGS[cfg]
reqs, _ = bench.load_workload(tr, 0, 1)
if nreq:
    reqs = reqs[:nreq]
shape = SHAPES[shape_name]
hp = HotPath(shape, budget_tokens=budget, image_fraction=frac)
drv = TraceDriver(hp)
hp.stage_pixels({i.content_hash: i for r in reqs for i in r.images}.values())
free_b, _ = torch.cuda.mem_get_info()
n_slots = int(min(600_000, 0.5 * free_b / shape.decoder.kv_bytes_per_token))
drv.run_decode(reqs[:4], max_active=4, n_slots=n_slots)
clocks: list = []
if "--clocks" in sys.argv:   # SM clock at every step's start (a sync per step)
    import pynvml

    from paper_2507_10069_b200.decode import DecodeSession
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    _step = DecodeSession.step

    def _clocked(self, *a, **k):
        torch.cuda.synchronize()
        clocks.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
        return _step(self, *a, **k)
    DecodeSession.step = _clocked
log: list = []
dd = drv.run_decode(reqs, max_active=64, n_slots=n_slots, step_log=log)
d = shape.decoder
wbytes = dd["hbm_bytes"] - sum(r[1] for r in log) * d.kv_layers * 2 * d.kv_dim * 2
wbytes /= dd["steps"]
row = d.kv_layers * 2 * d.kv_dim * 2
peak = bench.measured_peaks()["hbm_gbs"]
a = np.array([r[:3] + r[4:] for r in log], dtype=np.float64)   # b, rows, max, ms, admitted
print(f"# {cfg}: {dd['steps']} steps, {dd['generated_tokens']} tokens, "
      f"{dd['tokens_per_s']:.0f} tok/s, weights {wbytes / 1e9:.2f} GB/step, peak {peak} GB/s")
print(f"# overall {dd['hbm_bytes'] / dd['device_s'] / 1e9:.0f} GB/s")
edges = [0, 1, 2, 4, 8, 16, 24, 32, 40, 48, 56, 64]
for lo, hi in zip(edges[:-1], edges[1:]):
    m = (a[:, 0] > lo) & (a[:, 0] <= hi)
    if not m.any():
        continue
    s = a[m]
    by = s.shape[0] * wbytes + s[:, 1].sum() * row
    ms = s[:, 3].sum()
    print(f"B ({lo:2d},{hi:2d}]  steps {int(m.sum()):4d}  ms/step {ms / m.sum():6.3f}  "
          f"kv/row mean {s[:, 1].sum() / s[:, 0].sum():7.0f}  max {s[:, 2].max():6.0f}  "
          f"{by / ms / 1e6:6.0f} GB/s  {by / ms / 1e6 / peak:.2f}  share {ms / a[:, 3].sum():.2f}")
big = [r for r in log if r[0] == 64]
if big:
    r = big[len(big) // 2]
    print("# a 64-row step:", r[4], "ms, kv lengths", r[3])
json.dump(log, open(os.path.join(ROOT, "gpurun_out", f"decode_leg_{cfg}.json"), "w"))

# steps right after an admission (a prefill ran just before) vs steady steps
m64 = a[:, 0] == 64
for name, m in (("after admission", m64 & (a[:, 4] > 0)), ("1-3 after", None), ("steady", None)):
    pass
adm = np.where(a[:, 4] > 0)[0]
since = np.full(len(a), 10 ** 6)
last = -10 ** 6
for i in range(len(a)):
    if a[i, 4] > 0:
        last = i
    since[i] = i - last
for lo, hi in ((0, 0), (1, 3), (4, 10), (11, 30), (31, 10 ** 7)):
    m = m64 & (since >= lo) & (since <= hi)
    if m.any():
        ck = f", SM clock {np.mean(np.array(clocks)[m]):.0f} MHz" if len(clocks) == len(a) else ""
        print(f"# B=64 steps {lo}-{hi} after an admission: {int(m.sum())} steps, "
              f"{a[m, 3].mean():.3f} ms/step, kv/row {a[m, 1].sum() / a[m, 0].sum():.0f}{ck}")
