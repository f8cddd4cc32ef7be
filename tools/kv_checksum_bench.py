"""K6 checksum throughput: emm_kv_checksum over a Qwen2.5-VL-7B-shaped KV
buffer (28 layers x K/V x rows of 1 KiB), identity and scattered row maps;
bytes read / CUDA-event time against the measured HBM peak."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2507_10069_b200 import dataplane  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
L, slots, row = 28, 100_000, 512
planes = torch.randn(L, 2, slots, row, device="cuda").bfloat16()
for name, n, rows in (("identity", 80_000, None),
                      ("scattered", 80_000, torch.randperm(slots, device="cuda")[:80_000]
                       .to(torch.int32))):
    for _ in range(3):
        dataplane.kv_checksum(planes, rows, n)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        dataplane.kv_checksum(planes, rows, n)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    byts = L * 2 * n * row * 2
    print(f"kv_checksum {name}: {byts / 1e9:.2f} GB in {ms:.3f} ms = {byts / ms / 1e6:.0f} GB/s "
          f"({byts / ms / 1e6 / peak:.2f} of HBM)")
