"""K3 gather bandwidth: rows of a Qwen-7B-shaped pool [28, 2, slots, 512] bf16
gathered through a random (fragmented) or run-contiguous slot table."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_10069_b200 import dataplane  # noqa: E402

for L, kvd, n in [(28, 512, 8000), (28, 512, 60000), (32, 4096, 6000)]:
    pool = torch.empty(L, 2, 150000, kvd, device="cuda", dtype=torch.bfloat16).uniform_()
    dst = torch.empty(L, 2, n, kvd, device="cuda", dtype=torch.bfloat16)
    for kind in ("random", "runs"):
        if kind == "random":
            rows = torch.randperm(150000, device="cuda")[:n].int()
        else:
            rows = (torch.arange(n, device="cuda") + 1234).int()
        for _ in range(3):
            dataplane.kv_copy_rows(pool, rows, dst, None, n)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            dataplane.kv_copy_rows(pool, rows, dst, None, n)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        gb = 2.0 * n * L * 2 * kvd * 2 / 1e9
        ok = torch.equal(dst[:, :, :16], pool[:, :, rows[:16].long()])
        print(f"L={L} row={kvd * 2}B n={n} {kind}: {ms:.3f} ms {gb / ms * 1e3:.0f} GB/s ok={ok}",
              flush=True)
    del pool, dst
