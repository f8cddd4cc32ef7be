"""K6 transport microbenchmark: GB/s of moving one request's KV
([L, 2, rows, kv_dim] bf16, Qwen2-7B shape: 28 layers x 512) between two
devices with the SM copy kernel (peer loads / stores), the copy engines
(one strided cudaMemcpy2DAsync) and NCCL grouped send / recv, against the
measured peer bandwidth (B200_PROFILING.md: 770 GB/s per direction, 900
nominal).  One GPU: src = dst = cuda:0 (an HBM copy, read + write).

  python tools/kv_transport_bench.py [src_dev dst_dev]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_10069_b200 import dataplane  # noqa: E402
from paper_2507_10069_b200.nccl_p2p import NcclP2P  # noqa: E402


def main():
    a = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    b = int(sys.argv[2]) if len(sys.argv) > 2 else (1 if torch.cuda.device_count() > 1 else 0)
    if a != b:
        from paper_2507_10069_b200 import _lib
        import ctypes
        _lib.declare_more({"emm_enable_peer_access": (ctypes.c_int, [ctypes.c_int,
                                                                     ctypes.c_int])})
        for x, y in ((a, b), (b, a)):
            _lib.check(_lib.lib.emm_enable_peer_access(x, y))
    nc = NcclP2P(sorted({a, b}))
    res = {"src": a, "dst": b, "shape": "28 x 2 x rows x 512 bf16 (Qwen2-7B KV)"}
    for rows in (1024, 7410, 16384):
        buf = torch.randn(28, 2, rows + 64, 512, device=f"cuda:{a}").bfloat16()
        src = buf[:, :, 32:32 + rows]
        dst = torch.empty(28, 2, rows, 512, device=f"cuda:{b}", dtype=torch.bfloat16)
        nbytes = src.numel() * 2
        for tname in ("kernel", "copy_engine", "nccl"):
            def run():
                with torch.cuda.device(b):
                    if tname == "nccl":
                        nc.move_many([(src, dst, rows)])
                    else:
                        dataplane.kv_move(src, dst, rows, tname)
            for _ in range(3):
                run()
            torch.cuda.synchronize(a)
            torch.cuda.synchronize(b)
            with torch.cuda.device(b):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(10):
                    run()
                e.record()
                e.synchronize()
            ms = s.elapsed_time(e) / 10
            assert torch.equal(dst.to(f"cuda:{a}"), src), tname
            res[f"{tname}_rows{rows}_gbs"] = nbytes / ms / 1e6
            print(f"{tname:12s} rows {rows:6d}: {nbytes / 1e6:8.1f} MB  {ms * 1e3:8.1f} us  "
                  f"{nbytes / ms / 1e6:7.1f} GB/s one direction", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
