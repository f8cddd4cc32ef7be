"""Cold-L2 repeat probe for the kernels with cross-CTA or multi-phase
synchronisation: decode attention (per-request splits + merge), the
decode-size split-K GEMMs (unit counters) and the tile GEMM.  Every launch
starts with a cold L2 (a 256 MiB write), which slows the loads and widens
any ordering window (the single-tile attention race of session 5 showed up
exactly this way).  Every launch must give bytes identical to the first, and
the first must be within the parity bound against fp32.

  python tools/cold_l2_probe.py [--iters 200]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def repeat(name, fn, ref, iters, flush, rel_bound):
    first = None
    n_diff = 0
    for it in range(iters):
        flush.fill_(it & 255)
        out = fn()
        torch.cuda.synchronize()
        if first is None:
            first = out.clone()
        elif not torch.equal(out, first):
            n_diff += 1
    rel = ((first.float() - ref).norm() / ref.norm()).item()
    rec = {"kernel": name, "iters": iters, "differs_from_first": n_diff,
           "rel_err_vs_fp32": rel, "ok": n_diff == 0 and rel < rel_bound}
    print(json.dumps(rec), flush=True)
    return rec


def main(iters):
    from paper_2507_10069_b200 import ops
    from test_decode_gpu import _ref_decode
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(5)
    recs = []
    for lens in ([15000] + [17 * i % 900 + 1 for i in range(63)], [4400] * 64, [7000, 5, 4097]):
        hq, hkv, hd = 28, 4, 128
        n_slots = sum(lens) + 500
        K = torch.randn(n_slots, hkv * hd, device="cuda", generator=g).bfloat16()
        V = torch.randn(n_slots, hkv * hd, device="cuda", generator=g).bfloat16()
        bt = torch.randperm(n_slots, device="cuda", generator=g).to(torch.int32)[:sum(lens)]
        bt = bt.contiguous()
        off = [0]
        for x in lens:
            off.append(off[-1] + x)
        bt_off = torch.tensor(off, dtype=torch.int64, device="cuda")
        kv_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
        q = (torch.randn(len(lens), hq * hd, device="cuda", generator=g) * 2).bfloat16()
        ref = _ref_decode(q, K, V, bt, off, lens, hq, hkv, hd, hd ** -0.5)
        recs.append(repeat(f"decode_attention n={len(lens)} max={max(lens)}",
                           lambda: ops.decode_attention(q, K, V, bt, bt_off, kv_len, hkv, hd,
                                                        max(lens)),
                           ref, iters, flush, 1e-2))
    for M, N, K_ in ((1, 4608, 3584), (40, 3584, 3584), (64, 37888, 3584), (64, 3584, 18944),
                     (48, 3584, 18944), (4096, 4608, 3584)):
        a = torch.randn(M, K_, device="cuda", generator=g).bfloat16()
        b = (torch.randn(N, K_, device="cuda", generator=g) * K_ ** -0.5).bfloat16()
        ref = a.float() @ b.float().t()
        recs.append(repeat(f"gemm M={M} N={N} K={K_}", lambda: ops.gemm(a, b), ref, iters,
                           flush, 8e-3))
    print(json.dumps({"all_ok": all(r["ok"] for r in recs), "configs": len(recs)}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    main(ap.parse_args().iters)
