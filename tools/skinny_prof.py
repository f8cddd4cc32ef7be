"""Per-CTA timeline of one decode-size GEMM launch (csrc/gemm_skinny.cu,
EMM_SKINNY_PROF=1): %globaltimer stamps at entry, after the dependency wait,
first K stage landed, accumulator ready, partial published, all splits
arrived, epilogue done, CTA done — printed as percentiles in us from the
earliest entry.
    EMM_SKINNY_PROF=1 python tools/skinny_prof.py M N K [glu]"""
import ctypes
import os
import sys

os.environ["EMM_SKINNY_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_10069_b200 import _lib, ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
glu = len(sys.argv) > 4 and sys.argv[4] == "glu"
a = torch.randn(M, K, device="cuda").bfloat16()
ws = [(torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16() for _ in range(max(2, int(4e8 // (N * K * 2))))]
res = torch.randn(M, N // 2 if glu else N, device="cuda").bfloat16()
ss = ops.row_sumsq(a)


def run(w):
    if glu:
        ops.gemm_ex(a, w, epi=ops.EPI_GLU_SILU, row_ss_in=ss, rms_dim=K, rms_eps=1e-6)
    else:
        ops.gemm_ex(a, w, residual=res)


for w in ws:
    run(w)
torch.cuda.synchronize()
lib = _lib.lib
fn = lib.emm_skinny_prof_read
fn.restype = ctypes.c_int
for rep in range(3):
    run(ws[rep % len(ws)])
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (16 * 148))()
    assert fn(buf, 16 * 148) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(148, 16).astype(np.int64)
    live = t[:, 0] > 0
    t = t[live]
    t0 = t[:, 0].min()
    names = ["entry", "dep_wait", "stage0", "acc_ready", "published", "all_arrived", "epi_done",
             "t128_after_bar", "t0_after_bar", "t0_before_bar", "c0_tmem", "c0_done", "c1_tmem",
             "c1_done", "c2_tmem", "c2_done"]
    print(f"M={M} N={N} K={K} glu={glu} ctas={len(t)} (rep {rep})")
    for i, nm in enumerate(names):
        col = t[:, i]
        col = col[col >= t0]
        if len(col) == 0:
            continue
        q = np.percentile((col - t0) / 1e3, [0, 50, 90, 100])
        print(f"  {nm:12s} " + " ".join(f"{x:7.2f}" for x in q))
