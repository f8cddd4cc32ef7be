"""Where does bf16 error vs the fp32 oracle come from at full depth?

Per layer, for one C3 request (28-layer Qwen2-7B decoder) and one 7 410-token
image (32-layer Qwen2.5-VL ViT), three numbers:
  product  vs fp32 oracle     (what tests/test_fullshape_gpu.py checks)
  bf16-emu vs fp32 oracle     (the oracle's math with activations rounded to
                               bf16 wherever the product stores bf16: GEMM
                               outputs, residual stream, attention output —
                               i.e. ANY bf16-storage implementation)
  product  vs bf16-emu
If product ~ bf16-emu error, the drift is the format, not a kernel bug.
Writes gpurun_out/depth_error.json.  GPU box: python tools/depth_error_probe.py
"""
import json
import math
import os
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import model_ref as M  # noqa: E402

rb = lambda t: t.bfloat16().float()  # noqa: E731


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm()).item()


def decoder_layers(shape, Wd, x, pos3, emulate):
    """decoder_ref's math, returning per-layer (k, v, x_out)."""
    d = shape.decoder
    N = x.shape[0]
    rope = lambda t: M._rope_m(t, pos3, d.rope_theta, d.mrope_section)  # noqa: E731
    g = d.hq // d.hkv
    r = rb if emulate else (lambda t: t)
    x = r(x)
    out = []
    for L in Wd["layers"]:
        h = M._rms(x, M._f(L["in_w"]), d.eps)
        qkv = h @ M._f(L["qkv_w"]).t()
        if L["qkv_b"] is not None:
            qkv = qkv + M._f(L["qkv_b"])
        q, k, v = qkv.split([d.q_dim, d.kv_dim, d.kv_dim], dim=1)
        q = r(rope(q.view(N, d.hq, d.hd)))
        k = r(rope(k.view(N, d.hkv, d.hd)))
        v = r(v.view(N, d.hkv, d.hd))
        kk = k.repeat_interleave(g, 1).transpose(0, 1)
        vv = v.repeat_interleave(g, 1).transpose(0, 1)
        a = r(M.sdpa_ref(q.transpose(0, 1), kk, vv, causal=True).transpose(0, 1)
              .reshape(N, d.q_dim))
        x = r(x + a @ M._f(L["o_w"]).t())
        h = M._rms(x, M._f(L["post_w"]), d.eps)
        gate, up = M.deinterleave(M._f(L["gu_w"]))
        m = r(F.silu(h @ gate.t()) * (h @ up.t()))
        x = r(x + m @ M._f(L["down_w"]).t())
        out.append((k.reshape(N, -1), v.reshape(N, -1), x))
    return out


def main():
    from goldens import trace_path
    from paper_2507_10069_b200 import shapes
    from paper_2507_10069_b200.keys import TAG_IMG, request_keys
    from paper_2507_10069_b200.pipeline import HotPath
    from paper_2507_10069_b200.workload import read_trace
    shape = shapes.SHAPES["qwen-7b"]
    hp = HotPath(shape, budget_tokens=600_000)
    reqs = read_trace(trace_path("c3"))
    # one multimodal request and one text request, computed from scratch
    picks = [next(r for r in reqs if r.images), reqs[0]]
    res = {"decoder": {}, "vit": {}}
    for req in picks:
        imgs = list({i.content_hash: i for i in req.images}.values())
        if imgs:
            hp.encode(imgs)
        r = hp.prefill([req], [0])
        torch.cuda.synchronize()
        N = req.total_input_len
        kv = r.kv.req_kv[:, :, :N]
        keys, w = request_keys(hp.codec, req)
        rows = []
        for k, ww in zip(keys, w):
            if int(k) >> 62 == TAG_IMG:
                rows.append(hp.slabs[hp.codec.symbol(int(k))[1]].float())
            else:
                rows.append(hp.Wd["embed"][int(k) % shape.decoder.vocab].float()[None])
        x = torch.cat(rows, 0)
        syms = [("img", int(ww)) if int(k) >> 62 == TAG_IMG else ("txt", 1)
                for k, ww in zip(keys, w)]
        pos3 = M.mrope_positions_ref(syms).cuda()
        with torch.no_grad():
            f32 = decoder_layers(shape, hp.Wd, x, pos3, False)
            emu = decoder_layers(shape, hp.Wd, x, pos3, True)
        rows_out = []
        for li in range(len(f32)):
            rows_out.append({
                "layer": li,
                "K_product_vs_f32": rel(kv[li, 0], f32[li][0]),
                "K_emu_vs_f32": rel(emu[li][0], f32[li][0]),
                "K_product_vs_emu": rel(kv[li, 0], emu[li][0]),
                "V_product_vs_f32": rel(kv[li, 1], f32[li][1]),
                "V_emu_vs_f32": rel(emu[li][1], f32[li][1]),
                "x_emu_vs_f32": rel(emu[li][2], f32[li][2]),
            })
        allk = lambda src: torch.stack([t[0] for t in src])  # noqa: E731
        res["decoder"][f"req{req.id}_N{N}"] = {
            "per_layer": rows_out,
            "K_all_layers_product_vs_f32": rel(kv[:, 0], allk(f32)),
            "K_all_layers_emu_vs_f32": rel(allk(emu), allk(f32)),
        }
        hp.release_batch_kv()
    with open(os.path.join(ROOT, "gpurun_out", "depth_error.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    for k, v in res["decoder"].items():
        print(k, "all-layer K: product", round(v["K_all_layers_product_vs_f32"], 5),
              "bf16-emu", round(v["K_all_layers_emu_vs_f32"], 5))
        for row in v["per_layer"][::3]:
            print("  ", {a: (round(b, 5) if isinstance(b, float) else b) for a, b in row.items()})


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    main()
    print(math.pi if False else "done")
