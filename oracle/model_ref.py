"""fp32 numerics oracle — TEST INFRASTRUCTURE ONLY.

The reference has no encoder / prefill numerics at all: encode and prefill
are analytic durations (pkg/src/mmsim/costmodel.py:102-119),
so numeric parity is "builder-pinned": this is a straight-line fp32 torch
restatement of the public architectures in paper_2507_10069_b200/shapes.py
(CLIP-style pre-LN ViT + 2-layer GELU projector; Llama-style RMSNorm / RoPE
rotate-half / GQA / SwiGLU decoder), written with plain torch ops and NO
cached prefix: the decoder recomputes every position from scratch, so the
product's prefix-cached prefill is checked against full recompute.

Runs on CPU (bench cpu_baseline / --impl reference) or on a GPU in fp32
(the "plain PyTorch fp32 reference" of the numerics tests).
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def _f(t):
    return None if t is None else t.float()


def _act(name, x):
    if name == "quick_gelu":
        return x * torch.sigmoid(1.702 * x)
    if name == "gelu_tanh":
        return F.gelu(x, approximate="tanh")
    return F.gelu(x)


def patchify_ref(pixels_hwc: torch.Tensor, gh: int, gw: int, P: int, mean, std) -> torch.Tensor:
    x = pixels_hwc.float() / 255.0
    x = (x - torch.tensor(mean, device=x.device)) / torch.tensor(std, device=x.device)
    x = x.view(gh, P, gw, P, 3).permute(0, 2, 4, 1, 3)  # gh, gw, c, ky, kx
    return x.reshape(gh * gw, 3 * P * P)


def vit_ref(shape, Wv: dict, pixels_hwc: torch.Tensor, grid) -> torch.Tensor:
    """One image -> [n_patches, d_decoder] fp32 (CLS dropped)."""
    v = shape.vision
    gh, gw = grid
    n = gh * gw
    p = patchify_ref(pixels_hwc, gh, gw, v.patch, v.mean, v.std)
    x = p @ _f(Wv["patch_w"])[:, : v.k_in].t()
    if v.cls:
        x = torch.cat([_f(Wv["cls"])[None], x], 0)
    x = x + _f(Wv["pos"])[: x.shape[0]]
    if v.pre_norm:
        x = F.layer_norm(x, (v.d,), _f(Wv["pre_w"]), _f(Wv["pre_b"]), v.eps)
    T, H, hd = x.shape[0], v.heads, v.head_dim
    for L in Wv["layers"]:
        h = F.layer_norm(x, (v.d,), _f(L["ln1_w"]), _f(L["ln1_b"]), v.eps)
        qkv = h @ _f(L["qkv_w"]).t() + _f(L["qkv_b"])
        q, k, vv = qkv.split(v.d, dim=1)
        q = q.view(T, H, hd).transpose(0, 1)
        k = k.view(T, H, hd).transpose(0, 1)
        vv = vv.view(T, H, hd).transpose(0, 1)
        a = torch.softmax(q @ k.transpose(1, 2) / math.sqrt(hd), -1) @ vv
        a = a.transpose(0, 1).reshape(T, v.d)
        x = x + a @ _f(L["o_w"]).t() + _f(L["o_b"])
        h = F.layer_norm(x, (v.d,), _f(L["ln2_w"]), _f(L["ln2_b"]), v.eps)
        m = _act(v.act, h @ _f(L["fc1_w"]).t() + _f(L["fc1_b"]))
        x = x + m @ _f(L["fc2_w"]).t() + _f(L["fc2_b"])
    y = F.gelu(x @ _f(Wv["p1_w"]).t() + _f(Wv["p1_b"]))
    y = y @ _f(Wv["p2_w"]).t() + _f(Wv["p2_b"])
    return y[1:] if v.cls else y


def _rms(x, w, eps):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


def _rope(x, pos, theta):
    # x: [T, H, hd]; rotate-half convention
    hd = x.shape[-1]
    inv = theta ** (-torch.arange(0, hd // 2, device=x.device, dtype=torch.float64) * 2 / hd)
    ang = pos.double()[:, None] * inv[None, :]
    cos, sin = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]
    a, b = x[..., : hd // 2], x[..., hd // 2:]
    return torch.cat([a * cos - b * sin, b * cos + a * sin], -1)


def deinterleave(w, block=128):
    two_i, k = w.shape
    x = w.reshape(two_i // (2 * block), 2, block, k)
    return x[:, 0].reshape(-1, k), x[:, 1].reshape(-1, k)


def decoder_ref(shape, Wd: dict, x: torch.Tensor, layers=None):
    """Full-sequence causal prefill of ONE request from scratch.

    x: [N, d] fp32 input embeddings.  Returns (k_list, v_list, final_hidden
    [d] of the last token (normed), logits [vocab] of the last token)."""
    d = shape.decoder
    N = x.shape[0]
    pos = torch.arange(N, device=x.device)
    mask = torch.ones(N, N, device=x.device, dtype=torch.bool).tril()
    ks, vs = [], []
    g = d.hq // d.hkv
    for li, L in enumerate(Wd["layers"]):
        if layers is not None and li >= layers:
            break
        h = _rms(x, _f(L["in_w"]), d.eps)
        qkv = h @ _f(L["qkv_w"]).t()
        if L["qkv_b"] is not None:
            qkv = qkv + _f(L["qkv_b"])
        q, k, v = qkv.split([d.q_dim, d.kv_dim, d.kv_dim], dim=1)
        q = _rope(q.view(N, d.hq, d.hd), pos, d.rope_theta)
        k = _rope(k.view(N, d.hkv, d.hd), pos, d.rope_theta)
        v = v.view(N, d.hkv, d.hd)
        ks.append(k.reshape(N, d.kv_dim))
        vs.append(v.reshape(N, d.kv_dim))
        kk = k.repeat_interleave(g, 1).transpose(0, 1)
        vv = v.repeat_interleave(g, 1).transpose(0, 1)
        s = q.transpose(0, 1) @ kk.transpose(1, 2) / math.sqrt(d.hd)
        s = s.masked_fill(~mask, float("-inf"))
        a = (torch.softmax(s, -1) @ vv).transpose(0, 1).reshape(N, d.q_dim)
        x = x + a @ _f(L["o_w"]).t()
        h = _rms(x, _f(L["post_w"]), d.eps)
        gate, up = deinterleave(_f(L["gu_w"]))
        m = F.silu(h @ gate.t()) * (h @ up.t())
        x = x + m @ _f(L["down_w"]).t()
    hl = _rms(x[-1], _f(Wd["final_w"]), d.eps)
    logits = hl @ _f(Wd["lm_head"]).t()
    return ks, vs, hl, logits
