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
        a = sdpa_ref(q, k, vv).transpose(0, 1).reshape(T, v.d)
        x = x + a @ _f(L["o_w"]).t() + _f(L["o_b"])
        h = F.layer_norm(x, (v.d,), _f(L["ln2_w"]), _f(L["ln2_b"]), v.eps)
        m = _act(v.act, h @ _f(L["fc1_w"]).t() + _f(L["fc1_b"]))
        x = x + m @ _f(L["fc2_w"]).t() + _f(L["fc2_b"])
    y = F.gelu(x @ _f(Wv["p1_w"]).t() + _f(Wv["p1_b"]))
    y = y @ _f(Wv["p2_w"]).t() + _f(Wv["p2_b"])
    return y[1:] if v.cls else y


def sdpa_ref(q, k, v, causal: bool = False, chunk: int = 1024):
    """softmax(q k^T / sqrt(hd)) v in fp32, q [H, Nq, hd], k / v [H, Nk, hd];
    causal: query i sits at key position Nk - Nq + i.  Queries are processed
    in chunks so full-size sequences (29 640-patch ViT, 16k-token prefills)
    fit in memory; each query row's math is the plain formula."""
    H, Nq, hd = q.shape
    Nk = k.shape[1]
    out = torch.empty(H, Nq, v.shape[2], device=q.device, dtype=torch.float32)
    scale = 1.0 / math.sqrt(hd)
    kt = k.transpose(1, 2)
    for a in range(0, Nq, chunk):
        b = min(Nq, a + chunk)
        s = (q[:, a:b] @ kt) * scale
        if causal:
            qpos = torch.arange(Nk - Nq + a, Nk - Nq + b, device=q.device)
            kpos = torch.arange(Nk, device=q.device)
            s = s.masked_fill(kpos[None, None, :] > qpos[None, :, None], float("-inf"))
        out[:, a:b] = torch.softmax(s, -1) @ v
    return out


def _near_square(n):
    a = 1
    for i in range(1, int(math.isqrt(n)) + 1):
        if n % i == 0:
            a = i
    return a, n // a


def _rounder(round_bf16: bool):
    """Identity, or rounding to bf16 (kept in fp32) at the points where a
    bf16-storage implementation stores its activations: the "bf16 emulation"
    that separates the format's own drift from kernel error at full depth."""
    return (lambda t: t.bfloat16().float()) if round_bf16 else (lambda t: t)


def qwen_vit_ref(shape, Wv: dict, pixels_hwc: torch.Tensor, grid,
                 round_bf16: bool = False) -> torch.Tensor:
    """Qwen2.5-VL vision tower + merger, one image, fp32, in the processor's
    natural (raster) order: window attention is a per-window loop, not a
    permutation.  Returns [merged tokens in raster order, d_decoder].
    round_bf16: the same math with activations rounded to bf16 wherever the
    product stores them (GEMM outputs, residual stream, attention output)."""
    r = _rounder(round_bf16)
    v = shape.vision
    gh, gw = grid
    P, T, m = v.patch, v.temporal, v.merge
    x = pixels_hwc.float() / 255.0
    x = (x - torch.tensor(v.mean, device=x.device)) / torch.tensor(v.std, device=x.device)
    x = x.view(gh, P, gw, P, 3).permute(0, 2, 4, 1, 3)            # gh, gw, c, ky, kx
    x = x[:, :, :, None].expand(gh, gw, 3, T, P, P)               # still image: T equal frames
    x = r(r(x.reshape(gh * gw, 3 * T * P * P)) @ _f(Wv["patch_w"])[:, : v.k_in].t())
    py = torch.arange(gh, device=x.device).repeat_interleave(gw)
    px = torch.arange(gw, device=x.device).repeat(gh)
    hd, H, N = v.head_dim, v.heads, gh * gw
    half, quarter = hd // 2, hd // 4
    inv = v.rope_theta ** (-torch.arange(quarter, device=x.device, dtype=torch.float64) * 2 / half)
    ang = torch.cat([py.double()[:, None] * inv, px.double()[:, None] * inv], 1)  # [N, half]
    cos, sin = ang.cos().float()[:, None], ang.sin().float()[:, None]

    def rot(t):
        t = t.view(N, H, hd)
        a, b = t[..., :half], t[..., half:]
        return torch.cat([a * cos - b * sin, b * cos + a * sin], -1)
    ws = v.window // m
    nww = (gw // m + ws - 1) // ws
    wid = (py // m // ws) * nww + (px // m // ws)
    groups = [torch.nonzero(wid == g).flatten() for g in torch.unique(wid)]
    for li, L in enumerate(Wv["layers"]):
        h = _rms(x, _f(L["in_w"]), v.eps)
        qkv = h @ _f(L["qkv_w"]).t() + _f(L["qkv_b"])
        q, k, vv = qkv.split(v.d, 1)
        q, k, vv = r(rot(q)), r(rot(k)), r(vv.reshape(N, H, hd))
        a = torch.empty(N, H, hd, device=x.device)
        for idx in ([torch.arange(N, device=x.device)] if li in v.full_layers else groups):
            Q, K, V = q[idx].transpose(0, 1), k[idx].transpose(0, 1), vv[idx].transpose(0, 1)
            a[idx] = sdpa_ref(Q, K, V).transpose(0, 1)
        x = r(x + r(a.reshape(N, v.d)) @ _f(L["o_w"]).t() + _f(L["o_b"]))
        h = _rms(x, _f(L["post_w"]), v.eps)
        g_w, u_w = deinterleave(_f(L["gu_w"]))
        g_b, u_b = deinterleave(_f(L["gu_b"])[:, None])
        mm = r(F.silu(h @ g_w.t() + g_b[:, 0]) * (h @ u_w.t() + u_b[:, 0]))
        x = r(x + mm @ _f(L["down_w"]).t() + _f(L["down_b"]))
    h = r(_rms(x, _f(Wv["lnq_w"]), v.eps)).view(gh // m, m, gw // m, m, v.d)
    h = h.permute(0, 2, 1, 3, 4).reshape(N // (m * m), m * m * v.d)   # 2x2 units, raster
    y = r(F.gelu(h @ _f(Wv["p1_w"]).t() + _f(Wv["p1_b"])))
    return r(y @ _f(Wv["p2_w"]).t() + _f(Wv["p2_b"]))


def mrope_positions_ref(symbols):
    """Qwen2-VL get_rope_index for one unified sequence: symbols is a list of
    ("img", token_count) / ("txt", 1).  Returns [N, 3] (t, h, w) int64."""
    out, p = [], 0
    for kind, n in symbols:
        if kind == "img":
            mh, mw = _near_square(n)
            for i in range(n):
                out.append((p, p + i // mw, p + i % mw))
            p += max(mh, mw)
        else:
            for _ in range(n):
                out.append((p, p, p))
                p += 1
    return torch.tensor(out, dtype=torch.int64)


def _rope_m(x, pos3, theta, sections):
    """M-RoPE: rotary pair i rotates by component c(i) of the (t, h, w)
    position, sections = pairs per component."""
    hd = x.shape[-1]
    half = hd // 2
    inv = theta ** (-torch.arange(0, half, device=x.device, dtype=torch.float64) * 2 / hd)
    comp = torch.cat([torch.full((n,), c, dtype=torch.long) for c, n in enumerate(sections)])
    p = pos3.to(x.device).double()[:, comp.to(x.device)]                    # [N, half]
    ang = p * inv[None, :]
    cos, sin = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * cos - b * sin, b * cos + a * sin], -1)


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


def cross_layer_ref(d, L: dict, x: torch.Tensor, img: torch.Tensor):
    """One Mllama cross-attention decoder layer in fp32 (transformers
    MllamaCrossAttentionDecoderLayer.forward / MllamaTextCrossAttention, with
    the weight folds of paper_2507_10069_b200.weights.fold_cross_layer):
    x [N, d] text hidden, img [M, d] the request's image states (projector
    output).  Every text row attends to every image row (the reference's
    unified sequence puts images first).  Returns (x_out, k [M, kv_dim],
    v [M, kv_dim])."""
    N, M = x.shape[0], img.shape[0]
    g = d.hq // d.hkv
    h = _rms(x, _f(L["in_w"]), d.eps)
    q = (h @ _f(L["xq_w"]).t()).view(N, d.hq, d.hd)
    q = _rms(q, _f(L["xq_norm"]), d.eps)
    k = (img @ _f(L["xk_w"]).t()).view(M, d.hkv, d.hd)
    k = _rms(k, 1.0, d.eps)
    v = (img @ _f(L["xv_w"]).t()).view(M, d.hkv, d.hd)
    kk = k.repeat_interleave(g, 1).transpose(0, 1)
    vv = v.repeat_interleave(g, 1).transpose(0, 1)
    s = q.transpose(0, 1) @ kk.transpose(1, 2) / math.sqrt(d.hd)
    a = (torch.softmax(s, -1) @ vv).transpose(0, 1).reshape(N, d.q_dim)
    x = x + a @ _f(L["xo_w"]).t()
    h = _rms(x, _f(L["post_w"]), d.eps)
    gate, up = deinterleave(_f(L["gu_w"]))
    x = x + (F.silu(h @ gate.t()) * (h @ up.t())) @ _f(L["down_w"]).t()
    return x, k.reshape(M, d.kv_dim), v.reshape(M, d.kv_dim)


def decoder_ref(shape, Wd: dict, x: torch.Tensor, layers=None, pos3=None, img=None,
                past=None, round_bf16: bool = False):
    """Causal prefill of ONE request.

    x: [N, d] fp32 input embeddings of the rows to compute; pos3: [P + N, 3]
    M-RoPE positions of the whole sequence (shapes with mrope_section), else
    1-D positions.  past: None (recompute every position from scratch, the
    parity oracle), or (k_list, v_list) of the first P positions (the CPU
    port reusing a cached prefix: x then holds only the N suffix rows, which
    sit at positions P..P+N-1).  Cross-attention shapes (Llama-3.2-Vision,
    no past): x holds the TEXT tokens only and img [M, d] the request's
    image states (None: a text-only request, whose rows skip the cross
    layers, as Mllama's full_text_row_masked_out_mask does); the returned
    k / v lists then hold the self layers' text K/V followed by the cross
    layers' image K/V.  Returns (k_list, v_list) over all P + N positions,
    the final hidden [d] of the last token (normed) and its logits [vocab].
    round_bf16: activations rounded to bf16 where the product stores them
    (the bf16-format baseline of the full-depth tests; self layers only)."""
    d = shape.decoder
    r = _rounder(round_bf16)
    N = x.shape[0]
    P = 0 if past is None else past[0][0].shape[0]
    assert past is None or img is None, "past KV with cross-attention is not supported"
    pos = torch.arange(P, P + N, device=x.device)
    if d.mrope_section:
        assert pos3 is not None, "M-RoPE shape needs (t, h, w) positions"
        p3 = pos3[P:P + N]
        rope = lambda t: _rope_m(t, p3, d.rope_theta, d.mrope_section)
    else:
        rope = lambda t: _rope(t, pos, d.rope_theta)
    ks, vs = [], []
    g = d.hq // d.hkv
    xks, xvs = [], []
    si = 0
    for li, L in enumerate(Wd["layers"]):
        if layers is not None and li >= layers:
            break
        if L.get("cross"):
            if img is not None:
                x, kx, vx = cross_layer_ref(d, L, x, img)
                xks.append(kx)
                xvs.append(vx)
            continue
        h = _rms(x, _f(L["in_w"]), d.eps)
        qkv = h @ _f(L["qkv_w"]).t()
        if L["qkv_b"] is not None:
            qkv = qkv + _f(L["qkv_b"])
        q, k, v = qkv.split([d.q_dim, d.kv_dim, d.kv_dim], dim=1)
        q = r(rope(q.view(N, d.hq, d.hd)))
        k = r(rope(k.view(N, d.hkv, d.hd)).reshape(N, d.kv_dim))
        v = r(v.reshape(N, d.kv_dim))
        if past is not None:
            k = torch.cat([past[0][si], k], 0)
            v = torch.cat([past[1][si], v], 0)
        si += 1
        ks.append(k)
        vs.append(v)
        T = P + N
        kk = k.view(T, d.hkv, d.hd).repeat_interleave(g, 1).transpose(0, 1)
        vv = v.view(T, d.hkv, d.hd).repeat_interleave(g, 1).transpose(0, 1)
        a = sdpa_ref(q.transpose(0, 1), kk, vv, causal=True).transpose(0, 1).reshape(N, d.q_dim)
        x = r(x + r(a) @ _f(L["o_w"]).t())
        h = _rms(x, _f(L["post_w"]), d.eps)
        gate, up = deinterleave(_f(L["gu_w"]))
        m = r(F.silu(h @ gate.t()) * (h @ up.t()))
        x = r(x + m @ _f(L["down_w"]).t())
    hl = _rms(x[-1], _f(Wd["final_w"]), d.eps)
    logits = hl @ _f(Wd["lm_head"]).t()
    return ks + xks, vs + xvs, hl, logits


# ------------------------------------------------------------ CPU weights
def interleave(gate: torch.Tensor, up: torch.Tensor, block: int = 128) -> torch.Tensor:
    """Inverse of deinterleave: gate / up rows interleaved per `block`."""
    k = gate.shape[1]
    return torch.stack([gate.reshape(-1, block, k), up.reshape(-1, block, k)], 1).reshape(-1, k)


def random_weights_f32(shape, seed: int = 0, vit_layers=None, dec_layers=None,
                       vocab=None) -> tuple[dict, dict]:
    """fp32 CPU weights in the layout the refs above read (N(0, 0.02), norm
    weights 1, gate/up interleaved per 128 rows), for the CPU port timed by
    bench.py's cpu_baseline / --impl reference legs.  Not the product's
    weights (those live on the GPU, weights.py); same shapes and layout."""
    g = torch.Generator().manual_seed(seed)
    n = lambda *s: torch.randn(*s, generator=g) * 0.02
    v, d = shape.vision, shape.decoder
    Wv: dict = {}
    vl = v.layers if vit_layers is None else vit_layers
    pw = torch.zeros(v.d, v.k_pad)
    pw[:, :v.k_in] = n(v.d, v.k_in)
    Wv["patch_w"] = pw
    layers = []
    for _ in range(vl):
        if v.arch == "qwen":
            gate, up = n(v.d_ff_pad, v.d), n(v.d_ff_pad, v.d)
            gb, ub = n(v.d_ff_pad), n(v.d_ff_pad)
            layers.append({"in_w": torch.ones(v.d), "qkv_w": n(3 * v.d, v.d),
                           "qkv_b": n(3 * v.d), "o_w": n(v.d, v.d), "o_b": n(v.d),
                           "post_w": torch.ones(v.d), "gu_w": interleave(gate, up),
                           "gu_b": interleave(gb[:, None], ub[:, None])[:, 0],
                           "down_w": n(v.d, v.d_ff_pad), "down_b": n(v.d)})
        else:
            layers.append({"ln1_w": torch.ones(v.d), "ln1_b": torch.zeros(v.d),
                           "qkv_w": n(3 * v.d, v.d), "qkv_b": n(3 * v.d), "o_w": n(v.d, v.d),
                           "o_b": n(v.d), "ln2_w": torch.ones(v.d), "ln2_b": torch.zeros(v.d),
                           "fc1_w": n(v.d_ff, v.d), "fc1_b": n(v.d_ff),
                           "fc2_w": n(v.d, v.d_ff), "fc2_b": n(v.d)})
    Wv["layers"] = layers
    if v.arch == "qwen":
        Wv["lnq_w"] = torch.ones(v.d)
        Wv["p1_w"] = n(shape.proj_hidden, v.merged_dim)
    else:
        Wv["cls"] = n(v.d) if v.cls else None
        Wv["pos"] = n(v.max_pos, v.d)
        if v.pre_norm:
            Wv["pre_w"], Wv["pre_b"] = torch.ones(v.d), torch.zeros(v.d)
        Wv["p1_w"] = n(shape.proj_hidden, v.d)
    Wv["p1_b"] = n(shape.proj_hidden)
    Wv["p2_w"] = n(d.d, shape.proj_hidden)
    Wv["p2_b"] = n(d.d)
    V = d.vocab if vocab is None else vocab
    Wd: dict = {"embed": n(V, d.d)}
    dl = d.layers if dec_layers is None else dec_layers
    dls = []
    for _ in range(dl):
        gate, up = n(d.d_ff_pad, d.d), n(d.d_ff_pad, d.d)
        dls.append({"in_w": torch.ones(d.d), "qkv_w": n(d.q_dim + 2 * d.kv_dim, d.d),
                    "qkv_b": n(d.q_dim + 2 * d.kv_dim) if d.qkv_bias else None,
                    "o_w": n(d.d, d.q_dim), "post_w": torch.ones(d.d),
                    "gu_w": interleave(gate, up), "down_w": n(d.d, d.d_ff_pad)})
    Wd["layers"] = dls
    Wd["final_w"] = torch.ones(d.d)
    Wd["lm_head"] = n(V, d.d)
    return Wv, Wd
