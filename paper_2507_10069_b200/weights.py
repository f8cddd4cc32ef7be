"""Random-init bf16 weights of the model shapes (shapes.py), generated on the
device from a fixed seed (no checkpoints exist offline; SURVEY.md §8d:
torch.Generator seed 0, N(0, 0.02)).  Layouts are the kernels' layouts:
linear weights [out, in] (K-major B operand), gate/up interleaved per 128
rows for the fused SwiGLU epilogue, patch weights zero-padded to k_pad.
"""
from __future__ import annotations

import torch

from .ops import interleave_glu, interleave_glu_bias
from .shapes import ModelShape


def _n(gen, *shape, std=0.02, device="cuda"):
    return (torch.randn(*shape, generator=gen, device=device) * std).to(torch.bfloat16)


def _ones(gen, n, device="cuda"):
    return (1.0 + torch.randn(n, generator=gen, device=device) * 0.02).to(torch.bfloat16)


def init_vision(shape: ModelShape, seed: int = 0, device="cuda") -> dict:
    v, dec = shape.vision, shape.decoder
    if v.arch == "qwen":
        return init_vision_qwen(shape, seed, device)
    g = torch.Generator(device=device).manual_seed(seed)
    W: dict = {}
    pw = torch.zeros(v.d, v.k_pad, device=device, dtype=torch.bfloat16)
    pw[:, : v.k_in] = _n(g, v.d, v.k_in, device=device)
    W["patch_w"] = pw
    W["cls"] = _n(g, v.d, device=device) if v.cls else None
    W["pos"] = _n(g, v.max_pos, v.d, device=device)
    if v.pre_norm:
        W["pre_w"], W["pre_b"] = _ones(g, v.d, device), _n(g, v.d, device=device)
    layers = []
    for _ in range(v.layers):
        L = {
            "ln1_w": _ones(g, v.d, device), "ln1_b": _n(g, v.d, device=device),
            "qkv_w": _n(g, 3 * v.d, v.d, device=device), "qkv_b": _n(g, 3 * v.d, device=device),
            "o_w": _n(g, v.d, v.d, device=device), "o_b": _n(g, v.d, device=device),
            "ln2_w": _ones(g, v.d, device), "ln2_b": _n(g, v.d, device=device),
            "fc1_w": _n(g, v.d_ff, v.d, device=device), "fc1_b": _n(g, v.d_ff, device=device),
            "fc2_w": _n(g, v.d, v.d_ff, device=device), "fc2_b": _n(g, v.d, device=device),
        }
        layers.append(L)
    W["layers"] = layers
    W["p1_w"] = _n(g, shape.proj_hidden, v.d, device=device)
    W["p1_b"] = _n(g, shape.proj_hidden, device=device)
    W["p2_w"] = _n(g, dec.d, shape.proj_hidden, device=device)
    W["p2_b"] = _n(g, dec.d, device=device)
    return W


def _padded_glu(g, ff, ff_pad, d, w_norm, device):
    """gate/up [ff_pad, d] with zero padded rows, norm weight folded in,
    biases, interleaved for the GLU epilogue; down [d, ff_pad] + bias."""
    gate = _n(g, ff_pad, d, device=device)
    up = _n(g, ff_pad, d, device=device)
    gb = _n(g, ff_pad, device=device)
    ub = _n(g, ff_pad, device=device)
    down = _n(g, d, ff_pad, device=device)
    if ff_pad != ff:  # padded features contribute exactly zero
        for t in (gate, up, gb, ub):
            t[ff:] = 0
        down[:, ff:] = 0
    gate = (gate.float() * w_norm.float()[None]).to(torch.bfloat16)
    up = (up.float() * w_norm.float()[None]).to(torch.bfloat16)
    return interleave_glu(gate, up), interleave_glu_bias(gb, ub), down


def rope_pair_perm(d: int, hd: int, device="cuda") -> torch.Tensor:
    """Row order of a fused [q | k | v] weight (3d rows) that interleaves each
    head's rotary pairs: new row 2i (2i+1) of a q or k head = old row i
    (i + hd/2); v rows keep their order."""
    half = hd // 2
    head = torch.stack([torch.arange(half), torch.arange(half) + half], 1).reshape(-1)
    qk = torch.cat([h * hd + head for h in range(2 * d // hd)])
    return torch.cat([qk, torch.arange(2 * d, 3 * d)]).to(device)


def init_vision_qwen(shape: ModelShape, seed: int = 0, device="cuda") -> dict:
    """Qwen2.5-VL vision tower.  RMSNorm weights of norm1 / norm2 are folded
    into the QKV and gate/up matrices (the GEMM epilogue applies the row
    rsqrt), so the explicit in_w / post_w are exactly 1; the merger's ln_q
    weight stays explicit (its norm kernel also gathers rows)."""
    v, dec = shape.vision, shape.decoder
    g = torch.Generator(device=device).manual_seed(seed)
    W: dict = {}
    pw = torch.zeros(v.d, v.k_pad, device=device, dtype=torch.bfloat16)
    pw[:, : v.k_in] = _n(g, v.d, v.k_in, device=device)
    W["patch_w"] = pw
    layers = []
    for _ in range(v.layers):
        n1, n2 = _ones(g, v.d, device), _ones(g, v.d, device)
        qkv = (_n(g, 3 * v.d, v.d, device=device).float() * n1.float()[None]).to(torch.bfloat16)
        gu, gub, down = _padded_glu(g, v.d_ff, v.d_ff_pad, v.d, n2, device)
        qkv_b = _n(g, 3 * v.d, device=device)
        perm = rope_pair_perm(v.d, v.head_dim, device)
        layers.append({
            "in_w": torch.ones(v.d, device=device, dtype=torch.bfloat16),
            "qkv_w": qkv, "qkv_b": qkv_b,
            # kernel copy: q / k rows of every head reordered so that rotary
            # pair (i, i + hd/2) sits in adjacent columns (the GEMM epilogue
            # applies the 2-D RoPE there); q.k is invariant under the shared
            # permutation, v is untouched
            "qkv_w_pi": qkv[perm].contiguous(), "qkv_b_pi": qkv_b[perm].contiguous(),
            "o_w": _n(g, v.d, v.d, device=device), "o_b": _n(g, v.d, device=device),
            "post_w": torch.ones(v.d, device=device, dtype=torch.bfloat16),
            "gu_w": gu, "gu_b": gub, "down_w": down, "down_b": _n(g, v.d, device=device),
        })
    W["layers"] = layers
    W["lnq_w"] = _ones(g, v.d, device)
    W["p1_w"] = _n(g, shape.proj_hidden, v.merged_dim, device=device)
    W["p1_b"] = _n(g, shape.proj_hidden, device=device)
    W["p2_w"] = _n(g, dec.d, shape.proj_hidden, device=device)
    W["p2_b"] = _n(g, dec.d, device=device)
    return W


def init_decoder(shape: ModelShape, seed: int = 1, device="cuda") -> dict:
    d = shape.decoder
    g = torch.Generator(device=device).manual_seed(seed)
    W: dict = {"embed": _n(g, d.vocab, d.d, device=device)}
    layers = []
    qkv_out = d.q_dim + 2 * d.kv_dim
    for li in range(d.layers):
        if li in d.cross:
            layers.append(fold_cross_layer(random_cross_layer(g, d, device), d))
            continue
        gate = _n(g, d.d_ff_pad, d.d, device=device)
        up = _n(g, d.d_ff_pad, d.d, device=device)
        down = _n(g, d.d, d.d_ff_pad, device=device)
        if d.d_ff_pad != d.d_ff:  # padded features contribute exactly zero
            gate[d.d_ff:] = 0
            up[d.d_ff:] = 0
            down[:, d.d_ff:] = 0
        # RMSNorm weights are folded into the following projection (qkv_w,
        # gu_w hold W * diag(w)); the explicit norm weights are exactly 1
        L = {
            "in_w": torch.ones(d.d, device=device, dtype=torch.bfloat16),
            "qkv_w": _n(g, qkv_out, d.d, device=device),
            "qkv_b": _n(g, qkv_out, device=device) if d.qkv_bias else None,
            "o_w": _n(g, d.d, d.q_dim, device=device),
            "post_w": torch.ones(d.d, device=device, dtype=torch.bfloat16),
            "gu_w": interleave_glu(gate, up),
            "down_w": down,
        }
        del gate, up
        layers.append(L)
    W["layers"] = layers
    W["final_w"] = _ones(g, d.d, device)
    W["lm_head"] = _n(g, d.vocab, d.d, device=device)
    return W


def random_cross_layer(g, d, device="cuda", dtype=torch.bfloat16) -> dict:
    """Unfolded Mllama cross-attention decoder layer (transformers'
    MllamaCrossAttentionDecoderLayer parameter set): q/k/v/o projections,
    per-head q_norm / k_norm, input / post-attention RMSNorms, SwiGLU MLP and
    the two tanh gates.  Checkpoints initialise the gates at 0 (the layer is
    then an identity); random init uses 0.5 so the path carries signal."""
    n = lambda *sh: _n(g, *sh, device=device).to(dtype)
    one = lambda k: _ones(g, k, device).to(dtype)
    gate, up, down = n(d.d_ff_pad, d.d), n(d.d_ff_pad, d.d), n(d.d, d.d_ff_pad)
    if d.d_ff_pad != d.d_ff:
        gate[d.d_ff:] = 0
        up[d.d_ff:] = 0
        down[:, d.d_ff:] = 0
    return {"q_proj": n(d.q_dim, d.d), "k_proj": n(d.kv_dim, d.d), "v_proj": n(d.kv_dim, d.d),
            "o_proj": n(d.d, d.q_dim), "q_norm": one(d.hd), "k_norm": one(d.hd),
            "in_norm": one(d.d), "post_norm": one(d.d), "gate": gate, "up": up, "down": down,
            "attn_gate": 0.5, "mlp_gate": 0.5}


def fold_cross_layer(raw: dict, d) -> dict:
    """Kernel layout of a cross-attention layer.  Exact algebraic folds:
    input / post norm weights into the q and gate/up columns (the GEMM
    epilogue applies the row rsqrt), k_norm's weight into q_norm's
    (q.k = (q*wq*wk).(k_hat)), tanh(attn_gate) into o_proj, tanh(mlp_gate)
    into down_proj.  k_norm is then weight-free, so every cross layer's K/V
    projection of an image can run as one GEMM."""
    import math
    f = lambda t: t.float()
    dt = raw["q_proj"].dtype
    ta, tm = math.tanh(raw["attn_gate"]), math.tanh(raw["mlp_gate"])
    gate = f(raw["gate"]) * f(raw["post_norm"])[None]
    up = f(raw["up"]) * f(raw["post_norm"])[None]
    return {
        "cross": True,
        "in_w": torch.ones_like(raw["in_norm"]),
        "xq_w": (f(raw["q_proj"]) * f(raw["in_norm"])[None]).to(dt),
        "xk_w": raw["k_proj"], "xv_w": raw["v_proj"],
        "xq_norm": (f(raw["q_norm"]) * f(raw["k_norm"])).to(dt),
        "xo_w": (f(raw["o_proj"]) * ta).to(dt),
        "post_w": torch.ones_like(raw["post_norm"]),
        "gu_w": interleave_glu(gate.to(dt), up.to(dt)),
        "down_w": (f(raw["down"]) * tm).to(dt),
        "attn_gate": raw["attn_gate"], "mlp_gate": raw["mlp_gate"],
    }


def deinterleave_glu(w: torch.Tensor, block: int = 128):
    """Inverse of ops.interleave_glu -> (gate, up)."""
    two_i, k = w.shape
    x = w.reshape(two_i // (2 * block), 2, block, k)
    return x[:, 0].reshape(-1, k), x[:, 1].reshape(-1, k)
