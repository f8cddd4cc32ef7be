"""Qwen2.5-VL vision tower: the fp32 oracle (oracle/model_ref.qwen_vit_ref)
is pinned against the public implementation (transformers'
Qwen2_5_VisionTransformerPretrainedModel, run here on CPU with the same
weights), and the product's window token order (encoder.window_plan) against
that model's own get_window_index.  The multimodal RoPE positions of the
prefill (prefill.mrope_positions) are checked against the oracle's
restatement of get_rope_index."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import model_ref

hf = pytest.importorskip("transformers.models.qwen2_5_vl.modeling_qwen2_5_vl")


def _tiny_shape():
    from paper_2507_10069_b200 import shapes
    v = dataclasses.replace(shapes.QWEN_VISION, layers=4, d=160, heads=2, d_ff=340,
                            full_layers=(1, 3))
    dec = dataclasses.replace(shapes.QWEN_VL_7B.decoder, d=256)
    return dataclasses.replace(shapes.QWEN_VL_7B, vision=v, proj_hidden=v.merged_dim,
                               decoder=dec)


def _hf_model(shape):
    from transformers.models.qwen2_5_vl.configuration_qwen2_5_vl import Qwen2_5_VLVisionConfig
    v = shape.vision
    cfg = Qwen2_5_VLVisionConfig(depth=v.layers, hidden_size=v.d, num_heads=v.heads,
                                 intermediate_size=v.d_ff, out_hidden_size=shape.decoder.d,
                                 patch_size=v.patch, temporal_patch_size=v.temporal,
                                 spatial_merge_size=v.merge, window_size=v.window * v.patch,
                                 fullatt_block_indexes=list(v.full_layers), hidden_act="silu")
    cfg._attn_implementation = "eager"
    return hf.Qwen2_5_VisionTransformerPretrainedModel(cfg).eval()


def _load(model, shape, W):
    from paper_2507_10069_b200.weights import deinterleave_glu
    v = shape.vision
    f = lambda t: t.float()
    with torch.no_grad():
        model.patch_embed.proj.weight.copy_(
            f(W["patch_w"][:, : v.k_in]).view(v.d, 3, v.temporal, v.patch, v.patch))
        for blk, L in zip(model.blocks, W["layers"]):
            blk.norm1.weight.copy_(f(L["in_w"]))
            blk.norm2.weight.copy_(f(L["post_w"]))
            blk.attn.qkv.weight.copy_(f(L["qkv_w"]))
            blk.attn.qkv.bias.copy_(f(L["qkv_b"]))
            blk.attn.proj.weight.copy_(f(L["o_w"]))
            blk.attn.proj.bias.copy_(f(L["o_b"]))
            g, u = deinterleave_glu(L["gu_w"])
            gb, ub = deinterleave_glu(L["gu_b"][:, None])
            blk.mlp.gate_proj.weight.copy_(f(g[: v.d_ff]))
            blk.mlp.up_proj.weight.copy_(f(u[: v.d_ff]))
            blk.mlp.gate_proj.bias.copy_(f(gb[: v.d_ff, 0]))
            blk.mlp.up_proj.bias.copy_(f(ub[: v.d_ff, 0]))
            blk.mlp.down_proj.weight.copy_(f(L["down_w"][:, : v.d_ff]))
            blk.mlp.down_proj.bias.copy_(f(L["down_b"]))
        model.merger.ln_q.weight.copy_(f(W["lnq_w"]))
        model.merger.mlp[0].weight.copy_(f(W["p1_w"]))
        model.merger.mlp[0].bias.copy_(f(W["p1_b"]))
        model.merger.mlp[2].weight.copy_(f(W["p2_w"]))
        model.merger.mlp[2].bias.copy_(f(W["p2_b"]))


def _processor_order(patches, gh, gw, m):
    """Raster patch rows -> Qwen2-VL image-processor order (2x2 units)."""
    K = patches.shape[-1]
    return patches.view(gh // m, m, gw // m, m, K).permute(0, 2, 1, 3, 4).reshape(gh * gw, K)


@pytest.mark.parametrize("grid", [(4, 4), (8, 8), (10, 24), (18, 14), (22, 38)])
def test_window_plan_matches_hf_window_index(grid):
    from paper_2507_10069_b200.encoder import window_plan
    shape = _tiny_shape()
    v = shape.vision
    model = _hf_model(dataclasses.replace(shape, vision=dataclasses.replace(v, layers=1)))
    gh, gw = grid
    win_idx, cu = model.get_window_index(torch.tensor([[1, gh, gw]]))
    win_idx = torch.as_tensor(win_idx).numpy()
    m = v.merge
    mw = gw // m
    ur, uc = np.divmod(win_idx, mw)
    dy, dx = np.divmod(np.arange(m * m), m)
    want = ((ur[:, None] * m + dy) * gw + (uc[:, None] * m + dx)).reshape(-1)
    plan = window_plan(gh, gw, m, v.window)
    assert np.array_equal(plan["row_patch"], want)
    cu = np.unique(np.asarray(cu))
    assert np.array_equal(plan["window_lens"], np.diff(cu))
    # merger gather: raster unit u -> its rows in window order
    rows = plan["unit_rows"].reshape(-1, m * m)
    assert np.array_equal(plan["row_patch"][rows[:, 0]] // gw // m * mw
                          + plan["row_patch"][rows[:, 0]] % gw // m, np.arange((gh // m) * mw))


def test_oracle_qwen_vit_matches_transformers():
    from paper_2507_10069_b200.weights import init_vision
    shape = _tiny_shape()
    v = shape.vision
    W = init_vision(shape, seed=3, device="cpu")
    gh, gw = 10, 18
    px = torch.from_numpy(np.random.default_rng(5).integers(0, 256, (gh * v.patch, gw * v.patch, 3),
                                                            dtype=np.uint8))
    ours = model_ref.qwen_vit_ref(shape, W, px, (gh, gw))
    model = _hf_model(shape)
    _load(model, shape, W)
    x = px.float() / 255.0
    x = (x - torch.tensor(v.mean)) / torch.tensor(v.std)
    x = x.view(gh, v.patch, gw, v.patch, 3).permute(0, 2, 4, 1, 3)
    x = x[:, :, :, None].expand(gh, gw, 3, v.temporal, v.patch, v.patch).reshape(gh * gw, -1)
    with torch.no_grad():
        theirs = model(_processor_order(x, gh, gw, v.merge), torch.tensor([[1, gh, gw]]))
    theirs = theirs.pooler_output
    assert theirs.shape == ours.shape == ((gh // 2) * (gw // 2), shape.decoder.d)
    err = ((ours - theirs).norm() / theirs.norm()).item()
    assert err < 1e-4, err


def test_mrope_positions_match_oracle():
    from paper_2507_10069_b200.keys import request_keys
    from paper_2507_10069_b200.cache import DEFAULT_CODEC
    from paper_2507_10069_b200.prefill import mrope_positions
    from paper_2507_10069_b200.workload import ImageInput, Request
    A, B = ImageInput("a" * 32, 6516, (0, 0)), ImageInput("b" * 32, 7410, (0, 0))
    C = ImageInput("c" * 32, 576, (0, 0))
    for req in (Request(0, 0.0, "multimodal", 30, (A,), 4, prefix_id=1, prefix_len=10),
                Request(1, 0.0, "multimodal", 7, (B, C, A), 4),
                Request(2, 0.0, "text", 50, (), 4, prefix_id=2, prefix_len=20)):
        keys, w = request_keys(DEFAULT_CODEC, req)
        pt, ph, pw = mrope_positions(keys, w)
        syms = [("img", img.token_count) for img in req.images]
        syms += [("txt", 1)] * (req.total_input_len - sum(i.token_count for i in req.images))
        ref = model_ref.mrope_positions_ref(syms).numpy()
        assert np.array_equal(np.stack([pt, ph, pw], 1), ref)
