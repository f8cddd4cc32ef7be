"""The fp32 decoder oracle (oracle/model_ref.decoder_ref) pinned against the
public implementations, run here on CPU with the same weights (VERDICT r1
weak-2: the decoder restatement was never pinned):

* Qwen2.5-VL text decoder (transformers Qwen2_5_VLTextModel: RMSNorm, GQA
  with qkv bias, multimodal RoPE over (t, h, w) positions, SwiGLU) on a
  unified sequence with an image span and text, positions from the oracle's
  restatement of get_rope_index;
* Llama (transformers LlamaModel: 1-D RoPE, no bias) at the LLaVA decoder's
  head geometry.

Checked: every layer's K and V (post-RoPE keys, as the KV cache holds them),
the last token's normed hidden state and its logits."""
import dataclasses

import pytest
import torch

from oracle import model_ref

pytest.importorskip("transformers")


def _oracle_weights(shape, seed=0):
    """Random fp32 weights in the oracle layout, with non-trivial norm
    weights (the product folds them; the oracle applies them)."""
    Wv, Wd = model_ref.random_weights_f32(shape, seed=seed, vit_layers=1)
    g = torch.Generator().manual_seed(seed + 7)
    for L in Wd["layers"]:
        L["in_w"] = 1.0 + 0.1 * torch.randn(shape.decoder.d, generator=g)
        L["post_w"] = 1.0 + 0.1 * torch.randn(shape.decoder.d, generator=g)
    Wd["final_w"] = 1.0 + 0.1 * torch.randn(shape.decoder.d, generator=g)
    return Wd


def _load_layers(model_layers, Wd, d):
    with torch.no_grad():
        for blk, L in zip(model_layers, Wd["layers"]):
            blk.input_layernorm.weight.copy_(L["in_w"])
            blk.post_attention_layernorm.weight.copy_(L["post_w"])
            q, k, v = L["qkv_w"].split([d.q_dim, d.kv_dim, d.kv_dim], 0)
            blk.self_attn.q_proj.weight.copy_(q)
            blk.self_attn.k_proj.weight.copy_(k)
            blk.self_attn.v_proj.weight.copy_(v)
            if L["qkv_b"] is not None:
                qb, kb, vb = L["qkv_b"].split([d.q_dim, d.kv_dim, d.kv_dim], 0)
                blk.self_attn.q_proj.bias.copy_(qb)
                blk.self_attn.k_proj.bias.copy_(kb)
                blk.self_attn.v_proj.bias.copy_(vb)
            blk.self_attn.o_proj.weight.copy_(L["o_w"])
            gate, up = model_ref.deinterleave(L["gu_w"])
            blk.mlp.gate_proj.weight.copy_(gate[: d.d_ff])
            blk.mlp.up_proj.weight.copy_(up[: d.d_ff])
            blk.mlp.down_proj.weight.copy_(L["down_w"][:, : d.d_ff])


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


def _compare(out, ks, vs, hl, logits, model, lm_head, d, N):
    cache = out.past_key_values
    for li in range(len(ks)):
        hk, hv = (cache.layers[li].keys, cache.layers[li].values) if hasattr(cache, "layers") \
            else cache[li]
        hk = hk[0].transpose(0, 1).reshape(N, d.kv_dim)
        hv = hv[0].transpose(0, 1).reshape(N, d.kv_dim)
        assert _rel(ks[li], hk) < 1e-4, ("K", li, _rel(ks[li], hk))
        assert _rel(vs[li], hv) < 1e-4, ("V", li, _rel(vs[li], hv))
    h_last = out.last_hidden_state[0, -1]
    assert _rel(hl, h_last) < 1e-4
    assert _rel(logits, h_last @ lm_head.t()) < 1e-4


def test_decoder_ref_matches_transformers_qwen2_5_vl_text_mrope():
    from transformers.models.qwen2_5_vl.configuration_qwen2_5_vl import Qwen2_5_VLTextConfig
    from transformers.models.qwen2_5_vl.modeling_qwen2_5_vl import Qwen2_5_VLTextModel

    from paper_2507_10069_b200 import shapes
    s = shapes.QWEN_VL_7B
    dec = dataclasses.replace(s.decoder, layers=2, d=896, hq=7, hkv=1, d_ff=640, vocab=1000)
    shape = dataclasses.replace(s, decoder=dec)
    Wd = _oracle_weights(shape)
    cfg = Qwen2_5_VLTextConfig(
        vocab_size=dec.vocab, hidden_size=dec.d, intermediate_size=dec.d_ff,
        num_hidden_layers=dec.layers, num_attention_heads=dec.hq, num_key_value_heads=dec.hkv,
        rms_norm_eps=dec.eps, max_position_embeddings=4096,
        rope_parameters={"rope_type": "default", "rope_theta": dec.rope_theta,
                         "mrope_section": list(dec.mrope_section)})
    cfg._attn_implementation = "eager"
    model = Qwen2_5_VLTextModel(cfg).eval()
    _load_layers(model.layers, Wd, dec)
    with torch.no_grad():
        model.norm.weight.copy_(Wd["final_w"])
    # unified sequence: system prefix, a 6 x 4 merged-grid image, text
    syms = [("pfx", 1)] * 5 + [("img", 24)] + [("txt", 1)] * 9
    pos3 = model_ref.mrope_positions_ref(syms)
    N = pos3.shape[0]
    assert N == 5 + 24 + 9
    x = torch.randn(N, dec.d, generator=torch.Generator().manual_seed(3)) * 0.5
    with torch.no_grad():
        ks, vs, hl, logits = model_ref.decoder_ref(shape, Wd, x, pos3=pos3)
        out = model(inputs_embeds=x[None], position_ids=pos3.t()[:, None, :].long(),
                    use_cache=True)
    _compare(out, ks, vs, hl, logits, model, Wd["lm_head"], dec, N)


def test_decoder_ref_matches_transformers_llama():
    from transformers import LlamaConfig, LlamaModel

    from paper_2507_10069_b200 import shapes
    s = shapes.LLAVA_7B
    dec = dataclasses.replace(s.decoder, layers=2, d=512, hq=4, hkv=4, d_ff=768, vocab=1000)
    shape = dataclasses.replace(s, decoder=dec)
    Wd = _oracle_weights(shape, seed=1)
    cfg = LlamaConfig(vocab_size=dec.vocab, hidden_size=dec.d, intermediate_size=dec.d_ff,
                      num_hidden_layers=dec.layers, num_attention_heads=dec.hq,
                      num_key_value_heads=dec.hkv, rms_norm_eps=dec.eps,
                      max_position_embeddings=4096,
                      rope_parameters={"rope_type": "default", "rope_theta": dec.rope_theta})
    cfg._attn_implementation = "eager"
    model = LlamaModel(cfg).eval()
    _load_layers(model.layers, Wd, dec)
    with torch.no_grad():
        model.norm.weight.copy_(Wd["final_w"])
    N = 37
    x = torch.randn(N, dec.d, generator=torch.Generator().manual_seed(4)) * 0.5
    with torch.no_grad():
        ks, vs, hl, logits = model_ref.decoder_ref(shape, Wd, x)
        out = model(inputs_embeds=x[None], use_cache=True)
    _compare(out, ks, vs, hl, logits, model, Wd["lm_head"], dec, N)
