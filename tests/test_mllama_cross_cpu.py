"""Pin of the cross-attention oracle (§8f-3, Llama-3.2-Vision): the fp32
restatement oracle/model_ref.cross_layer_ref, fed the kernel-layout weights
of paper_2507_10069_b200.weights.fold_cross_layer, equals transformers'
own MllamaCrossAttentionDecoderLayer run on CPU with the unfolded weights
(transformers is a third-party package in this image; it plays the role of
the reference for this model family, which the ElasticMM simulator only
models analytically)."""
import pytest
import torch

from oracle import model_ref


def _mllama():
    try:
        from transformers.models.mllama import modeling_mllama as m
        from transformers.models.mllama.configuration_mllama import MllamaTextConfig
        return m, MllamaTextConfig
    except Exception:
        return None, None


@pytest.mark.parametrize("hq,hkv,N,M", [(4, 2, 37, 50), (8, 8, 5, 129), (8, 1, 64, 3)])
def test_cross_layer_matches_transformers(hq, hkv, N, M):
    m, Cfg = _mllama()
    if m is None:
        pytest.skip("transformers Mllama not importable")
    from paper_2507_10069_b200.shapes import DecoderShape
    from paper_2507_10069_b200.weights import fold_cross_layer, random_cross_layer
    hd, D, FF = 32, hq * 32, 256
    d = DecoderShape(layers=1, d=D, hq=hq, hkv=hkv, hd=hd, d_ff=FF, vocab=16,
                     cross_layers=(0,))
    g = torch.Generator().manual_seed(hq * 100 + M)
    raw = random_cross_layer(g, d, device="cpu", dtype=torch.float32)
    # larger-than-init weights so every term matters numerically
    for k in ("q_proj", "k_proj", "v_proj", "o_proj", "gate", "up", "down"):
        raw[k] = raw[k] * 25.0
    raw["attn_gate"], raw["mlp_gate"] = 0.7, -0.4
    cfg = Cfg(hidden_size=D, num_attention_heads=hq, num_key_value_heads=hkv,
              intermediate_size=FF, rms_norm_eps=d.eps, num_hidden_layers=1,
              cross_attention_layers=[0], vocab_size=16)
    cfg._attn_implementation = "eager"
    layer = m.MllamaCrossAttentionDecoderLayer(cfg, layer_idx=0).eval()
    ca = layer.cross_attn
    with torch.no_grad():
        ca.q_proj.weight.copy_(raw["q_proj"])
        ca.k_proj.weight.copy_(raw["k_proj"])
        ca.v_proj.weight.copy_(raw["v_proj"])
        ca.o_proj.weight.copy_(raw["o_proj"])
        ca.q_norm.weight.copy_(raw["q_norm"])
        ca.k_norm.weight.copy_(raw["k_norm"])
        layer.input_layernorm.weight.copy_(raw["in_norm"])
        layer.post_attention_layernorm.weight.copy_(raw["post_norm"])
        layer.mlp.gate_proj.weight.copy_(raw["gate"])
        layer.mlp.up_proj.weight.copy_(raw["up"])
        layer.mlp.down_proj.weight.copy_(raw["down"])
        layer.cross_attn_attn_gate.fill_(raw["attn_gate"])
        layer.cross_attn_mlp_gate.fill_(raw["mlp_gate"])
    x = torch.randn(N, D, generator=g)
    img = torch.randn(M, D, generator=g)
    with torch.no_grad():
        out = layer(x[None], cross_attention_states=img[None], cross_attention_mask=None,
                    attention_mask=None, full_text_row_masked_out_mask=None)
    ref = out[0] if isinstance(out, tuple) else out
    ref = ref[0]
    got, k, v = model_ref.cross_layer_ref(d, fold_cross_layer(raw, d), x, img)
    err = ((got - ref).norm() / ref.norm()).item()
    assert err < 1e-5, err
    # the cached cross K/V: the layer's keys normalised without k_norm's
    # weight (folded into q_norm's) and its raw values
    kr = ca.k_norm(ca.k_proj(img).view(M, hkv, hd))
    kw = (k.view(M, hkv, hd) * raw["k_norm"]).detach()
    assert torch.allclose(kw, kr.detach(), rtol=1e-4, atol=1e-5)
    assert torch.allclose(v, ca.v_proj(img).detach(), rtol=1e-5, atol=1e-5)
