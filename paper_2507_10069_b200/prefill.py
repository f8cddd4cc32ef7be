"""Prefill of the uncached suffix over the paged prefix KV (K3 + K5 + the
decoder layers) on tcgen05 kernels.

Replaces the analytic CostProfile.prefill_time (pkg/src/mmsim/costmodel.py:
113-119) charged by Engine.start_prefill (pkg/src/mmsim/engine.py:602-632)
for a batch of requests whose `cached_prefix` was fixed by
consult_prefix_cache (engine.py:539-547).  Per batch:

  request KV buffer  req_kv[L, 2, rows, kv_dim]: request r owns rows
                     [row0_r, row0_r + P_r + S_r)  (P = cached prefix,
                     S = uncached suffix, P + S = total_input_len)
  K3 gather          prefix rows <- paged pool slots via the block table
  decoder            S_total suffix tokens through every layer; RoPE'd K/V
                     written straight into req_kv; causal attention of each
                     suffix over its P + S keys (K5)
  output             next-token ids of every request (first token => TTFT)
"""
from __future__ import annotations

import numpy as np
import torch

from . import ops
from .keys import TAG_IMG
from .shapes import ModelShape, merged_grid


def mrope_positions(keys: np.ndarray, w: np.ndarray) -> tuple[np.ndarray, np.ndarray,
                                                               np.ndarray]:
    """Qwen2-VL multimodal RoPE positions (t, h, w) of every KV token of one
    unified sequence (engine.py:448-461 symbol order).  A text symbol takes
    (p, p, p) and advances p by 1; an image of token_count T on its merged
    grid (mh, mw) takes (p, p + row, p + col) for its token row * mw + col and
    advances p by max(mh, mw) (get_rope_index: the next text starts at the
    image's largest position + 1).  Positions depend only on the preceding
    symbols, so cached prefix KV stays valid for every continuation."""
    keys = np.asarray(keys, np.uint64)
    w = np.asarray(w, np.int64)
    is_img = (keys >> np.uint64(62)) == np.uint64(TAG_IMG)
    mw_sym = np.ones(len(w), np.int64)
    adv = np.ones(len(w), np.int64)
    for j in np.nonzero(is_img)[0]:
        mh, mw = merged_grid(int(w[j]))
        mw_sym[j], adv[j] = mw, max(mh, mw)
    start = np.zeros(len(w), np.int64)
    np.cumsum(adv[:-1], out=start[1:])
    sym = np.repeat(np.arange(len(w)), w)
    tok_start = np.zeros(len(w), np.int64)
    np.cumsum(w[:-1], out=tok_start[1:])
    within = np.arange(int(w.sum()), dtype=np.int64) - tok_start[sym]
    img = is_img[sym]
    base = start[sym]
    r, c = np.divmod(within, mw_sym[sym])
    pt = base
    ph = np.where(img, base + r, base)
    pwv = np.where(img, base + c, base)
    return pt.astype(np.int32), ph.astype(np.int32), pwv.astype(np.int32)


class Decoder:
    """Llama-style decoder whose RMSNorm weights are folded into the following
    projection (qkv_w, gu_w), so each GEMM consumes the residual stream x
    directly and applies rsqrt(mean(x^2)+eps) per row in its epilogue; the
    residual GEMMs (o_proj, down_proj) emit the per-row sum of squares the
    next norm needs.  RoPE + Q/K/V split + KV-cache write are fused into the
    QKV GEMM epilogue."""

    def __init__(self, shape: ModelShape, W: dict, max_pos: int = 65536):
        self.shape = shape
        self.W = W
        d = shape.decoder
        dev = W["embed"].device
        self.rope_cs = ops.rope_table(max_pos, d.hd, d.rope_theta, device=dev)
        self.max_pos = max_pos
        self.ones_hd = torch.ones(d.hd, device=dev, dtype=torch.bfloat16)

    def forward(self, x: torch.Tensor, req_kv: torch.Tensor, kv_row: torch.Tensor,
                pos: torch.Tensor, meta: ops.AttnMeta, last_rows: torch.Tensor,
                return_hidden: bool = False, pos_h: torch.Tensor | None = None,
                pos_w: torch.Tensor | None = None):
        """x: [S_total, d] input embeddings of the suffix tokens (bf16);
        kv_row / pos: int32 [S_total]; last_rows: int32 [n_req] index of each
        request's last suffix token.  pos_h / pos_w (M-RoPE shapes): the row
        and column positions (pos is then the temporal one).  Returns int32
        next-token ids [n_req] (and the final-normed last hidden states if
        return_hidden)."""
        d, W = self.shape.decoder, self.W
        T = x.shape[0]
        dev = x.device
        q = torch.empty(T, d.q_dim, device=dev, dtype=torch.bfloat16)
        ss = ops.row_sumsq(x)
        ss2 = torch.empty_like(ss)
        for li, L in enumerate(W["layers"]):
            kl, vl = req_kv[li, 0], req_kv[li, 1]
            ops.gemm_ex(x, L["qkv_w"], epi=ops.EPI_QKV_ROPE, bias=L["qkv_b"], row_ss_in=ss,
                        rms_dim=d.d, rms_eps=d.eps, row_ss_zero=ss2,
                        qkv=dict(q_out=q, k_out=kl, v_out=vl, kv_row=kv_row, pos=pos,
                                 rope_cs=self.rope_cs, hq=d.hq, hkv=d.hkv, hd=d.hd,
                                 pos_h=pos_h, pos_w=pos_w, mrope=d.mrope_section))
            a = ops.attention(q, kl, vl, meta, d.hkv, d.hd, label="attention_decoder")
            x2 = ops.gemm_ex(a, L["o_w"], residual=x, row_ss_out=ss2)
            m = ops.gemm_ex(x2, L["gu_w"], epi=ops.EPI_GLU_SILU, row_ss_in=ss2, rms_dim=d.d,
                            rms_eps=d.eps, row_ss_zero=ss)
            x = ops.gemm_ex(m, L["down_w"], residual=x2, row_ss_out=ss)
        hl = ops.norm(x, W["final_w"], None, d.eps, rows=last_rows)
        logits = ops.gemm(hl, W["lm_head"])
        ids = ops.argmax_rows(logits)
        if return_hidden:
            return ids, hl, logits
        return ids

    def forward_cross(self, x: torch.Tensor, req_kv: torch.Tensor, kv_row: torch.Tensor,
                      pos: torch.Tensor, meta_self: ops.AttnMeta, meta_cross, n_img_rows: int,
                      last_rows: torch.Tensor) -> torch.Tensor:
        """Cross-attention decoder stack (Llama-3.2-Vision): x [S, d] the
        suffix TEXT tokens, rows of requests with images first (n_img_rows of
        them).  Self layers as forward() (plane = self-layer index, RoPE at
        text positions); cross layer c on rows [0, n_img_rows) only: q =
        headnorm(x Wq), attention over the request's image rows of plane c
        (non-causal), gated o / MLP (gates folded into the weights), updated
        in place — text-only requests skip the layer, as Mllama's
        full_text_row_masked_out_mask does.  Returns next-token ids."""
        d, W = self.shape.decoder, self.W
        T = x.shape[0]
        dev = x.device
        q = torch.empty(T, d.q_dim, device=dev, dtype=torch.bfloat16)
        ss = ops.row_sumsq(x)
        ss2 = torch.empty_like(ss)
        plane = 0
        ci = 0
        for li, L in enumerate(W["layers"]):
            if L.get("cross"):
                c, ci = ci, ci + 1
                if meta_cross is None or n_img_rows == 0:
                    continue
                xv, ssv, ss2v = x[:n_img_rows], ss[:n_img_rows], ss2[:n_img_rows]
                qx = ops.gemm_ex(xv, L["xq_w"], row_ss_in=ssv, rms_dim=d.d, rms_eps=d.eps,
                                 row_ss_zero=ss2v)
                qh = qx.view(n_img_rows * d.hq, d.hd)
                ops.norm(qh, L["xq_norm"], None, d.eps, out=qh)
                a = ops.attention(qx, req_kv[c, 0], req_kv[c, 1], meta_cross, d.hkv, d.hd,
                                  label="attention_cross")
                x2 = ops.gemm_ex(a, L["xo_w"], residual=xv, row_ss_out=ss2v)
                m = ops.gemm_ex(x2, L["gu_w"], epi=ops.EPI_GLU_SILU, row_ss_in=ss2v,
                                rms_dim=d.d, rms_eps=d.eps, row_ss_zero=ssv)
                ops.gemm_ex(m, L["down_w"], out=xv, residual=x2, row_ss_out=ssv)
                continue
            kl, vl = req_kv[plane, 0], req_kv[plane, 1]
            plane += 1
            ops.gemm_ex(x, L["qkv_w"], epi=ops.EPI_QKV_ROPE, bias=L["qkv_b"], row_ss_in=ss,
                        rms_dim=d.d, rms_eps=d.eps, row_ss_zero=ss2,
                        qkv=dict(q_out=q, k_out=kl, v_out=vl, kv_row=kv_row, pos=pos,
                                 rope_cs=self.rope_cs, hq=d.hq, hkv=d.hkv, hd=d.hd))
            a = ops.attention(q, kl, vl, meta_self, d.hkv, d.hd, label="attention_decoder")
            x2 = ops.gemm_ex(a, L["o_w"], residual=x, row_ss_out=ss2)
            m = ops.gemm_ex(x2, L["gu_w"], epi=ops.EPI_GLU_SILU, row_ss_in=ss2, rms_dim=d.d,
                            rms_eps=d.eps, row_ss_zero=ss)
            x = ops.gemm_ex(m, L["down_w"], residual=x2, row_ss_out=ss)
        hl = ops.norm(x, W["final_w"], None, d.eps, rows=last_rows)
        logits = ops.gemm(hl, W["lm_head"])
        return ops.argmax_rows(logits)

    def decode_step(self, tok: torch.Tensor, arena_kv: torch.Tensor, slots: torch.Tensor,
                    pos: torch.Tensor, bt: torch.Tensor, bt_off: torch.Tensor,
                    kv_len: torch.Tensor, max_kv_len: int, return_logits: bool = False,
                    cross: dict | None = None):
        """One decode step of a batch: tok int32 [B]
        (the previous step's tokens, on the device), arena_kv [L, 2, slots,
        kv_dim] the paged decode arena, slots int32 [B] the arena row each
        request's new K/V goes to (written by the fused QKV epilogue, RoPE'd
        at pos), bt / bt_off / kv_len the block tables incl. the new token.
        Same layer code as forward() with the paged decode attention kernel;
        returns int32 next-token ids [B] (and the logits).

        Cross-attention models: bt / kv_len cover the TEXT rows (self
        layers, planes = self-layer index) and `cross` = dict(bt, bt_off,
        kv_len, max_kv_len, xmask) the image rows (plane c of cross layer
        c).  A row without images attends to no key (output 0) and its
        gated MLP is masked through the down GEMM's row scale: xmask[row] =
        inf gives rsqrt(inf) = 0, (1 - eps) * d gives 1 (Mllama's
        full_text_row_masked_out_mask)."""
        d, W = self.shape.decoder, self.W
        B = tok.shape[0]
        dev = tok.device
        x = ops.embed_rows(W["embed"], tok)
        q = torch.empty(B, d.q_dim, device=dev, dtype=torch.bfloat16)
        ss = ops.row_sumsq(x)
        ss2 = torch.empty_like(ss)
        mrope = bool(d.mrope_section)
        plane, ci = 0, 0
        for li, L in enumerate(W["layers"]):
            if L.get("cross"):
                c, ci = ci, ci + 1
                qx = ops.gemm_ex(x, L["xq_w"], row_ss_in=ss, rms_dim=d.d, rms_eps=d.eps,
                                 row_ss_zero=ss2)
                qh = qx.view(B * d.hq, d.hd)
                ops.norm(qh, L["xq_norm"], None, d.eps, out=qh)
                a = ops.decode_attention(qx, arena_kv[c, 0], arena_kv[c, 1], cross["bt"],
                                         cross["bt_off"], cross["kv_len"], d.hkv, d.hd,
                                         max(1, cross["max_kv_len"]))
                x2 = ops.gemm_ex(a, L["xo_w"], residual=x, row_ss_out=ss2)
                m = ops.gemm_ex(x2, L["gu_w"], epi=ops.EPI_GLU_SILU, row_ss_in=ss2,
                                rms_dim=d.d, rms_eps=d.eps, row_ss_zero=ss)
                x = ops.gemm_ex(m, L["down_w"], residual=x2, row_ss_out=ss,
                                row_ss_in=cross["xmask"], rms_dim=d.d, rms_eps=d.eps)
                continue
            kl, vl = arena_kv[plane, 0], arena_kv[plane, 1]
            plane += 1
            # decode tokens are text: M-RoPE (t, h, w) = (p, p, p)
            ops.gemm_ex(x, L["qkv_w"], epi=ops.EPI_QKV_ROPE, bias=L["qkv_b"], row_ss_in=ss,
                        rms_dim=d.d, rms_eps=d.eps, row_ss_zero=ss2,
                        qkv=dict(q_out=q, k_out=kl, v_out=vl, kv_row=slots, pos=pos,
                                 rope_cs=self.rope_cs, hq=d.hq, hkv=d.hkv, hd=d.hd,
                                 pos_h=pos if mrope else None, pos_w=pos if mrope else None,
                                 mrope=d.mrope_section))
            a = ops.decode_attention(q, kl, vl, bt, bt_off, kv_len, d.hkv, d.hd, max_kv_len)
            x2 = ops.gemm_ex(a, L["o_w"], residual=x, row_ss_out=ss2)
            m = ops.gemm_ex(x2, L["gu_w"], epi=ops.EPI_GLU_SILU, row_ss_in=ss2, rms_dim=d.d,
                            rms_eps=d.eps, row_ss_zero=ss)
            x = ops.gemm_ex(m, L["down_w"], residual=x2, row_ss_out=ss)
        hl = ops.norm(x, W["final_w"], None, d.eps)
        logits = ops.gemm(hl, W["lm_head"])
        ids = ops.argmax_rows(logits)
        if return_logits:
            return ids, logits
        return ids
