"""Batched ViT encoder for uncached images (K4) on tcgen05 kernels.

Replaces the analytic CostProfile.encode_time (pkg/src/mmsim/costmodel.py:
102-111) that Engine.start_encode charges (pkg/src/mmsim/engine.py:565-580):
every missed image of an encode job is patchified from its pixels, run
through the vision tower (pre-LN transformer, bidirectional attention per
image) and the projector, producing exactly `token_count` decoder-space rows
per image (the image slab inserted into the image pool,
engine.py:582-600 -> cache.py:381-383).
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import ops
from .shapes import ModelShape

_ACT = {"quick_gelu": ops.EPI_QUICK_GELU, "gelu_tanh": ops.EPI_GELU_TANH,
        "gelu_erf": ops.EPI_GELU_ERF}


class VisionEncoder:
    def __init__(self, shape: ModelShape, W: dict):
        self.shape = shape
        self.W = W
        self.last_flops = 0.0

    def encode(self, pix: torch.Tensor, pix_off, grids) -> tuple[torch.Tensor, list]:
        """pix: packed uint8 HWC images on the device; pix_off[i]: byte offset
        of image i; grids[i] = (gh, gw) patch grid.  Returns (rows, spans):
        image i's embeddings are rows[spans[i][0]:spans[i][1]] (its patches
        only; CLS excluded), [n_patches_i, d_decoder]."""
        v, W = self.shape.vision, self.W
        dev = pix.device
        n_img = len(grids)
        n_p = np.array([gh * gw for gh, gw in grids], np.int64)
        patch_off = np.zeros(n_img + 1, np.int64)
        np.cumsum(n_p, out=patch_off[1:])
        cls = 1 if v.cls else 0
        tok_off = np.zeros(n_img + 1, np.int64)
        np.cumsum(n_p + cls, out=tok_off[1:])
        assert int((n_p + cls).max()) <= v.max_pos, "position table too small for the grid"
        n_rows = int(tok_off[-1])
        i64 = lambda a: ops.h2d(a, dev, np.int64)
        i32 = lambda a: ops.h2d(a, dev, np.int32)
        patches = torch.empty(int(patch_off[-1]), v.k_pad, device=dev, dtype=torch.bfloat16)
        ops.patchify(pix, i64(pix_off), i32([g[0] for g in grids]), i32([g[1] for g in grids]),
                     i64(patch_off[:-1]), int(n_p.max()), v.patch, v.k_pad, v.mean, v.std,
                     patches)
        pe = ops.gemm(patches, W["patch_w"])
        x = torch.empty(n_rows, v.d, device=dev, dtype=torch.bfloat16)
        ops.vit_embed(pe, W["cls"], W["pos"], i64(tok_off), i64(patch_off[:-1]), x)
        if v.pre_norm:
            x = ops.norm(x, W["pre_w"], W["pre_b"], v.eps)
        hd = v.head_dim
        meta = ops.AttnMeta(tok_off[:-1], n_p + cls, tok_off[:-1], n_p + cls, v.heads,
                            causal=False, device=dev)
        act = _ACT[v.act]
        d = v.d
        for L in W["layers"]:
            h = ops.norm(x, L["ln1_w"], L["ln1_b"], v.eps)
            qkv = ops.gemm(h, L["qkv_w"], bias=L["qkv_b"])
            # q / k / v read in place from the fused QKV rows (strided TMA maps)
            a = ops.attention(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], meta, v.heads, hd,
                              label="attention_vit_full")
            x = ops.gemm(a, L["o_w"], bias=L["o_b"], residual=x)
            h = ops.norm(x, L["ln2_w"], L["ln2_b"], v.eps)
            m = ops.gemm(h, L["fc1_w"], bias=L["fc1_b"], epi=act)
            x = ops.gemm(m, L["fc2_w"], bias=L["fc2_b"], residual=x)
        y = ops.gemm(x, W["p1_w"], bias=W["p1_b"], epi=ops.EPI_GELU_ERF)
        y = ops.gemm(y, W["p2_w"], bias=W["p2_b"])
        self.last_flops = float(sum(self.shape.vit_flops(int(n)) for n in n_p))
        spans = [(int(tok_off[i]) + cls, int(tok_off[i + 1])) for i in range(n_img)]
        return y, spans


# ----------------------------------------------------------------- Qwen2.5-VL
from .encoder_plan import window_plan  # noqa: E402,F401  (pure numpy, shared with bench.py)


class QwenVisionEncoder:
    """Qwen2.5-VL vision tower + patch merger on tcgen05 kernels (K4).

    Per layer: folded-RMSNorm QKV GEMM (+bias) -> in-place 2-D RoPE of the q
    and k heads -> varlen attention straight from the fused QKV buffer
    (head_dim 80; windows of 8x8 patches, or the whole image in
    full_layers) -> O GEMM (+bias, +residual, row sum of squares for the
    next norm) -> gate/up GEMM with the SwiGLU epilogue -> down GEMM
    (+bias, +residual).  Merger: RMSNorm gathering each 2x2 unit's rows in
    raster order -> [N/4, 4d] -> GELU MLP -> decoder width."""

    def __init__(self, shape: ModelShape, W: dict):
        self.shape = shape
        self.W = W
        self.last_flops = 0.0
        self._plans: dict = {}

    def plan(self, grid) -> dict:
        p = self._plans.get(grid)
        if p is None:
            v = self.shape.vision
            p = window_plan(grid[0], grid[1], v.merge, v.window)
            self._plans[grid] = p
        return p

    def _rope2_table(self, dev):
        """(cos, sin) of pos * theta^(-2j/(hd/2)), j < hd/4, for patch-grid
        positions up to 4096 (Qwen2.5-VL VisionRotaryEmbedding(hd / 2))."""
        t = getattr(self, "_rope2", None)
        if t is None or t.device != dev:
            v = self.shape.vision
            t = ops.rope_table(4096, v.head_dim // 2, v.rope_theta, device=dev)
            self._rope2 = t
        return t

    def encode(self, pix: torch.Tensor, pix_off, grids) -> tuple[torch.Tensor, list]:
        v, W = self.shape.vision, self.W
        dev = pix.device
        d, hd, m2 = v.d, v.head_dim, v.merge * v.merge
        plans = [self.plan(tuple(g)) for g in grids]
        n_p = np.array([gh * gw for gh, gw in grids], np.int64)
        off = np.zeros(len(grids) + 1, np.int64)
        np.cumsum(n_p, out=off[1:])
        N = int(off[-1])
        cat = lambda k: np.concatenate([p[k] for p in plans])
        row_img = np.repeat(np.arange(len(grids), dtype=np.int32), n_p)
        unit_rows = np.concatenate([p["unit_rows"] + off[i] for i, p in enumerate(plans)])
        i32 = lambda a: ops.h2d(a, dev, np.int32)
        pos_h, pos_w = i32(cat("pos_h")), i32(cat("pos_w"))
        patches = torch.empty(N, v.k_pad, device=dev, dtype=torch.bfloat16)
        ops.patchify_rows(pix, ops.h2d(pix_off, dev, np.int64), i32([g[1] for g in grids]),
                          i32(row_img), i32(cat("row_patch")), v.patch, v.temporal, v.k_pad,
                          v.mean, v.std, patches)
        x = ops.gemm(patches, W["patch_w"])
        del patches
        # windowed layers: each image is one sequence whose rows see only
        # their own window (contiguous in this row order)
        wins = [p["window_lens"] for p in plans]
        if (max(int(w.max()) for w in wins) <= 128
                and os.environ.get("EMM_VIT_WINDOW_PACK", "1") != "0"):
            # whole windows packed <= 128 rows per tile, one key block each
            meta_win = ops.AttnMeta.window_packed(off[:-1], wins, v.heads, device=dev)
        else:
            meta_win = ops.AttnMeta(off[:-1], n_p, off[:-1], n_p, v.heads, causal=False,
                                    device=dev, windows=wins)
        meta_full = ops.AttnMeta(off[:-1], n_p, off[:-1], n_p, v.heads, causal=False, device=dev)
        ss = ops.row_sumsq(x)
        ss2 = torch.empty_like(ss)
        rope2 = dict(cs=self._rope2_table(dev), cols=2 * d, hd=hd, pos_h=pos_h, pos_w=pos_w)
        for li, L in enumerate(W["layers"]):
            # fused QKV GEMM: folded RMSNorm, bias and the 2-D RoPE of q / k in
            # the epilogue (pair-interleaved weight rows, weights.rope_pair_perm)
            qkv = ops.gemm_ex(x, L["qkv_w_pi"], bias=L["qkv_b_pi"], row_ss_in=ss, rms_dim=d,
                              rms_eps=v.eps, row_ss_zero=ss2, rope2=rope2)
            full = li in v.full_layers
            a = ops.attention(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:],
                              meta_full if full else meta_win, v.heads, hd,
                              label="attention_vit_full" if full else "attention_vit_window")
            del qkv
            x2 = ops.gemm_ex(a, L["o_w"], bias=L["o_b"], residual=x, row_ss_out=ss2)
            h = ops.gemm_ex(x2, L["gu_w"], epi=ops.EPI_GLU_SILU, bias=L["gu_b"], row_ss_in=ss2,
                            rms_dim=d, rms_eps=v.eps, row_ss_zero=ss)
            x = ops.gemm_ex(h, L["down_w"], bias=L["down_b"], residual=x2, row_ss_out=ss)
            del h, x2
        hq = ops.norm(x, W["lnq_w"], None, v.eps, rows=i32(unit_rows))
        hq = hq.view(N // m2, m2 * d)
        y = ops.gemm(hq, W["p1_w"], bias=W["p1_b"], epi=ops.EPI_GELU_ERF)
        y = ops.gemm(y, W["p2_w"], bias=W["p2_b"])
        self.last_flops = float(sum(self.shape.vit_flops(int(n), p["window_lens"])
                                    for n, p in zip(n_p, plans)))
        spans = [(int(off[i]) // m2, int(off[i + 1]) // m2) for i in range(len(grids))]
        return y, spans


def make_encoder(shape: ModelShape, W: dict):
    return QwenVisionEncoder(shape, W) if shape.vision.arch == "qwen" else VisionEncoder(shape, W)
