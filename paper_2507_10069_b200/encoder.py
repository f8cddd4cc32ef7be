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
        ident = torch.arange(n_rows, device=dev, dtype=torch.int32)
        q = torch.empty(n_rows, v.d, device=dev, dtype=torch.bfloat16)
        k = torch.empty_like(q)
        vv = torch.empty_like(q)
        act = _ACT[v.act]
        for L in W["layers"]:
            h = ops.norm(x, L["ln1_w"], L["ln1_b"], v.eps)
            qkv = ops.gemm(h, L["qkv_w"], bias=L["qkv_b"])
            ops.rope_split(qkv, v.heads, v.heads, hd, q, k, vv, ident)
            a = ops.attention(q, k, vv, meta, v.heads, hd)
            x = ops.gemm(a, L["o_w"], bias=L["o_b"], residual=x)
            h = ops.norm(x, L["ln2_w"], L["ln2_b"], v.eps)
            m = ops.gemm(h, L["fc1_w"], bias=L["fc1_b"], epi=act)
            x = ops.gemm(m, L["fc2_w"], bias=L["fc2_b"], residual=x)
        y = ops.gemm(x, W["p1_w"], bias=W["p1_b"], epi=ops.EPI_GELU_ERF)
        y = ops.gemm(y, W["p2_w"], bias=W["p2_b"])
        self.last_flops = float(sum(self.shape.vit_flops(int(n)) for n in n_p))
        spans = [(int(tok_off[i]) + cls, int(tok_off[i + 1])) for i in range(n_img)]
        return y, spans
