"""Model shapes for the BASELINE.json configs (random-init weights of these
architectures).  The reference has no models: encode /
prefill are analytic there (pkg/src/mmsim/costmodel.py:102-119), so these
are the public architectures of the named model families.

Image token accounting follows the reference: an image symbol weighs
`token_count` KV tokens (pkg/src/mmsim/engine.py:451-453), so the encoder
must emit exactly token_count rows per image.  Patch grid
for token_count T with merge m: factor T*m^2 into a near-square (gh, gw).
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class VisionShape:
    layers: int          # layers actually run (LLaVA uses the penultimate)
    d: int
    heads: int
    d_ff: int
    patch: int = 14
    act: str = "quick_gelu"     # quick_gelu | gelu_tanh | gelu_erf
    cls: bool = True
    pre_norm: bool = True       # CLIP "pre_layrnorm" before the encoder
    eps: float = 1e-5
    max_pos: int = 577          # learned absolute position embeddings
    mean: tuple = (0.48145466, 0.4578275, 0.40821073)
    std: tuple = (0.26862954, 0.26130258, 0.27577711)

    @property
    def head_dim(self) -> int:
        return self.d // self.heads

    @property
    def k_in(self) -> int:
        return 3 * self.patch * self.patch

    @property
    def k_pad(self) -> int:
        return (self.k_in + 63) // 64 * 64


@dataclass(frozen=True)
class DecoderShape:
    layers: int
    d: int
    hq: int
    hkv: int
    hd: int
    d_ff: int
    vocab: int
    rope_theta: float = 10000.0
    qkv_bias: bool = False
    eps: float = 1e-5

    @property
    def q_dim(self) -> int:
        return self.hq * self.hd

    @property
    def kv_dim(self) -> int:
        return self.hkv * self.hd

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.layers * self.kv_dim * 2

    @property
    def d_ff_pad(self) -> int:
        return (self.d_ff + 127) // 128 * 128

    def linear_flops_per_token(self) -> float:
        d, ff = self.d, self.d_ff
        per_layer = 2 * d * (self.q_dim + 2 * self.kv_dim) + 2 * self.q_dim * d + 2 * d * 2 * ff \
            + 2 * ff * d
        return self.layers * per_layer


@dataclass(frozen=True)
class ModelShape:
    name: str
    vision: VisionShape
    proj_hidden: int
    decoder: DecoderShape

    def vit_flops(self, n_patches: int) -> float:
        """Algorithmic FLOPs of encoding one image of n_patches patches
        (patch embed + layers incl. full attention + projector)."""
        v = self.vision
        L = n_patches + (1 if v.cls else 0)
        f = 2.0 * n_patches * v.k_in * v.d
        f += v.layers * (2.0 * L * v.d * 3 * v.d + 2.0 * L * v.d * v.d + 4.0 * L * v.d * v.d_ff
                         + 4.0 * L * L * v.d)
        f += 2.0 * L * v.d * self.proj_hidden + 2.0 * L * self.proj_hidden * self.decoder.d
        return f


TINY = ModelShape(
    "tiny-mllm",
    VisionShape(layers=2, d=256, heads=4, d_ff=1024, act="quick_gelu", cls=False,
                pre_norm=True, max_pos=16384),
    proj_hidden=256,
    decoder=DecoderShape(layers=2, d=256, hq=4, hkv=2, hd=64, d_ff=1024, vocab=32000),
)

# LLaVA-1.5-7B: CLIP ViT-L/14-336 (features of the penultimate of 24 layers)
# + 2-layer GELU projector + Llama-2/Vicuna-7B.
LLAVA_7B = ModelShape(
    "llava-1.5-7b",
    VisionShape(layers=23, d=1024, heads=16, d_ff=4096, act="quick_gelu", cls=True,
                pre_norm=True, max_pos=577),
    proj_hidden=4096,
    decoder=DecoderShape(layers=32, d=4096, hq=32, hkv=32, hd=128, d_ff=11008, vocab=32000,
                         rope_theta=10000.0, eps=1e-5),
)

# Qwen2.5-VL-7B decoder (C3): GQA 28/4, qkv bias, rope theta 1e6.  The vision
# tower here is the CLIP-style stand-in (the Qwen ViT's windowed attention /
# 2-D RoPE / 2x2 merger are listed as next in DESIGN.md).
QWEN_VL_7B = ModelShape(
    "qwen2.5-vl-7b",
    VisionShape(layers=32, d=1280, heads=10, d_ff=3456, act="gelu_tanh", cls=False,
                pre_norm=False, max_pos=32768),
    proj_hidden=5120,
    decoder=DecoderShape(layers=28, d=3584, hq=28, hkv=4, hd=128, d_ff=18944, vocab=152064,
                         rope_theta=1e6, qkv_bias=True, eps=1e-6),
)

# Qwen2.5-VL-72B decoder (C5): GQA 64/8, qkv bias.
QWEN_VL_72B = ModelShape(
    "qwen2.5-vl-72b",
    VisionShape(layers=32, d=1280, heads=10, d_ff=3456, act="gelu_tanh", cls=False,
                pre_norm=False, max_pos=32768),
    proj_hidden=5120,
    decoder=DecoderShape(layers=80, d=8192, hq=64, hkv=8, hd=128, d_ff=29568, vocab=152064,
                         rope_theta=1e6, qkv_bias=True, eps=1e-6),
)

# Llama-3.2-11B-Vision text decoder self-attention stack (C4); the 8 gated
# cross-attention layers are listed as next in DESIGN.md.
LLAMA32_11B_V = ModelShape(
    "llama-3.2-11b-vision",
    VisionShape(layers=32, d=1280, heads=10, d_ff=5120, act="gelu_erf", cls=True,
                pre_norm=True, max_pos=32768),
    proj_hidden=4096,
    decoder=DecoderShape(layers=32, d=4096, hq=32, hkv=8, hd=128, d_ff=14336, vocab=128256,
                         rope_theta=500000.0, eps=1e-5),
)

SHAPES = {"tiny": TINY, "llava-7b": LLAVA_7B, "qwen-7b": QWEN_VL_7B, "qwen-72b": QWEN_VL_72B,
          "llama-11b-v": LLAMA32_11B_V}


def patch_grid(token_count: int, merge: int = 1) -> tuple[int, int]:
    """Near-square factorisation (gh, gw) of token_count*merge^2 patches."""
    n = token_count * merge * merge
    best = (1, n)
    for a in range(1, int(math.isqrt(n)) + 1):
        if n % a == 0:
            best = (a, n // a)
    return best
