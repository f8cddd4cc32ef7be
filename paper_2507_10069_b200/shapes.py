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
    # Qwen2.5-VL vision tower ("qwen"): RMSNorm, SwiGLU MLP with biases, 2-D
    # rotary positions, no CLS / absolute positions, Conv3d patch embed over
    # `temporal` duplicated frames, windowed attention (window x window
    # patches) except in `full_layers`, 2x2 patch merger (`merge`).
    arch: str = "clip"          # clip | qwen
    temporal: int = 1
    merge: int = 1
    window: int = 0             # patches per window side (0: full attention everywhere)
    full_layers: tuple = ()
    rope_theta: float = 10000.0

    @property
    def head_dim(self) -> int:
        return self.d // self.heads

    @property
    def k_in(self) -> int:
        return 3 * self.temporal * self.patch * self.patch

    @property
    def d_ff_pad(self) -> int:
        return (self.d_ff + 127) // 128 * 128

    @property
    def merged_dim(self) -> int:
        return self.d * self.merge * self.merge

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
    # multimodal RoPE (Qwen2-VL): rotary pairs [0, s0) rotate by the temporal
    # position, [s0, s0+s1) by the row, the rest by the column (images);
    # text tokens carry t = h = w, i.e. plain 1-D RoPE.  () = 1-D RoPE.
    mrope_section: tuple = ()
    # Llama-3.2-Vision (Mllama): indices (into the `layers` layer stack) of the
    # gated cross-attention layers; text tokens attend to the request's image
    # tokens there, and images occupy no self-attention positions (§8f-3)
    cross_layers: tuple = ()

    @property
    def q_dim(self) -> int:
        return self.hq * self.hd

    @property
    def cross(self) -> tuple:
        """Cross-attention layer indices present in this (possibly truncated)
        stack."""
        return tuple(c for c in self.cross_layers if c < self.layers)

    @property
    def kv_layers(self) -> int:
        """KV planes per token row: the self-attention layers (a text token's
        K/V) — an image token's row holds its cross-attention K/V in planes
        0..len(cross)-1."""
        return self.layers - len(self.cross)

    @property
    def kv_dim(self) -> int:
        return self.hkv * self.hd

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.kv_layers * self.kv_dim * 2

    @property
    def d_ff_pad(self) -> int:
        return (self.d_ff + 127) // 128 * 128

    def linear_flops_per_token(self) -> float:
        """GEMM FLOPs of one (text) token through the decoder stack."""
        d, ff = self.d, self.d_ff
        mlp = 2 * d * 2 * ff + 2 * ff * d
        per_layer = 2 * d * (self.q_dim + 2 * self.kv_dim) + 2 * self.q_dim * d + mlp
        per_cross = 2 * d * self.q_dim + 2 * self.q_dim * d + mlp
        return self.kv_layers * per_layer + len(self.cross) * per_cross

    def cross_kv_flops_per_image_token(self) -> float:
        """Cross-attention K/V projections of one image token (all layers)."""
        return len(self.cross) * 2 * self.d * 2 * self.kv_dim


@dataclass(frozen=True)
class ModelShape:
    name: str
    vision: VisionShape
    proj_hidden: int
    decoder: DecoderShape

    def vit_flops(self, n_patches: int, window_lens=None) -> float:
        """Algorithmic FLOPs of encoding one image of n_patches patches
        (patch embed + layers incl. attention + projector / merger).
        window_lens: patch counts of the attention windows (Qwen)."""
        v = self.vision
        if v.arch == "qwen":
            N, d = float(n_patches), v.d
            f = 2.0 * N * v.k_in * d
            lin = 2.0 * N * d * 3 * d + 2.0 * N * d * d + 2.0 * N * d * 2 * v.d_ff \
                + 2.0 * N * v.d_ff * d
            n_full = sum(1 for i in range(v.layers) if i in v.full_layers)
            wl = window_lens if window_lens is not None else [n_patches]
            win = 4.0 * d * float(sum(int(x) * int(x) for x in wl))
            f += v.layers * lin + n_full * 4.0 * N * N * d + (v.layers - n_full) * win
            Nm = N / (v.merge * v.merge)
            f += 2.0 * Nm * v.merged_dim * self.proj_hidden \
                + 2.0 * Nm * self.proj_hidden * self.decoder.d
            return f
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

# Qwen2.5-VL vision tower (shared by 7B and 72B): 32 layers, d 1280, 16
# heads of 80, SwiGLU 3420, RMSNorm 1e-6, patch 14 x 14 x 2 frames, 112-px
# windows (8 x 8 patches) except layers 7/15/23/31, 2x2 merger -> 5120 ->
# decoder width.
QWEN_VISION = VisionShape(layers=32, d=1280, heads=16, d_ff=3420, act="silu", cls=False,
                          pre_norm=False, eps=1e-6, max_pos=0, arch="qwen", temporal=2,
                          merge=2, window=8, full_layers=(7, 15, 23, 31), rope_theta=10000.0)

# Qwen2.5-VL-7B (C3): decoder GQA 28/4, qkv bias, rope theta 1e6, M-RoPE
# sections (16, 24, 24).
QWEN_VL_7B = ModelShape(
    "qwen2.5-vl-7b",
    QWEN_VISION,
    proj_hidden=5120,
    decoder=DecoderShape(layers=28, d=3584, hq=28, hkv=4, hd=128, d_ff=18944, vocab=152064,
                         rope_theta=1e6, qkv_bias=True, eps=1e-6, mrope_section=(16, 24, 24)),
)

# Qwen2.5-VL-72B (C5): decoder GQA 64/8, qkv bias, M-RoPE.
QWEN_VL_72B = ModelShape(
    "qwen2.5-vl-72b",
    QWEN_VISION,
    proj_hidden=5120,
    decoder=DecoderShape(layers=80, d=8192, hq=64, hkv=8, hd=128, d_ff=29568, vocab=152064,
                         rope_theta=1e6, qkv_bias=True, eps=1e-6, mrope_section=(16, 24, 24)),
)

# Llama-3.2-11B-Vision (C4): 40-layer text decoder whose layers 3, 8, ..., 38
# are gated cross-attention layers over the image tokens.
LLAMA32_11B_V = ModelShape(
    "llama-3.2-11b-vision",
    # vision: 32 local + 8 global layers of width 1280, 16 heads (hd 80), run
    # as plain pre-LN layers (the global layers' tanh gates and the tile /
    # aspect-ratio embeddings are not modelled)
    VisionShape(layers=40, d=1280, heads=16, d_ff=5120, act="gelu_erf", cls=True,
                pre_norm=True, max_pos=32768),
    proj_hidden=4096,
    decoder=DecoderShape(layers=40, d=4096, hq=32, hkv=8, hd=128, d_ff=14336, vocab=128256,
                         rope_theta=500000.0, eps=1e-5,
                         cross_layers=(3, 8, 13, 18, 23, 28, 33, 38)),
)

# tiny cross-attention model (tests): self, cross, self
TINY_X = ModelShape(
    "tiny-mllama",
    VisionShape(layers=1, d=256, heads=4, d_ff=1024, act="gelu_erf", cls=True,
                pre_norm=True, max_pos=16384),
    proj_hidden=256,
    decoder=DecoderShape(layers=3, d=256, hq=4, hkv=2, hd=64, d_ff=1024, vocab=32000,
                         rope_theta=500000.0, cross_layers=(1,)),
)

SHAPES = {"tiny": TINY, "llava-7b": LLAVA_7B, "qwen-7b": QWEN_VL_7B, "qwen-72b": QWEN_VL_72B,
          "llama-11b-v": LLAMA32_11B_V, "tiny-x": TINY_X}


def patch_grid(token_count: int, merge: int = 1) -> tuple[int, int]:
    """Patch grid (gh, gw) of an image that must yield token_count decoder
    tokens: the merged grid is the near-square factorisation (mh, mw) of
    token_count (mh <= mw), and each merged token covers merge x merge
    patches, so (gh, gw) = (merge mh, merge mw)."""
    mh, mw = merged_grid(token_count)
    return mh * merge, mw * merge


def merged_grid(token_count: int) -> tuple[int, int]:
    n = token_count
    best = (1, n)
    for a in range(1, int(math.isqrt(n)) + 1):
        if n % a == 0:
            best = (a, n // a)
    return best
