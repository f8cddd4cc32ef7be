"""B200-native unified multimodal prefix cache feeding encode and prefill.

A drop-in for the hot path of ElasticMM's reference simulator (`mmsim`,
arXiv 2507.10069): `GpuUnifiedCache` replaces `mmsim.cache.UnifiedCache`,
`B200Engine` / `install()` route the encode and prefill stage entry points to
hand-written sm_100a kernels in libemm.so.  See DESIGN.md.
"""

__all__ = ["GpuUnifiedCache", "ImagePool", "PrefixTree", "ReleaseWithoutMatch"]


def __getattr__(name):
    if name in __all__:
        from . import cache
        return getattr(cache, name)
    raise AttributeError(name)
