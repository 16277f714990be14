"""B200-native LongFlow (arXiv 2603.11504) fused decode-step operator.

The product is the C-ABI library ``liblongflow.so`` (include/longflow.h) built from
``csrc/`` for sm_100a; ``binding`` is its thin ctypes wrapper.  See DESIGN.md.
"""
from .binding import Cache, CacheConfig, LFError, load, make_config, cache_bytes  # noqa: F401

__all__ = ["Cache", "CacheConfig", "LFError", "load", "make_config", "cache_bytes"]
