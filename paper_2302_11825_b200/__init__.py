"""B200-native boundary value caching (BVC) — the hot path of arXiv 2302.11825.

The product is libbvc_b200.so (C ABI: include/bvc_b200.h): sm_100a CUDA kernels
for the cache-construction walks and the interior gather, with C++ host code for
the scene, solve region and BVH. `api` mirrors the reference's C++ operator API
(/root/reference/proj/core/include/bvc/cache.h, pointwise.h, scene.h) in Python.
"""
from . import abi  # noqa: F401
from .api import *  # noqa: F401,F403
from .api import lib, library_path  # noqa: F401

__all__ = [name for name in dir() if not name.startswith("_")]
