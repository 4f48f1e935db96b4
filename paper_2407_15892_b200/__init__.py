"""B200-native (sm_100a) Mini-Sequence Transformer hot path.

The product is `lib/libmst.so` (tcgen05/TMEM/TMA kernels + C ABI declared in
include/mst/mst.h).  `miniseq` mirrors the reference operator API
 over that ABI.
"""
from ._build import LIB_PATH, build_lib  # noqa: F401

__all__ = ["LIB_PATH", "build_lib"]
