"""B200-native SELL-C-sigma sparse hot path (GHOST, arXiv:1507.08101).

The product is the C-ABI library lib/libsellkit_b200.so (include/sellkit.h);
this package holds its CUDA sources (csrc/), the ctypes mirror of the C ABI
(sellkit.py) and the host-side distributed driver (dist.py).
"""
__all__ = ["sellkit"]
