"""B200-native coefficient-domain multi-Gabor matching pursuit (arXiv 2202.12380).

The product is libmpgabor.so (CUDA, sm_100a) behind the C ABI in
include/mpgabor.h; ``mpgabor`` is its thin ctypes binding.
"""
from .build import build_library, LIB_PATH  # noqa: F401
