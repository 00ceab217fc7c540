"""B200-native Yin-Yang AC direction-splitting time step (arXiv 1905.02300).

Thin ctypes binding over the C ABI of ``include/yy.h`` (``libyy.so``, built for
sm_100a by ``csrc/build.sh``).  Argument marshalling only: every step of the
hot path runs in the CUDA kernels of ``csrc/``.  There is no CPU fallback —
importing :mod:`paper_1905_02300_b200.yy` raises if the library is missing.
"""
from .yy import (YY_CHI, YY_FIXED_ITERS, YY_MAX_ITERS, YY_SCHWARZ, YYError, Shell, lib_path,  # noqa: F401
                 load_library, nccl_unique_id, use_torch_allocator)

__all__ = ["Shell", "YYError", "load_library", "lib_path", "nccl_unique_id", "use_torch_allocator", "YY_CHI", "YY_MAX_ITERS", "YY_FIXED_ITERS", "YY_SCHWARZ"]
