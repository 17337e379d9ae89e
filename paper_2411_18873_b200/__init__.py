"""B200-native scoring hot path of arXiv 2411.18873 (energy-aware schedule search).

The product is the C-ABI shared library ``lib/libetune_cuda.so`` (include/etune_cuda.h),
built from ``csrc/`` for sm_100a.  ``capi`` is a thin ctypes binding for Python callers.
"""
from . import capi  # noqa: F401

__all__ = ["capi"]
