"""B200-native weighted-Gaussian row-wise IGA assembly (arXiv 1710.01048).

The product is the CUDA/C++ library ``libwgq.so`` (C-ABI in ``include/wgq.h``);
``wgq`` is its thin ctypes binding and ``api`` the tensor-level convenience layer
(allocation, slabs, streams) on top of it.
"""
from . import wgq  # noqa: F401
