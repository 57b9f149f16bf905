"""B200-native exhaustive launch-order evaluation (arXiv 1511.07983).

The product path is ``librk.so`` (C-ABI declared in ``include/rk.h``: host
validation, Algorithm 1, rank/unrank, and the sm_100a CUDA kernels) plus the
thin ctypes binding in :mod:`paper_1511_07983_b200.rk`.  Nothing here imports
the oracle; there is no CPU fallback for any compute call.
"""
__all__ = ["rk", "workloads", "dist"]
