"""B200-native HugeCTR sparse-embedding hot path (arXiv 2210.08803).

The product is libhps_gpu.so (hand-written sm_100a CUDA behind the C-ABI in
include/hps_gpu.h). This package is its Python host mirror: ctypes binding
(_lib), torch-memory API (api), placement planners (placement), multi-GPU
orchestration (sharded) and the synthetic workload generators (workload).
"""
from ._lib import HpsError, load  # noqa: F401
from .api import Context, DistTable, EmbeddingTableGroup, HotCache, opt_params  # noqa: F401

__all__ = ["Context", "DistTable", "EmbeddingTableGroup", "HotCache", "HpsError", "load", "opt_params"]
