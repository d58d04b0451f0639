"""B200-native EARL data dispatcher (arXiv 2510.05943): layout-aware decentralized dispatch of
variable-length RL batches between parallel layouts.

Modules:
  earl       -- ctypes binding of libearl_dispatch.so (include/earl_dispatch.h); no CPU fallback
  dispatch   -- user-facing helpers (torch tensors in, torch tensors out) over the binding
  workloads  -- seeded synthetic inputs shared by tests and bench.py (no dispatch arithmetic)
  build      -- nvcc build of the CUDA library for sm_100a
"""
__version__ = "0.1.0"
