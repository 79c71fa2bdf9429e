"""B200-native preconditioned Bi-CGSTAB Poisson hot path (arXiv 2503.08935).

The solver lives in the CUDA C-ABI library `lib/libbcgs.so` (include/bcgs.h); `bcgs` is its
ctypes binding.  There is no CPU fallback.
"""
from .bcgs import Solver, load, workspace_bytes, chebyshev_constants, nccl_unique_id  # noqa: F401

__all__ = ["Solver", "load", "workspace_bytes", "chebyshev_constants", "nccl_unique_id"]
