"""B200-native policy epoch of Nalar's global controller (arXiv 2601.05109).

The hot path (readiness / depth / doom sweep, per-workflow aggregation,
priority key, capacity-constrained assignment) runs in hand-written sm_100a
kernels inside libnalar.so behind the C ABI of include/nalar.h; ``nalar`` is
the ctypes binding with the same names.  No CPU fallback exists.
"""
from . import nalar  # noqa: F401  (raises if libnalar.so is missing)
from .nalar import Context, NalarError  # noqa: F401

__all__ = ["nalar", "Context", "NalarError"]
