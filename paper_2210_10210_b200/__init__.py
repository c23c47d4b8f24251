"""B200-native (sm_100a) EFGP hot path: type-1 NUFFT -> Toeplitz CG -> type-2 NUFFT.

The computation lives in libefgp.so (include/efgp.h); this package is the thin binding.
"""
from .efgp import EFGP, EFGPError, full_to_half, half_to_full  # noqa: F401

__all__ = ["EFGP", "EFGPError", "half_to_full", "full_to_half"]
