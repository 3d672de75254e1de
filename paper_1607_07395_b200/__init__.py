"""B200-native hot path of Cascaded Bilateral Sampling (CABS, arXiv 1607.07395).

libcabs.so (hand-written sm_100a CUDA behind the C ABI in include/cabs.h) runs
every step; this package is the thin Python binding (`cabs`), the multi-GPU
plumbing (`dist`) and the Algorithm-2 driver (`pipeline`).
"""
from . import cabs  # noqa: F401
from .cabs import CabsError, load  # noqa: F401

__all__ = ["cabs", "CabsError", "load"]
