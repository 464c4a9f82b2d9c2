"""B200-native hot path of Aurora's online speculator training (arXiv 2602.06932).

The product is libaurora.so (CUDA kernels for sm_100a behind the C-ABI in
include/aurora.h); `aurora` is its ctypes binding.
"""
from . import aurora  # noqa: F401
from .aurora import SpecTrainStep, AuroraError  # noqa: F401

__all__ = ["aurora", "SpecTrainStep", "AuroraError"]
