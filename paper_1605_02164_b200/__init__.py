"""B200-native Monte Carlo Shiftable Filter (arXiv 1605.02164) -- Python binding.

The compute path is libbfvec.so (CUDA, sm_100a) behind the C ABI of
include/bfvec.h; this package only marshals arguments (torch provides device
buffers, streams and process groups). Importing it fails loudly if the
library has not been built.
"""
from . import _lib

_lib.load()

from .api import BF_W_ALIAS, BF_W_SMALL_Z, BfVecError, Plan, philox4x64_10, plan_for_config  # noqa: E402

__all__ = ["Plan", "BfVecError", "philox4x64_10", "plan_for_config", "BF_W_ALIAS", "BF_W_SMALL_Z"]
