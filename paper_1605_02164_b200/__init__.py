"""B200-native Monte Carlo Shiftable Filter (arXiv 1605.02164) -- Python binding.

The compute path is libbfvec.so (CUDA, sm_100a) behind the C ABI of
include/bfvec.h; this package only marshals arguments (torch provides device
buffers, streams and process groups). Importing it fails loudly if the
library has not been built.
"""
from . import _lib

_lib.load()

from .api import (BF_W_ALIAS, BF_W_SMALL_Z, BfVecError, Plan, lab_to_srgb, philox4x64_10,  # noqa: E402
                  plan_for_config, srgb_to_lab)

__all__ = ["Plan", "BfVecError", "philox4x64_10", "plan_for_config", "srgb_to_lab", "lab_to_srgb",
           "BF_W_ALIAS", "BF_W_SMALL_Z"]
