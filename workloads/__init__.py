"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no phases, no kernels, no
filtering). It only builds the five BASELINE.json configurations: the filter
parameters (sigma_s, C, N, M, seed) and the synthetic images that stand in for
the paper's Dome / Peppers / House photographs,
which are not available here. See DESIGN.md "Input recipe".
"""
from .configs import CONFIGS, Config, get_config, make_image, make_image_rows  # noqa: F401
