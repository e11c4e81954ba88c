"""Seeded synthetic inputs shared by the tests, bench.py and smoke().

This module holds NONE of the method's arithmetic: it only draws Q, K, V (and
selection targets) with the shapes and value structure of the paper's
workloads (DESIGN.md §5 "Input recipe").  Both the CUDA path and the oracle are
fed the same tensors from here; neither side imports the other.
"""

from .synth import (
    Layout, CONFIGS, layout_for, sharpness, generate_qkv, step_seed, random_masses,
)

__all__ = ["Layout", "CONFIGS", "layout_for", "sharpness", "generate_qkv", "step_seed",
           "random_masses"]
