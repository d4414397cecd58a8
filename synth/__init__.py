"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This package holds NO arithmetic of the RAIRS method (no assignment, no PQ, no
LUT, no scoring). It only draws base/query vectors with the shapes and value
distributions of BASELINE.json's configs.
"""
from .generators import CONFIGS, GPU_KINDS, ConfigSpec, make_dataset, get_config  # noqa: F401
