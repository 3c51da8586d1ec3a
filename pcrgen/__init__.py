"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the PCR method (no hashing, no tree policy,
no attention).  It only draws seeded random numbers and packs them into the
shapes of the paper's workloads.  bf16 values are
produced by round-to-nearest-even from fp32 and carried as uint16 bit patterns,
so both sides of a parity test see bit-identical inputs.
"""
from .synth import *  # noqa: F401,F403
