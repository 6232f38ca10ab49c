"""Seeded synthetic-input generators shared by the oracle and the GPU path.

This package holds NO arithmetic of the method (no SVT, no sketching, no
orthonormalisation, no ALM): only the counter-based random streams and the
BASELINE.json config recipes (SURVEY.md §8(d) "Generator specification") that
turn them into the input matrices. Both sides of every parity test consume the
bytes produced here; neither side imports the other.
"""
from .philox import philox4x32_10, uniform, normal, omega
from .recipes import SEED0, make_config, CONFIGS

__all__ = ["philox4x32_10", "uniform", "normal", "omega", "SEED0",
           "make_config", "CONFIGS"]
