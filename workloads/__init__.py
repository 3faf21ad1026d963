"""Seeded synthetic input generators shared by the tests, bench.py and smoke().

This package holds none of the method's arithmetic (no transforms, tables, projection,
transport or collision): it only evaluates the paper's initial/boundary profiles at the
velocity nodes and draws seeded random numbers.  Both the CUDA path and the oracle consume
its bytes; neither imports the other.
"""
from .gen import (CONFIGS, config, initial_state, family, ghost_vectors, solid_mask,  # noqa: F401
                  reentry_inflow_velocity, reentry_inflow_ghost, ScaledField)
