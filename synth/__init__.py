"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no forward/backward, no schedule,
no balancer).  It only describes the BASELINE.json model configurations as plain
data (layer lists) and draws seeded random inputs and parameters.
Both sides -- `oracle/` and the CUDA path -- receive these arrays as data.
"""
