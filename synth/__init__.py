"""Seeded synthetic input generators shared by the tests, smoke() and bench.py.

This package holds NO arithmetic of the method (no counting, no costs, no
partitioning).  It only draws random inputs with the shapes and distributions
of the paper's workloads (recipes in DESIGN.md "Input recipe").  Both the
CUDA path and the oracle consume its outputs; neither is imported here.
"""
from .gen import *  # noqa: F401,F403
