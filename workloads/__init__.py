"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no kernel, no scan, no solver):
only numpy PCG64 draws shaped like the configs of BASELINE.json and the
paper's simulated workloads (PAPER.md L721-724 [§3.1]: x ~ U[0,1]^d), plus the
seeded row sampler used to check large-N outputs.  See DESIGN.md "Input recipe".
"""
from .synth import *  # noqa: F401,F403
