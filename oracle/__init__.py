"""TEST INFRASTRUCTURE ONLY -- the independent CPU oracle for arXiv 2508.01864.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline
leg and ``--impl reference``) may import this package.  The product package
``paper_2508_01864_b200`` never imports it, and it never imports the product.
It shares no code with the CUDA path: the only common module is ``workloads``
(seeded random inputs, no arithmetic of the method).

Contents
  * ``matern_oracle.c`` -- dense O(N M) kernel sums from the closed-form Matern
    profiles in L1 / product form (L414-422), long-double
    accumulation, OpenMP over rows.
  * ``oracle.py`` -- ctypes wrapper, dense kernel blocks, and the dense GP
    pipeline (OLS, GLS, alpha, posterior mean).

Parity pins: every function is pinned in ``tests/test_oracle.py`` against values
the paper / mathematics fix (mpmath Bessel definition, geometric-series closed
forms, Kronecker identities, worked examples, brute force at 40 digits).
"""
from .oracle import *  # noqa: F401,F403
