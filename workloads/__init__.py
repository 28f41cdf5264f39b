"""Seeded synthetic inputs for the Chebyshev-Hutchinson log-det hot path.

This package is shared by the CUDA path's tests/bench and by the oracle's tests.
It only *builds inputs* (CSR matrices, workload parameters).  It contains none of
the method's arithmetic: no Chebyshev coefficients, no probes, no recurrence, no
spectral-bound estimation.  See DESIGN.md "Input recipe".
"""
from .csr import CSR, transpose, to_dense
from .generators import (grid_gmrf, torus_laplacian, random_nonsingular,
                         triangular_b, complete_graph_laplacian, random_spd,
                         splitmix64_at)
from .configs import CONFIGS, Workload, get_workload

__all__ = ["CSR", "transpose", "to_dense", "grid_gmrf", "torus_laplacian",
           "random_nonsingular", "triangular_b", "complete_graph_laplacian",
           "random_spd", "splitmix64_at", "CONFIGS", "Workload", "get_workload"]
