"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, fp64 CPU implementation of the Chebyshev-Hutchinson log-det
estimator (arXiv 1503.06394, Algorithm 1/2 in [a,b] form), written from the
paper (§2.1-§3.2) and pinned by tests/test_oracle_pins.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import anything under oracle/.  The product path
(paper_1503_06394_b200) never imports it and shares no code with it.
"""
from .runner import (Op, build_oracle, lib, cheb_nodes, coeffs_from_values,
                     coeffs_log, cheb_eval, splitmix64, rademacher, apply_tilde,
                     moments_vec, moments, logdet, bounds_btb, gamma_from_moments,
                     taylor_coeffs, power_moments_vec, taylor_logdet, affine_power_moments,
                     affine_power_moments_vec, gershgorin, quadform,
                     lanczos, ritz, spectrum_bounds)

__all__ = ["Op", "build_oracle", "lib", "cheb_nodes", "coeffs_from_values",
           "coeffs_log", "cheb_eval", "splitmix64", "rademacher", "apply_tilde",
           "moments_vec", "moments", "logdet", "bounds_btb", "gamma_from_moments",
           "taylor_coeffs", "power_moments_vec", "taylor_logdet", "affine_power_moments",
           "affine_power_moments_vec", "gershgorin", "quadform",
           "lanczos", "ritz", "spectrum_bounds"]
