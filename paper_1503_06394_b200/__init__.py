"""B200-native Chebyshev-Hutchinson log-determinant hot path (arXiv 1503.06394).

The compute lives in libchebld.so (include/cheb_logdet.h, csrc/); this package
is the thin Python binding (api.py) and the multi-GPU probe-sharding driver
(dist.py).  There is no CPU fallback: importing the API without the built
library raises.
"""
from .api import (DeviceCSR, Operator, Result, Estimator, coeffs_log, workspace_bytes,
                  power_moments, taylor_coeffs, taylor_logdet, affine_power_moments, norm_bound,
                  spectrum_bounds, logdet_auto,
                  alloc_workspace, moments, moments_host, finalize, logdet, logdet_host, bounds_btb, probes,
                  launch_count, profile_begin, profile_end, set_persistent, set_small_tiles, get_small_tiles, set_doubling, set_resident, get_resident, last_schedule,
                  get_doubling, release_cache, workspace_status, check_estimate, log_abs_det_from_btb, log_tau_from_rank1)
from ._lib import ChebError, load as load_library

__all__ = ["DeviceCSR", "Operator", "Result", "Estimator", "coeffs_log", "workspace_bytes",
           "power_moments", "taylor_coeffs", "taylor_logdet", "affine_power_moments", "norm_bound",
           "spectrum_bounds", "logdet_auto",
           "alloc_workspace", "moments", "moments_host", "finalize", "logdet", "logdet_host", "bounds_btb",
           "probes", "launch_count", "profile_begin", "profile_end", "set_persistent", "set_small_tiles",
           "get_small_tiles", "set_doubling", "get_doubling", "set_resident", "get_resident", "last_schedule", "release_cache", "workspace_status", "check_estimate",
           "log_abs_det_from_btb",
           "log_tau_from_rank1", "ChebError", "load_library"]
