"""GMRF log-likelihood scan (§5.2).

For the precision family J(theta) = D + theta*O (the grid GMRF: D = I, O = -Adj) and an
observed field x, the Gaussian log-likelihood is

    log p(x | theta) = 1/2 log det J(theta) - 1/2 x^T J(theta) x - d/2 log(2 pi)

(the paper's display, lacks the 1/2 factors -- reading G16).  Each log det is a
Chebyshev-Hutchinson estimate on the device; every theta uses the SAME probes (same seed:
common random numbers), so differences across theta carry little Monte-Carlo noise.
Every arithmetic step runs in libchebld.so kernels: J(theta)'s values are built on the
device from the base pattern (input construction), the interval comes from the device
Gershgorin kernel, x^T J x from cheb_quadform.
"""
import ctypes
import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check
from .api import DeviceCSR, Estimator, Operator, _stream_ptr


def quadform(A: DeviceCSR, x: torch.Tensor) -> float:
    """x^T A x on the device (deterministic)."""
    if x.dtype != torch.float64 or not x.is_cuda or x.numel() != A.n_rows:
        raise TypeError("x must be a CUDA float64 vector of length d")
    out = ctypes.c_double()
    s = A.struct()
    check(_lib.load().cheb_quadform(ctypes.byref(s), x.contiguous().data_ptr(), ctypes.byref(out),
                                    _stream_ptr()))
    return out.value


def gershgorin(A: DeviceCSR):
    """(lo, hi) Gershgorin interval of a symmetric device CSR."""
    lh = np.empty(2)
    s = A.struct()
    check(_lib.load().cheb_gershgorin(ctypes.byref(s), lh.ctypes.data, _stream_ptr()))
    return float(lh[0]), float(lh[1])


class PrecisionFamily:
    """J(theta) = D + theta*O on a fixed sparsity pattern: `base` holds D on the diagonal
    and O off the diagonal (for the grid GMRF: base = I - Adj, J(theta) = I - theta*Adj)."""

    def __init__(self, base: DeviceCSR):
        self.base = base
        rows = torch.repeat_interleave(torch.arange(base.n_rows, device=base.val.device),
                                       base.row_ptr[1:] - base.row_ptr[:-1])
        self.is_diag = rows == base.col_idx.to(torch.int64)

    def at(self, theta: float) -> DeviceCSR:
        val = torch.where(self.is_diag, self.base.val, self.base.val * theta)
        return DeviceCSR(self.base.n_rows, self.base.n_cols, self.base.row_ptr, self.base.col_idx, val)


@dataclass
class ScanResult:
    thetas: np.ndarray
    logdet: np.ndarray     # estimates of log det J(theta)
    stderr: np.ndarray
    quad: np.ndarray       # sum over samples of x^T J(theta) x
    loglik: np.ndarray     # sum over samples of log p(x_r | theta)
    n_samples: int

    @property
    def argmax(self) -> float:
        return float(self.thetas[int(np.argmax(self.loglik))])


def likelihood_scan(family: PrecisionFamily, thetas: Sequence[float], xs: Sequence[torch.Tensor],
                    degree: int, num_probes: int, seed: int = 1, k: int = 0) -> ScanResult:
    """Log-likelihood of the samples xs under J(theta) for every theta (common probes)."""
    d = family.base.n_rows
    k = k or next((kk for kk in (8, 16, 32, 64) if kk >= num_probes), 64)
    R = len(xs)
    out = {"logdet": [], "stderr": [], "quad": [], "loglik": []}
    for th in thetas:
        J = family.at(float(th))
        a, b = gershgorin(J)
        if not a > 0:
            raise ValueError(f"J({th}) not certified positive definite by Gershgorin (lo={a})")
        est = Estimator(Operator("csr", J), a, b, degree, num_probes, k, seed)
        _, stats = est.run(check=True)  # raises on a device timeout / non-finite estimate
        st = stats.cpu().numpy()
        q = sum(quadform(J, x) for x in xs)
        out["logdet"].append(st[0])
        out["stderr"].append(st[1])
        out["quad"].append(q)
        out["loglik"].append(0.5 * R * st[0] - 0.5 * q - 0.5 * R * d * math.log(2 * math.pi))
    return ScanResult(np.asarray(thetas, dtype=float), *(np.array(out[k_]) for k_ in
                                                          ("logdet", "stderr", "quad", "loglik")), R)
