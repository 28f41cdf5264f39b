"""GMRF log-likelihood scan (§5.2).

For the precision family J(theta) = D + theta*O (the grid GMRF: D = I, O = -Adj) and observed
fields x_s, the Gaussian log-likelihood is

    log p(x | theta) = 1/2 log det J(theta) - 1/2 x^T J(theta) x - d/2 log(2 pi)

(the paper's display, lacks the 1/2 factors -- reading G16).  All values of theta are
estimated in ONE batched pass (cheb_family_moments): the R members ride in the columns of every
probe block, so each pass over the matrix serves all of them, and every member sees the SAME probes
(common random numbers), so differences across theta carry little Monte-Carlo noise.  The
intervals come from the device Gershgorin kernel (cheb_family_gershgorin), x^T J x = x^T D x +
theta x^T O x from cheb_quadform_split, the Chebyshev coefficients per member from cheb_coeffs_log,
Gamma_r from cheb_finalize.  The only arithmetic here is the log-likelihood formula above (finishing
scalars, like a7).
"""
import ctypes
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check
from .api import DeviceCSR, Operator, _stream_ptr, alloc_workspace, coeffs_log, finalize, check_estimate, moments, workspace_status


def quadform(A: DeviceCSR, x: torch.Tensor) -> float:
    """x^T A x on the device (deterministic)."""
    if x.dtype != torch.float64 or not x.is_cuda or x.numel() != A.n_rows:
        raise TypeError("x must be a CUDA float64 vector of length d")
    out = ctypes.c_double()
    s = A.struct()
    check(_lib.load().cheb_quadform(ctypes.byref(s), x.contiguous().data_ptr(), ctypes.byref(out),
                                    _stream_ptr()))
    return out.value


def quadform_split(A: DeviceCSR, x: torch.Tensor):
    """(x^T D x, x^T O x) for A = D + O on the device (cheb_quadform_split)."""
    if x.dtype != torch.float64 or not x.is_cuda or x.numel() != A.n_rows:
        raise TypeError("x must be a CUDA float64 vector of length d")
    out = np.empty(2)
    s = A.struct()
    check(_lib.load().cheb_quadform_split(ctypes.byref(s), x.contiguous().data_ptr(), out.ctypes.data,
                                          _stream_ptr()))
    return float(out[0]), float(out[1])


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
        """One member as its own CSR (input construction; the scan itself never builds one)."""
        val = torch.where(self.is_diag, self.base.val, self.base.val * theta)
        return DeviceCSR(self.base.n_rows, self.base.n_cols, self.base.row_ptr, self.base.col_idx, val)

    def gershgorin(self, thetas: Sequence[float]) -> np.ndarray:
        """[R][2] Gershgorin intervals of the members (cheb_family_gershgorin)."""
        th = np.ascontiguousarray(thetas, dtype=np.float64)
        lh = np.empty((th.size, 2))
        s = self.base.struct()
        check(_lib.load().cheb_family_gershgorin(ctypes.byref(s), int(th.size), th.ctypes.data, lh.ctypes.data,
                                                 _stream_ptr()))
        return lh

    def moments(self, thetas: Sequence[float], intervals: np.ndarray, degree: int, probe_begin: int,
                probe_end: int, seed: int, k: int, workspace=None, stream=None) -> torch.Tensor:
        """mu[r][p - probe_begin][j] = v_p^T T_j(Ã_r) v_p for every member in one batched pass
        (cheb_family_moments); asynchronous."""
        th = np.ascontiguousarray(thetas, dtype=np.float64)
        ab = np.ascontiguousarray(intervals, dtype=np.float64).reshape(th.size, 2)
        R = th.size
        mu = torch.empty((R, probe_end - probe_begin, degree + 1), dtype=torch.float64, device=self.base.val.device)
        if workspace is None:
            workspace = alloc_workspace(Operator("family", self.base), k)
        s = self.base.struct()
        check(_lib.load().cheb_family_moments(ctypes.byref(s), int(R), th.ctypes.data, ab.ctypes.data, int(degree),
                                              int(probe_begin), int(probe_end), int(seed) & (2 ** 64 - 1), int(k),
                                              workspace.data_ptr(), workspace.numel(), mu.data_ptr(),
                                              _stream_ptr(stream)))
        self._workspace = workspace
        return mu


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


def scan_probe_block(R: int, num_probes: int) -> int:
    """Probe block of the batched scan: R members (padded to a power of two) x up to 16 probes
    each, 16..64 columns (64-column blocks are the fastest step kernels on B200; 128 only when 33-64
    members need 2 probes each)."""
    rpad = 1 << max(0, (R - 1).bit_length())
    if 2 * rpad > 128:
        raise ValueError(f"at most 64 family members per scan (got {R})")
    cap = 64 if 2 * rpad <= 64 else 128
    kp = min(max(2, 1 << max(0, (num_probes - 1).bit_length())), 16, cap // rpad)
    return max(16, rpad * kp)


def likelihood_scan(family: PrecisionFamily, thetas: Sequence[float], xs: Sequence[torch.Tensor],
                    degree: int, num_probes: int, seed: int = 1, k: int = 0,
                    batched: Optional[bool] = None) -> ScanResult:
    """Log-likelihood of the samples xs under J(theta) for every theta: all log det J(theta) with
    common probes, device quadratic forms, device Gershgorin intervals.
    batched=True: every member in the columns of each probe block (cheb_family_moments, one pass
    over the matrix for all members); False: one estimate per member, sharing a workspace.  Default:
    separate estimates.  Since the per-step kernels read the compressed matrix copy (3 bytes per
    entry at k <= 16) the matrix bytes a batched pass shares are small, and the
    batched kernel's per-column scalars cost more than they save (configs[3]-size scan, 8 members:
    64 probes each 6.16 s batched vs 5.34 s separate, 16 probes each 1.60 s vs 1.41 s;
    profiles/r02_extras.jsonl)."""
    th = np.asarray(thetas, dtype=np.float64)
    R, d, S = th.size, family.base.n_rows, len(xs)
    if batched is None:
        batched = False
    lh = family.gershgorin(th)
    if not np.all(lh[:, 0] > 0):
        bad = th[~(lh[:, 0] > 0)]
        raise ValueError(f"J(theta) not certified positive definite by Gershgorin for theta in {bad}")
    if batched:
        k = k or scan_probe_block(R, num_probes)
        mu = family.moments(th, lh, degree, 0, num_probes, seed, k)
    else:
        k = k or next((kk for kk in (8, 16, 32, 64) if kk >= num_probes), 64)
        ws = alloc_workspace(Operator("csr", family.base), k)
        mu = torch.empty((R, num_probes, degree + 1), dtype=torch.float64, device=family.base.val.device)
        for r in range(R):
            moments(Operator("csr", family.at(float(th[r]))), lh[r, 0], lh[r, 1], degree, 0, num_probes, seed, k,
                    mu_out=mu[r], workspace=ws)
            if workspace_status(ws) & 3:  # the status word is per moments call: check each member
                raise _lib.ChebError(_lib.CL_ENONFINITE, f"moments of J({th[r]}) failed (status {workspace_status(ws)})")
        family._workspace = None
    out = {"logdet": [], "stderr": [], "quad": [], "loglik": []}
    qs = [quadform_split(family.base, x) for x in xs]
    for r in range(R):
        c = torch.from_numpy(coeffs_log(lh[r, 0], lh[r, 1], degree)).to(mu.device)
        _, stats = finalize(mu[r].contiguous(), c)
        check_estimate(stats, family._workspace if r == 0 else None)
        st = stats.cpu().numpy()
        q = sum(qd + th[r] * qo for qd, qo in qs)
        out["logdet"].append(st[0])
        out["stderr"].append(st[1])
        out["quad"].append(q)
        out["loglik"].append(0.5 * S * st[0] - 0.5 * q - 0.5 * S * d * math.log(2 * math.pi))
    return ScanResult(th, *(np.array(out[k_]) for k_ in ("logdet", "stderr", "quad", "loglik")), S)
