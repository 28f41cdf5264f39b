"""Python face of the C ABI (include/cheb_logdet.h).

PyTorch is plumbing here: it owns device memory and streams.  Every arithmetic
step of the path (probes, Chebyshev steps, reductions, accumulation, bounds)
runs in libchebld.so's CUDA kernels; this module only marshals pointers.
"""
import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import CLCsr, CLOperator, CLResult, OP_KIND, check


@dataclass
class DeviceCSR:
    """CSR resident on a CUDA device: row_ptr int64, col_idx int32, val float64."""
    n_rows: int
    n_cols: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    val: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    @classmethod
    def from_host(cls, csr, device="cuda"):
        """Upload any object with n_rows, n_cols, row_ptr, col_idx, val (numpy)."""
        return cls(int(csr.n_rows), int(csr.n_cols),
                   torch.from_numpy(np.ascontiguousarray(csr.row_ptr, dtype=np.int64)).to(device),
                   torch.from_numpy(np.ascontiguousarray(csr.col_idx, dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(csr.val, dtype=np.float64)).to(device))

    def struct(self) -> CLCsr:
        for t, dt in ((self.row_ptr, torch.int64), (self.col_idx, torch.int32), (self.val, torch.float64)):
            if t.dtype != dt or not t.is_contiguous() or not t.is_cuda:
                raise TypeError("DeviceCSR tensors must be contiguous CUDA int64/int32/float64")
        return CLCsr(self.n_rows, self.n_cols, self.nnz, self.row_ptr.data_ptr(),
                     self.col_idx.data_ptr(), self.val.data_ptr())


def _host_ptr(x, np_dtype, torch_dtype, keep):
    """Host pointer of a numpy array or a (pinned) CPU torch tensor, no copy if
    already contiguous with the right dtype."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda or x.dtype != torch_dtype or not x.is_contiguous():
            raise TypeError("host CSR tensors must be contiguous CPU tensors of the right dtype")
        keep.append(x)
        return x.data_ptr(), x.numel()
    a = np.ascontiguousarray(x, dtype=np_dtype)
    keep.append(a)
    return a.ctypes.data, a.size


def _host_csr_struct(csr, keep):
    rp, _ = _host_ptr(csr.row_ptr, np.int64, torch.int64, keep)
    ci, nnz = _host_ptr(csr.col_idx, np.int32, torch.int32, keep)
    va, _ = _host_ptr(csr.val, np.float64, torch.float64, keep)
    return CLCsr(int(csr.n_rows), int(csr.n_cols), int(nnz), rp, ci, va)


@dataclass
class Operator:
    """M = A (kind "csr"), A + c u u^T ("rank1", u None = ones), or B^T B ("btb",
    A = B, At = exact CSR of B^T)."""
    kind: str
    A: DeviceCSR
    At: Optional[DeviceCSR] = None
    c: float = 0.0
    u: Optional[torch.Tensor] = None

    @property
    def d(self) -> int:
        return self.A.n_cols

    def struct(self) -> CLOperator:
        s = CLOperator()
        s.kind = OP_KIND[self.kind]
        s.A = self.A.struct()
        if self.kind == "btb":
            if self.At is None:
                raise ValueError("btb operator needs At (CSR of B^T)")
            s.At = self.At.struct()
        s.r1_c = float(self.c)
        s.r1_u = self.u.data_ptr() if (self.kind == "rank1" and self.u is not None) else None
        return s


@dataclass
class Result:
    logdet: float          # Gamma: estimate of log det M
    stderr: float
    num_probes: int
    degree: int
    probe_block: int
    gamma_p: np.ndarray
    moments: Optional[np.ndarray]
    elapsed_s: float


def _stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def coeffs_log(a: float, b: float, degree: int) -> np.ndarray:
    """Host fp64 Chebyshev coefficients of log on [a,b] (library routine)."""
    c = np.empty(degree + 1 if degree >= 0 else 1)
    check(_lib.load().cheb_coeffs_log(float(a), float(b), int(degree), c.ctypes.data))
    return c


def workspace_bytes(op: Operator, k: int) -> int:
    L = _lib.load()
    s = op.struct()
    n = L.cheb_workspace_bytes(ctypes.byref(s), int(k))
    if n == 0:
        raise _lib.ChebError(-1, L.cheb_last_error().decode())
    return int(n)


def alloc_workspace(op: Operator, k: int) -> torch.Tensor:
    n = workspace_bytes(op, k)
    return torch.empty(n, dtype=torch.uint8, device=op.A.val.device)


def moments(op: Operator, a: float, b: float, degree: int, probe_begin: int, probe_end: int,
            seed: int, k: int, mu_out: Optional[torch.Tensor] = None,
            workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Asynchronous: mu[(p - probe_begin), j] = v_p^T T_j(Ã) v_p on the device."""
    dev = op.A.val.device
    if mu_out is None:
        mu_out = torch.empty((probe_end - probe_begin, degree + 1), dtype=torch.float64, device=dev)
    if workspace is None:
        workspace = alloc_workspace(op, k)
    s = op.struct()
    check(_lib.load().cheb_moments(ctypes.byref(s), float(a), float(b), int(degree), int(probe_begin),
                                   int(probe_end), int(seed) & (2 ** 64 - 1), int(k),
                                   workspace.data_ptr(), workspace.numel(), mu_out.data_ptr(),
                                   _stream_ptr(stream)))
    return mu_out


def power_moments(op: Operator, s: float, degree: int, probe_begin: int, probe_end: int, seed: int,
                  k: int, mu_out: Optional[torch.Tensor] = None,
                  workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Asynchronous Taylor-baseline moments mu[(p - probe_begin), j] = v_p^T (I - M/s)^j v_p."""
    dev = op.A.val.device
    if mu_out is None:
        mu_out = torch.empty((probe_end - probe_begin, degree + 1), dtype=torch.float64, device=dev)
    if workspace is None:
        workspace = alloc_workspace(op, k)
    st = op.struct()
    check(_lib.load().cheb_power_moments(ctypes.byref(st), float(s), int(degree), int(probe_begin),
                                         int(probe_end), int(seed) & (2 ** 64 - 1), int(k),
                                         workspace.data_ptr(), workspace.numel(), mu_out.data_ptr(),
                                         _stream_ptr(stream)))
    return mu_out


def affine_power_moments(op: Operator, alpha: float, beta: float, degree: int, probe_begin: int,
                         probe_end: int, seed: int, k: int, workspace: Optional[torch.Tensor] = None,
                         stream=None) -> torch.Tensor:
    """mu[(p - probe_begin), j] = v_p^T (alpha M - beta I)^j v_p on the device."""
    dev = op.A.val.device
    mu_out = torch.empty((probe_end - probe_begin, degree + 1), dtype=torch.float64, device=dev)
    if workspace is None:
        workspace = alloc_workspace(op, k)
    st = op.struct()
    check(_lib.load().cheb_affine_power_moments(ctypes.byref(st), float(alpha), float(beta), int(degree),
                                                int(probe_begin), int(probe_end), int(seed) & (2 ** 64 - 1),
                                                int(k), workspace.data_ptr(), workspace.numel(),
                                                mu_out.data_ptr(), _stream_ptr(stream)))
    return mu_out


def norm_bound(op: Operator, stream=None) -> float:
    """Device upper bound s >= lambda_max(M) (Gershgorin / ||B||_1 ||B||_inf)."""
    s = ctypes.c_double()
    st = op.struct()
    check(_lib.load().cheb_norm_bound(ctypes.byref(st), ctypes.byref(s), _stream_ptr(stream)))
    return s.value


def spectrum_bounds(op: Operator, lanczos_steps: int = 100, probes: int = 8, seed: int = 12345,
                    want_jacobi: bool = False) -> dict:
    """Spectral interval of M from the matrix (cheb_spectrum_bounds, reading
    G26): `probes` Lanczos runs of `lanczos_steps` steps on the device.  Returns lambda_min /
    lambda_max (extreme Ritz values), res_min / res_max (residual bounds), a / b (the interval to
    pass to logdet), hi_bound (device norm bound), lanczos_steps (used), and with want_jacobi the
    per-probe Lanczos tridiagonals (alpha[N], beta[N])."""
    out = _lib.CLSpectrum()
    jac = np.empty((probes, 2 * lanczos_steps)) if want_jacobi else None
    st = op.struct()
    check(_lib.load().cheb_spectrum_bounds(ctypes.byref(st), int(lanczos_steps), int(probes),
                                           int(seed) & (2 ** 64 - 1), ctypes.byref(out),
                                           jac.ctypes.data if jac is not None else None))
    r = {f: getattr(out, f) for f, _ in _lib.CLSpectrum._fields_}
    if jac is not None:
        r["jacobi"] = [(row[:lanczos_steps], row[lanczos_steps:]) for row in jac]
    return r


def logdet_auto(op: Operator, degree: int = 15, num_probes: int = 30, seed: int = 1, k: int = 0,
                lanczos_steps: int = 100, bound_probes: int = 8, want_moments: bool = False):
    """log det M without a caller-supplied interval: [a, b] from spectrum_bounds (device Lanczos),
    then the estimate (cheb_logdet).  Returns (Result, spectrum dict)."""
    sb = spectrum_bounds(op, lanczos_steps, bound_probes, seed=seed ^ 0x5DEECE66D)
    if not sb["a"] > 0.0:
        raise _lib.ChebError(_lib.CL_EINVAL, f"Lanczos lower bound not positive ({sb['a']}); pass [a, b]")
    return logdet(op, sb["a"], sb["b"], degree, num_probes, seed, k, want_moments), sb


def taylor_coeffs(s: float, degree: int) -> np.ndarray:
    c = np.empty(degree + 1)
    check(_lib.load().cheb_taylor_coeffs(float(s), int(degree), c.ctypes.data))
    return c


def taylor_logdet(op: Operator, s: float, degree: int, num_probes: int, seed: int = 1, k: int = 16):
    """Taylor-baseline estimate of log det M (scale s >= lambda_max): returns
    (Gamma, stderr, mu[m][n+1]) -- all steps on the device."""
    mu = power_moments(op, s, degree, 0, num_probes, seed, k)
    c = torch.from_numpy(taylor_coeffs(s, degree)).to(mu.device)
    gp, stats = finalize(mu, c)
    st = stats.cpu().numpy()
    return float(st[0]), float(st[1]), mu.cpu().numpy()


def finalize(mu: torch.Tensor, c: torch.Tensor, stream=None):
    """Asynchronous device accumulation: returns (gamma_p[m], stats[3]) tensors;
    stats = (Gamma, stderr, all-finite flag)."""
    m, n1 = mu.shape
    gp = torch.empty(m, dtype=torch.float64, device=mu.device)
    stats = torch.empty(3, dtype=torch.float64, device=mu.device)
    check(_lib.load().cheb_finalize(mu.data_ptr(), c.data_ptr(), int(m), int(n1 - 1), gp.data_ptr(),
                                    stats.data_ptr(), _stream_ptr(stream)))
    return gp, stats


def _result(r: CLResult, gp, mu) -> Result:
    return Result(r.logdet, r.stderr_, int(r.num_probes), int(r.degree), int(r.probe_block), gp, mu,
                  r.elapsed_s)


def logdet(op: Operator, a: float, b: float, degree: int = 15, num_probes: int = 30, seed: int = 1,
           k: int = 0, want_moments: bool = False) -> Result:
    """Synchronous estimate of log det M (cheb_logdet; device-resident operator)."""
    gp = np.empty(num_probes)
    mu = np.empty((num_probes, degree + 1)) if want_moments else None
    r = CLResult()
    r.per_probe = gp.ctypes.data
    r.moments = mu.ctypes.data if mu is not None else None
    s = op.struct()
    check(_lib.load().cheb_logdet(ctypes.byref(s), float(a), float(b), int(degree), int(num_probes),
                                  int(seed) & (2 ** 64 - 1), int(k), ctypes.byref(r)))
    return _result(r, gp, mu)


def _host_operator(kind, A, At, c, u, keep) -> CLOperator:
    s = CLOperator()
    s.kind = OP_KIND[kind]
    s.A = _host_csr_struct(A, keep)
    if kind == "btb":
        s.At = _host_csr_struct(At, keep)
    s.r1_c = float(c)
    if kind == "rank1" and u is not None:
        uu = np.ascontiguousarray(u, dtype=np.float64)
        keep.append(uu)
        s.r1_u = uu.ctypes.data
    return s


def moments_host(kind: str, A, a: float, b: float, degree: int, probe_begin: int, probe_end: int,
                 seed: int, k: int, At=None, c: float = 0.0, u: Optional[np.ndarray] = None,
                 out: Optional[np.ndarray] = None) -> np.ndarray:
    """Synchronous shard moments from HOST CSR arrays (cheb_moments_host): H2D copy of the
    operator, moments of global probes [probe_begin, probe_end), D2H of mu[rows][n+1]."""
    keep = []
    s = _host_operator(kind, A, At, c, u, keep)
    if out is None:
        out = np.empty((probe_end - probe_begin, degree + 1))
    if out.dtype != np.float64 or not out.flags.c_contiguous or out.shape != (probe_end - probe_begin, degree + 1):
        raise TypeError("out must be a C-contiguous float64 array [rows][degree+1]")
    check(_lib.load().cheb_moments_host(ctypes.byref(s), float(a), float(b), int(degree), int(probe_begin),
                                        int(probe_end), int(seed) & (2 ** 64 - 1), int(k), out.ctypes.data))
    return out


def logdet_host(kind: str, A, a: float, b: float, degree: int = 15, num_probes: int = 30,
                seed: int = 1, k: int = 0, At=None, c: float = 0.0, u: Optional[np.ndarray] = None,
                want_moments: bool = False) -> Result:
    """Synchronous estimate from HOST (numpy) CSR arrays: the library copies the
    operator to the device inside the call (cheb_logdet_host)."""
    keep = []
    s = _host_operator(kind, A, At, c, u, keep)
    gp = np.empty(num_probes)
    mu = np.empty((num_probes, degree + 1)) if want_moments else None
    r = CLResult()
    r.per_probe = gp.ctypes.data
    r.moments = mu.ctypes.data if mu is not None else None
    check(_lib.load().cheb_logdet_host(ctypes.byref(s), float(a), float(b), int(degree),
                                       int(num_probes), int(seed) & (2 ** 64 - 1), int(k),
                                       ctypes.byref(r)))
    return _result(r, gp, mu)


def bounds_btb(op: Operator, stream=None):
    """(a, b) spectral interval of B^T B from the device kernel."""
    ab = np.empty(2)
    s = op.struct()
    check(_lib.load().cheb_bounds_btb(ctypes.byref(s), ab.ctypes.data, _stream_ptr(stream)))
    return float(ab[0]), float(ab[1])


def probes(d: int, seed: int, probe_begin: int, k: int, device="cuda") -> torch.Tensor:
    """The path's probes v_p[i] for p in [probe_begin, probe_begin+k): tensor [d, k]."""
    v = torch.empty((d, k), dtype=torch.float64, device=device)
    check(_lib.load().cheb_probes(int(d), int(seed) & (2 ** 64 - 1), int(probe_begin), int(k),
                                  v.data_ptr(), _stream_ptr()))
    return v


def launch_count() -> int:
    return int(_lib.load().cheb_launch_count())


def profile_begin():
    check(_lib.load().cheb_profile_begin())


def profile_end():
    """Stop recording; returns {"single": (ms, launches), "spmm": (ms, launches),
    "persistent": (ms, launches)}: the Chebyshev step kernel, the B^T B spmm kernel (Y = B w) and
    the persistent multi-step kernel, each summed over its launches (CUDA events on the launching
    stream)."""
    L = _lib.load()
    ms, n = ctypes.c_double(), ctypes.c_int64()
    check(L.cheb_profile_end(ctypes.byref(ms), ctypes.byref(n)))
    sms, sn = ctypes.c_double(), ctypes.c_int64()
    check(L.cheb_profile_spmm(ctypes.byref(sms), ctypes.byref(sn)))
    pms, pn = ctypes.c_double(), ctypes.c_int64()
    check(L.cheb_profile_persistent(ctypes.byref(pms), ctypes.byref(pn)))
    return {"single": (ms.value, n.value), "spmm": (sms.value, sn.value),
            "persistent": (pms.value, pn.value)}


STATUS_TIMEOUT, STATUS_NONFINITE, STATUS_COMPRESSED = 1, 2, 0x100  # 0x100: informational


def workspace_status(workspace: torch.Tensor, stream=None) -> int:
    """Device status word of the last moments call that used `workspace` (cheb_workspace_status):
    bit 0 = a persistent-kernel spin wait timed out (its moments were set to NaN), bit 1 = a
    non-finite moment.  Synchronises the stream."""
    st = ctypes.c_uint32()
    check(_lib.load().cheb_workspace_status(workspace.data_ptr(), ctypes.byref(st), _stream_ptr(stream)))
    return int(st.value)


def check_estimate(stats: torch.Tensor, workspace: Optional[torch.Tensor] = None, stream=None):
    """Raise ChebError unless an estimate is valid (synchronises): CL_ECUDA if a device spin wait
    timed out, CL_ENONFINITE if any Gamma_p is not finite (stats[2] from cheb_finalize is the
    all-finite flag; the [a,b] interval likely misses the spectrum)."""
    status = workspace_status(workspace, stream) if workspace is not None else 0
    ok = float(stats[2].item()) == 1.0 and math.isfinite(float(stats[0].item()))
    if status & STATUS_TIMEOUT:
        raise _lib.ChebError(_lib.CL_ECUDA, "persistent-kernel grid wait timed out; moments set to NaN")
    if not ok or status & STATUS_NONFINITE:
        raise _lib.ChebError(_lib.CL_ENONFINITE,
                             "non-finite estimate: [a,b] likely does not enclose the spectrum")


def set_persistent(mode: int):
    """Persistent multi-step kernel (csr/rank-1): 0 off, 1 auto (default), 2 always."""
    check(_lib.load().cheb_set_persistent(int(mode)))


def set_small_tiles(mode: int):
    """Tile geometry of the Algorithm-1 kernels (cheb_set_small_tiles): 1 auto (default; 16-row
    tiles at k = 64 for L2-resident operators), 0 always the standard geometry."""
    check(_lib.load().cheb_set_small_tiles(int(mode)))


def get_small_tiles() -> int:
    return int(_lib.load().cheb_get_small_tiles())


def set_doubling(on: bool):
    """Moment-doubling schedule (cheb_set_doubling; reading G25): ceil(n/2)
    applications of Ã per probe give mu_0..mu_n via T_{2j} = 2T_j^2 - I and
    T_{2j+1} = 2T_{j+1}T_j - T_1 (symmetric operators only).  Process-wide; default off."""
    check(_lib.load().cheb_set_doubling(1 if on else 0))


def set_resident(mode: int):
    """Shared-memory-resident multi-step kernel (cheb_set_resident): 1 auto (default; csr/rank-1
    probe blocks that fit in the SMs' shared memory, in the automatic persistent mode), 0 off."""
    check(_lib.load().cheb_set_resident(int(mode)))


def get_resident() -> int:
    return int(_lib.load().cheb_get_resident())


SCHEDULES = {0: "per_step", 1: "persistent", 2: "resident"}


def last_schedule() -> str:
    """Schedule of this thread's last moments call: "per_step", "persistent" or "resident"."""
    return SCHEDULES.get(int(_lib.load().cheb_last_schedule()), "none")


def release_cache():
    """Free this thread's device arenas of cheb_logdet / cheb_logdet_host."""
    check(_lib.load().cheb_release_cache())


def get_doubling() -> bool:
    return bool(_lib.load().cheb_get_doubling())


class Estimator:
    """Reusable device state for repeated estimates on one operator (bench,
    multi-GPU driver): workspace, coefficients and moment buffer stay resident."""

    def __init__(self, op: Operator, a: float, b: float, degree: int, num_probes: int,
                 k: int, seed: int = 1, probe_begin: int = 0, probe_end: Optional[int] = None,
                 basis: str = "chebyshev"):
        """basis "chebyshev" (the paper's estimator) or "taylor" (the Fig. 1(d) baseline,
        scale s = a + b)."""
        if basis not in ("chebyshev", "taylor"):
            raise ValueError("basis must be 'chebyshev' or 'taylor'")
        self.op, self.a, self.b, self.degree, self.k, self.seed = op, a, b, degree, k, seed
        self.basis = basis
        self.m = num_probes
        self.probe_begin = probe_begin
        self.probe_end = num_probes if probe_end is None else probe_end
        dev = op.A.val.device
        self.workspace = alloc_workspace(op, k)
        c = coeffs_log(a, b, degree) if basis == "chebyshev" else taylor_coeffs(a + b, degree)
        self.c = torch.from_numpy(c).to(dev)
        self.mu = torch.zeros((num_probes, degree + 1), dtype=torch.float64, device=dev)

    def enqueue_moments(self, stream=None):
        """Fill this shard's rows [probe_begin, probe_end) of mu (others untouched)."""
        if self.probe_end > self.probe_begin:
            rows = self.mu[self.probe_begin:self.probe_end]
            if self.basis == "chebyshev":
                moments(self.op, self.a, self.b, self.degree, self.probe_begin, self.probe_end, self.seed,
                        self.k, mu_out=rows, workspace=self.workspace, stream=stream)
            else:
                power_moments(self.op, self.a + self.b, self.degree, self.probe_begin, self.probe_end,
                              self.seed, self.k, mu_out=rows, workspace=self.workspace, stream=stream)
        return self.mu

    def enqueue_finalize(self, stream=None):
        return finalize(self.mu, self.c, stream=stream)

    def run(self, stream=None, check: bool = False):
        """Enqueue one whole estimate; returns device (gamma_p, stats).  check=True synchronises and
        raises ChebError on a device timeout or a non-finite estimate (check_estimate)."""
        self.enqueue_moments(stream)
        gp, stats = self.enqueue_finalize(stream)
        if check:
            self.check(stats, stream)
        return gp, stats

    def check(self, stats, stream=None):
        """Raise ChebError if the estimate behind `stats` is invalid (synchronises)."""
        check_estimate(stats, self.workspace, stream)

    def capture(self):
        """Capture one whole estimate (operator prep, probe init, every step launch, finalize) into
        a CUDA graph; returns (replay, gamma_p, stats): replay() re-runs it with one launch call on
        the capture stream's successors and refreshes gamma_p / stats in place.  Useful when many
        small estimates are served (launch gaps dominate below ~1 ms per estimate); the schedule
        switches (persistent / small tiles / doubling) in effect at capture time are baked in.  The
        captured sequence performs no host synchronisation (cheb_moments never synchronises), so
        every schedule is capturable; check a replay's stats with check()."""
        s = torch.cuda.Stream(device=self.mu.device)
        s.wait_stream(torch.cuda.current_stream(self.mu.device))
        with torch.cuda.stream(s):
            self.run(s)  # warm-up outside the capture: kernel attributes, lazy module loading
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gp, stats = self.run(s)

        def replay():
            g.replay()
            return gp, stats

        self._graph = g  # keep the graph (and its memory pool) alive with the estimator
        return replay, gp, stats


def log_abs_det_from_btb(gamma: float) -> float:
    """Alg. 2: log|det B| = 1/2 log det B^T B ([a,b] form: the
    d log(s) shift is already inside c_0)."""
    return 0.5 * gamma


def log_tau_from_rank1(gamma: float, c: float, n_vertices: int) -> float:
    """Spanning trees via M = L + c 11^T: log tau = log det M - log(c N^2)."""
    return gamma - math.log(c * n_vertices * n_vertices)
