"""Python runner for the C oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

ctypes marshalling around oracle/cheb_oracle.c plus a process pool that runs one
probe per task (single-threaded workers).  The only arithmetic
done in Python is the final ascending sum over probes (Algorithm 1 line
"Gamma <- Gamma + v^T u / m", reading G7) and the sample standard error.
"""
import ctypes
import math
import multiprocessing as mp
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cheb_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

OP_KIND = {"csr": 0, "rank1": 1, "btb": 2}


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with plain gcc (-O2 -ffp-contract=off, no SIMD intrinsics)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-std=c11", "-D_GNU_SOURCE", "-shared", "-fPIC",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class _CSR(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p),
                ("val", ctypes.c_void_p)]


class _OP(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("A", _CSR), ("r1_c", ctypes.c_double),
                ("r1_u", ctypes.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build_oracle())
        D, I32, I64, U64, P = (ctypes.c_double, ctypes.c_int32, ctypes.c_int64,
                               ctypes.c_uint64, ctypes.c_void_p)
        L.orc_cheb_nodes.argtypes = [I32, P]
        L.orc_cheb_coeffs_from_values.argtypes = [I32, P, P]
        L.orc_cheb_coeffs_log.argtypes = [D, D, I32, P]
        L.orc_cheb_coeffs_log.restype = I32
        L.orc_cheb_eval.argtypes = [I32, P, D]
        L.orc_cheb_eval.restype = D
        L.orc_splitmix64.argtypes = [U64, U64]
        L.orc_splitmix64.restype = U64
        L.orc_rademacher.argtypes = [U64, I64, I64, P]
        L.orc_apply_tilde.argtypes = [ctypes.POINTER(_OP), D, D, P, P]
        L.orc_apply_tilde.restype = I32
        L.orc_moments_vec.argtypes = [ctypes.POINTER(_OP), D, D, I32, P, P]
        L.orc_moments_vec.restype = I32
        L.orc_moments_probe.argtypes = [ctypes.POINTER(_OP), D, D, I32, U64, I64, P]
        L.orc_moments_probe.restype = I32
        L.orc_gamma_probe.argtypes = [I32, P, P]
        L.orc_gamma_probe.restype = D
        L.orc_bounds_btb.argtypes = [ctypes.POINTER(_CSR), P, P]
        L.orc_bounds_btb.restype = I32
        L.orc_taylor_coeffs.argtypes = [D, I32, P]
        L.orc_taylor_coeffs.restype = I32
        L.orc_power_moments_vec.argtypes = [ctypes.POINTER(_OP), D, I32, P, P]
        L.orc_power_moments_vec.restype = I32
        L.orc_power_moments_probe.argtypes = [ctypes.POINTER(_OP), D, I32, U64, I64, P]
        L.orc_power_moments_probe.restype = I32
        L.orc_affine_power_moments_vec.argtypes = [ctypes.POINTER(_OP), D, D, I32, P, P]
        L.orc_affine_power_moments_vec.restype = I32
        L.orc_affine_power_moments_probe.argtypes = [ctypes.POINTER(_OP), D, D, I32, U64, I64, P]
        L.orc_affine_power_moments_probe.restype = I32
        L.orc_gershgorin.argtypes = [ctypes.POINTER(_CSR)]
        L.orc_gershgorin.restype = D
        L.orc_quadform.argtypes = [ctypes.POINTER(_CSR), P]
        L.orc_quadform.restype = D
        L.orc_lanczos_tilde.argtypes = [ctypes.POINTER(_OP), D, D, I32, P, P, P]
        L.orc_lanczos_tilde.restype = I32
        L.orc_lanczos_probe.argtypes = [ctypes.POINTER(_OP), D, D, I32, U64, I64, P, P]
        L.orc_lanczos_probe.restype = I32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Op:
    """Operator M in one of the three modes (SURVEY §8 preamble).

    kind "csr": M = A; "rank1": M = A + c u u^T (u None = all ones);
    "btb": M = B^T B with B = A (the oracle applies B^T by scatter and never
    uses a transpose CSR).
    """
    kind: str
    A: object            # workloads.CSR (duck-typed: n_rows, n_cols, row_ptr, col_idx, val)
    c: float = 0.0
    u: Optional[np.ndarray] = None

    @property
    def d(self) -> int:
        return int(self.A.n_cols)

    def _struct(self):
        A = self.A
        self._keep = [np.ascontiguousarray(A.row_ptr, dtype=np.int64),
                      np.ascontiguousarray(A.col_idx, dtype=np.int32),
                      np.ascontiguousarray(A.val, dtype=np.float64)]
        uptr = None
        if self.u is not None:
            self._keep.append(np.ascontiguousarray(self.u, dtype=np.float64))
            uptr = _ptr(self._keep[-1])
        cs = _CSR(A.n_rows, A.n_cols, _ptr(self._keep[0]), _ptr(self._keep[1]),
                  _ptr(self._keep[2]))
        return _OP(OP_KIND[self.kind], cs, float(self.c), uptr)


def cheb_nodes(n: int) -> np.ndarray:
    x = np.empty(n + 1)
    lib().orc_cheb_nodes(n, _ptr(x))
    return x


def coeffs_from_values(fx: np.ndarray) -> np.ndarray:
    fx = np.ascontiguousarray(fx, dtype=np.float64)
    n = fx.size - 1
    c = np.empty(n + 1)
    lib().orc_cheb_coeffs_from_values(n, _ptr(fx), _ptr(c))
    return c


def coeffs_log(a: float, b: float, n: int) -> np.ndarray:
    c = np.empty(max(n, 0) + 1)
    rc = lib().orc_cheb_coeffs_log(a, b, n, _ptr(c))
    if rc != 0:
        raise ValueError(f"orc_cheb_coeffs_log rc={rc}")
    return c


def cheb_eval(c: np.ndarray, x: float) -> float:
    c = np.ascontiguousarray(c, dtype=np.float64)
    return lib().orc_cheb_eval(c.size - 1, _ptr(c), float(x))


def splitmix64(seed: int, t: int) -> int:
    return int(lib().orc_splitmix64(seed, t))


def rademacher(seed: int, p: int, d: int) -> np.ndarray:
    v = np.empty(d)
    lib().orc_rademacher(seed, p, d, _ptr(v))
    return v


def apply_tilde(op: Op, a: float, b: float, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(op.d)
    s = op._struct()
    rc = lib().orc_apply_tilde(ctypes.byref(s), a, b, _ptr(x), _ptr(y))
    if rc != 0:
        raise RuntimeError(f"orc_apply_tilde rc={rc}")
    return y


def moments_vec(op: Op, a: float, b: float, n: int, v: np.ndarray) -> np.ndarray:
    """mu_j = v^T T_j(Ã) v, j = 0..n, for an explicit probe vector v."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    mu = np.empty(n + 1)
    s = op._struct()
    rc = lib().orc_moments_vec(ctypes.byref(s), a, b, n, _ptr(v), _ptr(mu))
    if rc not in (0, -5):
        raise RuntimeError(f"orc_moments_vec rc={rc}")
    return mu


def taylor_coeffs(s: float, n: int) -> np.ndarray:
    c = np.empty(n + 1)
    if lib().orc_taylor_coeffs(s, n, _ptr(c)) != 0:
        raise ValueError("orc_taylor_coeffs")
    return c


def power_moments_vec(op: Op, s: float, n: int, v: np.ndarray) -> np.ndarray:
    """mu_k = v^T (I - M/s)^k v, k = 0..n (Taylor baseline)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    mu = np.empty(n + 1)
    st = op._struct()
    rc = lib().orc_power_moments_vec(ctypes.byref(st), s, n, _ptr(v), _ptr(mu))
    if rc not in (0, -5):
        raise RuntimeError(f"orc_power_moments_vec rc={rc}")
    return mu


# ---- probe-parallel pool (fork start method shares the CSR copy-on-write) ----
_G = {}


def _probe_task(p):
    op, a, b, n, seed, power = _G["args"]
    mu = np.empty(n + 1)
    s = op._struct()
    if power:
        rc = lib().orc_power_moments_probe(ctypes.byref(s), a, n, seed, int(p), _ptr(mu))
    else:
        rc = lib().orc_moments_probe(ctypes.byref(s), a, b, n, seed, int(p), _ptr(mu))
    if rc not in (0, -5):
        raise RuntimeError(f"oracle moments rc={rc}")
    return mu


def moments(op: Op, a: float, b: float, n: int, seed: int, probes: Sequence[int],
            workers: Optional[int] = None, power: bool = False) -> np.ndarray:
    """mu[len(probes)][n+1] for Rademacher probes with the given GLOBAL indices.
    power=True: Taylor-baseline power moments with scale s = a (b ignored)."""
    probes = [int(p) for p in probes]
    workers = workers or 1
    workers = max(1, min(workers, len(probes)))
    lib()
    _G["args"] = (op, a, b, n, seed, power)
    if workers == 1:
        rows = [_probe_task(p) for p in probes]
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(workers) as pool:
            rows = pool.map(_probe_task, probes, chunksize=1)
    _G.clear()
    return np.array(rows).reshape(len(probes), n + 1)


def gamma_from_moments(c: np.ndarray, mu: np.ndarray):
    """Gamma_p = sum_j c_j mu_{p,j} (ascending j, in C); Gamma = (sum_p Gamma_p)/m
    ascending p; stderr = sample sd / sqrt(m)."""
    c = np.ascontiguousarray(c, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    m, n1 = mu.shape
    gp = np.array([lib().orc_gamma_probe(n1 - 1, _ptr(c), _ptr(mu[p])) for p in range(m)])
    s = 0.0
    for g in gp:
        s += float(g)
    gamma = s / m
    if m > 1:
        var = 0.0
        for g in gp:
            var += (float(g) - gamma) ** 2
        stderr = math.sqrt(var / (m - 1)) / math.sqrt(m)
    else:
        stderr = 0.0
    return gamma, gp, stderr


def logdet(op: Op, a: float, b: float, n: int, m: int, seed: int,
           workers: Optional[int] = None, probe_begin: int = 0):
    """Algorithm 1 ([a,b] form) over probes probe_begin..probe_begin+m-1.
    Returns dict(gamma, gamma_p, stderr, mu, c)."""
    c = coeffs_log(a, b, n)
    mu = moments(op, a, b, n, seed, range(probe_begin, probe_begin + m), workers)
    gamma, gp, se = gamma_from_moments(c, mu)
    return {"gamma": gamma, "gamma_p": gp, "stderr": se, "mu": mu, "c": c}


def affine_power_moments(op: Op, alpha: float, beta: float, n: int, seed: int,
                         probes: Sequence[int]) -> np.ndarray:
    """mu[p][j] = v_p^T (alpha M - beta I)^j v_p for Rademacher probes (block power iteration)."""
    out = []
    st = op._struct()
    for p in probes:
        mu = np.empty(n + 1)
        rc = lib().orc_affine_power_moments_probe(ctypes.byref(st), alpha, beta, n, seed, int(p), _ptr(mu))
        if rc != 0:
            raise RuntimeError(f"orc_affine_power_moments_probe rc={rc}")
        out.append(mu)
    return np.array(out)


def affine_power_moments_vec(op: Op, alpha: float, beta: float, n: int, v: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float64)
    mu = np.empty(n + 1)
    st = op._struct()
    if lib().orc_affine_power_moments_vec(ctypes.byref(st), alpha, beta, n, _ptr(v), _ptr(mu)) != 0:
        raise RuntimeError("orc_affine_power_moments_vec")
    return mu


def gershgorin(A) -> float:
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_idx, dtype=np.int32)
    va = np.ascontiguousarray(A.val, dtype=np.float64)
    cs = _CSR(A.n_rows, A.n_cols, _ptr(rp), _ptr(ci), _ptr(va))
    return float(lib().orc_gershgorin(ctypes.byref(cs)))


def quadform(A, x: np.ndarray) -> float:
    """x^T A x (compensated)."""
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_idx, dtype=np.int32)
    va = np.ascontiguousarray(A.val, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    cs = _CSR(A.n_rows, A.n_cols, _ptr(rp), _ptr(ci), _ptr(va))
    return float(lib().orc_quadform(ctypes.byref(cs), _ptr(x)))


def taylor_logdet(op: Op, s: float, n: int, m: int, seed: int, workers: Optional[int] = None):
    """Taylor baseline over probes 0..m-1: dict(gamma, gamma_p, stderr, mu, c)."""
    c = taylor_coeffs(s, n)
    mu = moments(op, s, 0.0, n, seed, range(m), workers, power=True)
    gamma, gp, se = gamma_from_moments(c, mu)
    return {"gamma": gamma, "gamma_p": gp, "stderr": se, "mu": mu, "c": c}


def bounds_btb(B) -> tuple:
    """(a, b) = (Johnson sigma_min bound^2, ||B||_1 ||B||_inf) -- P:300-310."""
    rp = np.ascontiguousarray(B.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(B.col_idx, dtype=np.int32)
    va = np.ascontiguousarray(B.val, dtype=np.float64)
    cs = _CSR(B.n_rows, B.n_cols, _ptr(rp), _ptr(ci), _ptr(va))
    a = np.empty(1)
    b = np.empty(1)
    rc = lib().orc_bounds_btb(ctypes.byref(cs), _ptr(a), _ptr(b))
    if rc != 0:
        raise ValueError(f"orc_bounds_btb rc={rc} (Johnson bound not positive?)")
    return float(a[0]), float(b[0])


# ---- spectral interval by Lanczos (reading G26) ----
def lanczos(op: Op, a: float, b: float, N: int, v: np.ndarray = None, seed: int = None, p: int = None):
    """N Lanczos steps on Ã = alpha M - beta I ([a,b] map) with full re-orthogonalisation from the
    start vector v (or the Rademacher probe p of `seed`): returns (alpha[N], beta[N]) -- the Jacobi
    matrix T_N (diagonal alpha, off-diagonal beta[:-1]) and the residual factor beta[N-1]."""
    al, be = np.empty(N), np.empty(N)
    st = op._struct()
    if v is not None:
        v = np.ascontiguousarray(v, dtype=np.float64)
        rc = lib().orc_lanczos_tilde(ctypes.byref(st), a, b, N, _ptr(v), _ptr(al), _ptr(be))
    else:
        rc = lib().orc_lanczos_probe(ctypes.byref(st), a, b, N, seed, p, _ptr(al), _ptr(be))
    if rc <= -100:  # invariant subspace after -rc - 100 steps: T_j is exact (beta_j = 0)
        j = -rc - 100
        return al[:j], be[:j]
    if rc != 0:
        raise RuntimeError(f"orc_lanczos rc={rc}")
    return al, be


def ritz(alpha: np.ndarray, beta: np.ndarray):
    """Ritz values theta (ascending) of T_N and their residual bounds beta_N |s_N| (an eigenvalue of
    Ã lies within the bound of each theta), by numpy's symmetric eigensolver."""
    N = alpha.size
    T = np.diag(alpha) + np.diag(beta[:N - 1], 1) + np.diag(beta[:N - 1], -1)
    th, S = np.linalg.eigh(T)
    return th, beta[N - 1] * np.abs(S[N - 1, :])


def spectrum_bounds(op: Op, lo: float, hi: float, N: int, seed: int, probes: Sequence[int]):
    """Interval [a, b] for the estimator from Lanczos on each probe, in M-space (lambda = (theta +
    beta)/alpha for the map of [lo, hi]): a = min_p (theta_min - r_min) / ..., b = min(max_p
    (theta_max + r_max), hi); also the extreme Ritz values and residuals themselves."""
    alpha, beta = 2.0 / (hi - lo), (hi + lo) / (hi - lo)
    lmin, lmax, rmin, rmax, rows = np.inf, -np.inf, 0.0, 0.0, []
    for p in probes:
        al, be = lanczos(op, lo, hi, N, seed=seed, p=p)
        th, r = ritz(al, be)
        rows.append((al, be))
        if (th[0] + beta) / alpha < lmin:
            lmin, rmin = (th[0] + beta) / alpha, r[0] / alpha
        if (th[-1] + beta) / alpha > lmax:
            lmax, rmax = (th[-1] + beta) / alpha, r[-1] / alpha
    return {"lambda_min": lmin, "lambda_max": lmax, "res_min": rmin, "res_max": rmax,
            "a": max(lmin - rmin, 0.0), "b": min(lmax + rmax, hi), "jacobi": rows}
