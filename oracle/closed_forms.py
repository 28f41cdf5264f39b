"""Closed forms used to PIN the oracle (TEST INFRASTRUCTURE ONLY).

These are mathematical facts independent of the estimator:
* eigenvalues of the grid GMRF precision I - theta*Adj (free boundary):
  1 - 2 theta (cos(pi i/(N+1)) + cos(pi j/(N+1))), i,j = 1..N
  (Adj of the path P_N has eigenvalues 2cos(pi k/(N+1)); grid = P_N (+) P_N);
* eigenvalues of the N x N torus Laplacian: 4 - 2cos(2 pi i/N) - 2cos(2 pi j/N);
* the matrix-tree theorem: tau(G) = (1/|V|) prod of non-zero
  Laplacian eigenvalues;
* Cayley: tau(K_n) = n^(n-2);
* the Chebyshev series of log(x + c), c > 1:
  log(x+c) = log(rho/2) + sum_k 2(-1)^(k+1) rho^(-k)/k T_k(x), rho = c + sqrt(c^2-1);
* T_j(x) = cos(j arccos x) on [-1,1] (and cosh form outside).
"""
import math

import numpy as np


def grid_eigs(N: int, theta: float, M: int = None) -> np.ndarray:
    M = N if M is None else M
    ci = np.cos(np.pi * np.arange(1, N + 1) / (N + 1))
    cj = np.cos(np.pi * np.arange(1, M + 1) / (M + 1))
    return (1.0 - 2.0 * theta * (ci[:, None] + cj[None, :])).reshape(-1)


def grid_logdet(N: int, theta: float, M: int = None) -> float:
    """Exact log det(I - theta Adj) via fsum of log of closed-form eigenvalues
    (log1p of the deviation from 1 for accuracy)."""
    M = N if M is None else M
    ci = np.cos(np.pi * np.arange(1, N + 1) / (N + 1))
    cj = np.cos(np.pi * np.arange(1, M + 1) / (M + 1))
    tot = []
    for x in ci:
        tot.append(math.fsum(np.log1p(-2.0 * theta * (x + cj))))
    return math.fsum(tot)


def torus_eigs(N: int) -> np.ndarray:
    c = np.cos(2.0 * np.pi * np.arange(N) / N)
    return (4.0 - 2.0 * c[:, None] - 2.0 * c[None, :]).reshape(-1)


def torus_rank1_eigs(N: int, c: float) -> np.ndarray:
    """Eigenvalues of L + c 11^T: the zero mode (i,j)=(0,0) becomes c*N^2."""
    e = torus_eigs(N)
    e[0] = c * N * N
    return e


def torus_log_tau(N: int) -> float:
    """log tau(C_N x C_N) by the matrix-tree theorem with closed-form eigenvalues."""
    c = np.cos(2.0 * np.pi * np.arange(N) / N)
    parts = []
    for i in range(N):
        row = 4.0 - 2.0 * c[i] - 2.0 * c
        if i == 0:
            row = row[1:]
        parts.append(math.fsum(np.log(row)))
    return math.fsum(parts) - math.log(N * N)


def cheb_T(j: int, x):
    """T_j(x) in closed form: cos(j arccos x) for |x|<=1, cosh form outside."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    inside = np.abs(x) <= 1.0
    out[inside] = np.cos(j * np.arccos(x[inside]))
    xo = x[~inside]
    out[~inside] = np.sign(xo) ** j * np.cosh(j * np.arccosh(np.abs(xo)))
    return out


def cheb_poly_closed(c: np.ndarray, x) -> np.ndarray:
    """p_n(x) = sum_j c_j T_j(x) with T_j in closed (trigonometric) form."""
    x = np.asarray(x, dtype=np.float64)
    return sum(c[j] * cheb_T(j, x) for j in range(len(c)))


def log_series_coeffs(a: float, b: float, jmax: int) -> np.ndarray:
    """Chebyshev series coefficients a_0..a_jmax of f(x)=log(((b-a)x+(b+a))/2):
    f(x) = log((b-a)/2) + log(x + c), c = (b+a)/(b-a)."""
    c = (b + a) / (b - a)
    rho = c + math.sqrt(c * c - 1.0)
    out = np.empty(jmax + 1)
    out[0] = math.log((b - a) / 2.0) + math.log(rho / 2.0)
    j = np.arange(1, jmax + 1)
    out[1:] = 2.0 * (-1.0) ** (j + 1) * rho ** (-j.astype(float)) / j
    return out


def theorem3_bound(delta: float, n: int) -> float:
    """Theorem 3 / Lemma 1 envelope per eigenvalue:
    20 log(2(1/delta - 1)) / ((K-1) K^n), K = (sqrt(2-delta)+sqrt(delta))/(sqrt(2-delta)-sqrt(delta))."""
    K = (math.sqrt(2 - delta) + math.sqrt(delta)) / (math.sqrt(2 - delta) - math.sqrt(delta))
    return 20.0 * math.log(2.0 * (1.0 / delta - 1.0)) / ((K - 1.0) * K ** n)
