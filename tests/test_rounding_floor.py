"""Rounding floor of the oracle per BASELINE config ("Check the floor on the box").

The 1e-10 GPU-vs-oracle contract is meaningful only if the oracle's own result is stable far
below it under a change of summation order.  Each config runs the oracle twice on the same probe:
once as given and once on the row-reversed problem A' = P A P^T, v' = P v (P the reversal
permutation).  The moments are equal in exact arithmetic (v'^T T_j(Ã') v' = v^T T_j(Ã) v), but every
SpMV row sum and every dot product is accumulated in the opposite order.  Required:
|Gamma_p - Gamma_p'| <= 1e-12 |Gamma_p| (two orders of magnitude below the parity contract).
CPU only (no GPU code involved).
"""
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import workloads as W
from workloads.csr import CSR


def reverse_csr(A: CSR) -> CSR:
    """P A P^T for the reversal permutation i -> n-1-i (square A): reversing the whole entry
    array reverses the row order and each row's entries, which keeps columns ascending."""
    n = A.n_rows
    nnz = A.nnz
    rp = (nnz - A.row_ptr[::-1]).astype(np.int64)
    ci = (n - 1 - A.col_idx.astype(np.int64))[::-1].astype(np.int32)
    return CSR(n, A.n_cols, np.ascontiguousarray(rp), np.ascontiguousarray(ci),
               np.ascontiguousarray(A.val[::-1]))


def _gamma(name: str, reverse: bool, probe: int) -> float:
    import oracle as orc
    wl = W.get_workload(name)
    A, _ = wl.matrices()
    a, b = (wl.a, wl.b) if wl.a is not None else orc.bounds_btb(A)
    v = orc.rademacher(wl.seed, probe, A.n_cols)
    if reverse:
        A = reverse_csr(A)
        v = np.ascontiguousarray(v[::-1])
    mu = orc.moments_vec(orc.Op(wl.mode, A, wl.r1_c), a, b, wl.degree, v)
    return float(orc.gamma_from_moments(orc.coeffs_log(a, b, wl.degree), mu[None, :])[0])


def test_reverse_csr_is_the_permuted_matrix():
    A = W.random_spd(300, 5)
    R = reverse_csr(A)
    R.check()
    Ad, Rd = W.csr.to_dense(A), W.csr.to_dense(R)
    assert np.array_equal(Rd, Ad[::-1, ::-1])


@pytest.mark.parametrize("name", ["gmrf32", "torus256", "gmrf1000", "btb4m",
                                  pytest.param("gmrf5000", marks=pytest.mark.slow)])
def test_oracle_rounding_floor(orc, name):
    with ProcessPoolExecutor(max_workers=2) as ex:
        fwd, rev = ex.submit(_gamma, name, False, 0), ex.submit(_gamma, name, True, 0)
        g0, g1 = fwd.result(), rev.result()
    assert np.isfinite(g0) and np.isfinite(g1)
    assert abs(g0 - g1) <= 1e-12 * abs(g0), (name, g0, g1, abs(g0 - g1) / abs(g0))
