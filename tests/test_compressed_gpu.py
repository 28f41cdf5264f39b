"""GPU tests of the compressed gather-matrix copy (CV format: uniform padded rows, int16 column
deltas, uint8 indices into a table of <= 128 distinct values) read by the per-step
kernels.  The decoded (column, value) pairs equal the plain copy's, so moments must be
BIT-IDENTICAL with and without it (CHEB_CV=0); operators outside the format must fall back
(status bit 0x100 clear) and still match the oracle.
"""
import os

import numpy as np
import pytest

import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_1503_06394_b200 as P  # noqa: E402
from paper_1503_06394_b200.api import STATUS_COMPRESSED  # noqa: E402


@pytest.fixture
def per_step():
    P.set_persistent(0)  # the compressed copy is read by the per-step kernels
    yield
    P.set_persistent(1)
    P.set_doubling(False)
    os.environ.pop("CHEB_CV", None)


def _op(kind, A, c=0.0):
    return P.Operator(kind, P.DeviceCSR.from_host(A), None, c)


def _moments(op, a, b, n, m, seed, k, cv, power=False):
    os.environ["CHEB_CV"] = "1" if cv else "0"
    ws = P.alloc_workspace(op, k)
    if power:
        mu = P.power_moments(op, a, n, 0, m, seed, k, workspace=ws)
    else:
        mu = P.moments(op, a, b, n, 0, m, seed, k, workspace=ws)
    st = P.workspace_status(ws)
    return mu.cpu().numpy(), st


@pytest.mark.parametrize("name,k", [("gmrf_s", 16), ("gmrf_s", 8), ("gmrf32", 8), ("torus_s", 16),
                                    ("torus_s", 8), ("gmrf5000_rows", 16)])
@pytest.mark.parametrize("dbl", [False, True])
def test_compressed_bit_identical(per_step, name, k, dbl):
    if name == "gmrf5000_rows":  # a 300 x 5000 strip of the configs[3] stencil: HBM-sized tiles
        wl = W.get_workload("gmrf5000")
        A = W.grid_gmrf(300, 0.24, 5000)
        op, m, n = _op("csr", A), 24, 12
    else:
        wl = W.get_workload(name)
        A, _ = wl.matrices()
        op, m, n = _op(wl.mode, A, wl.r1_c), wl.num_probes, wl.degree
    P.set_doubling(dbl)
    mu1, st1 = _moments(op, wl.a, wl.b, n, m, wl.seed, k, True)
    mu0, st0 = _moments(op, wl.a, wl.b, n, m, wl.seed, k, False)
    assert st1 & STATUS_COMPRESSED and not st0 & STATUS_COMPRESSED
    assert st1 & 3 == 0 and st0 & 3 == 0
    assert np.array_equal(mu1, mu0)


def test_compressed_power_basis_bit_identical(per_step):
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    op = _op("csr", A)
    s = wl.a + wl.b
    mu1, st1 = _moments(op, s, 0.0, 12, 16, 5, 16, True, power=True)
    mu0, _ = _moments(op, s, 0.0, 12, 16, 5, 16, False, power=True)
    assert st1 & STATUS_COMPRESSED
    assert np.array_equal(mu1, mu0)


def _perturbed_gmrf(N, seed):
    """The grid stencil with a distinct off-diagonal value per entry (> 128 values)."""
    G = W.grid_gmrf(N, 0.2)
    rows = np.repeat(np.arange(G.n_rows), np.diff(G.row_ptr))
    val = G.val.copy()
    off = rows != G.col_idx
    lo, hi = np.minimum(rows, G.col_idx), np.maximum(rows, G.col_idx)
    val[off] = -0.2 * (1.0 + 0.01 * np.sin(lo[off] * 7.0 + hi[off] * 3.0 + seed))  # symmetric
    return W.csr.from_coo(G.n_rows, G.n_cols, rows, G.col_idx, val)


def _far_band(d, off):
    """Tridiagonal plus a symmetric band at distance `off` (> 32767: outside int16 deltas)."""
    i = np.arange(d)
    r = [i, i[:-1], i[1:], i[:-off], i[off:]]
    c = [i, i[1:], i[:-1], i[off:], i[:-off]]
    v = [np.full(d, 1.0), np.full(d - 1, -0.2), np.full(d - 1, -0.2), np.full(d - off, -0.1),
         np.full(d - off, -0.1)]
    return W.csr.from_coo(d, d, np.concatenate(r), np.concatenate(c), np.concatenate(v))


@pytest.mark.parametrize("case", ["many_values", "far_columns", "ragged_rows"])
def test_compressed_fallback(orc, per_step, case):
    if case == "many_values":
        A, a, b = _perturbed_gmrf(40, 3), 0.15, 1.85
    elif case == "far_columns":
        A, a, b = _far_band(40000, 33000), 0.3, 1.7
    else:  # rows of 6+ entries: padded to 10, not uniform
        A = W.random_spd(3000, 4)
        rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
        a, b = 1e-3, float(np.bincount(rows, np.abs(A.val), A.n_rows).max()) * 1.001
    op = _op("csr", A)
    mu1, st1 = _moments(op, a, b, 20, 8, 7, 8, True)
    assert not st1 & STATUS_COMPRESSED and st1 & 3 == 0
    mu = orc.moments(orc.Op("csr", A), a, b, 20, 7, range(8))
    scale = np.maximum(np.abs(mu).max(axis=0), A.n_rows)
    assert np.all(np.abs(mu1 - mu) <= 1e-11 * scale)


@pytest.mark.parametrize("k", [32, 64, 128])
def test_compressed_not_used_above_k16(per_step, k):
    """Probe blocks k > 16 keep the plain copy (the matrix is a small share of their bytes; k = 128
    on 16-row-per-group tiles would also have 8-row tiles, whose value slices are not 16-byte
    aligned): the status says so."""
    wl = W.get_workload("gmrf32")
    A, _ = wl.matrices()
    op = _op("csr", A)
    mu1, st1 = _moments(op, wl.a, wl.b, 10, 40, 3, k, True)
    assert not st1 & STATUS_COMPRESSED and st1 & 3 == 0


def test_compressed_far_columns_within_int16(orc, per_step):
    """A band at distance 32767 (the int16 limit) stays in the format and matches the oracle."""
    A = _far_band(40000, 32767)
    op = _op("csr", A)
    mu1, st1 = _moments(op, 0.3, 1.7, 20, 8, 7, 8, True)
    assert st1 & STATUS_COMPRESSED
    mu = orc.moments(orc.Op("csr", A), 0.3, 1.7, 20, 7, range(8))
    assert np.abs(mu1 - mu).max() <= 1e-11 * A.n_rows


def test_compressed_cuda_graph_replay(per_step):
    """The compressed-copy set-up (memsets + two kernels) is capturable: a CUDA-graph replay
    reproduces the eager estimate bit for bit."""
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    op = _op("csr", A)
    est = P.Estimator(op, wl.a, wl.b, wl.degree, 32, 16, seed=wl.seed)
    gp0, st0 = est.run()
    torch.cuda.synchronize()
    assert P.workspace_status(est.workspace) & STATUS_COMPRESSED
    gp0, st0 = gp0.clone(), st0.clone()
    replay, gp, st = est.capture()
    for _ in range(3):
        replay()
    torch.cuda.synchronize()
    assert torch.equal(st, st0) and torch.equal(gp, gp0)


def test_family_mode_reads_the_plain_copy(orc):
    """Family mode (f2) keeps the plain copy (status bit clear) and matches the oracle per member."""
    import paper_1503_06394_b200.gmrf as G
    base = W.grid_gmrf(37, 1.0)  # I - Adj: D = I, O = -Adj
    fam = G.PrecisionFamily(P.DeviceCSR.from_host(base))
    thetas = [-0.24, 0.05, 0.2, 0.23]
    lh = fam.gershgorin(thetas)
    n, m, seed = 25, 13, 4
    ws = P.alloc_workspace(P.Operator("family", fam.base), 64)
    mu = fam.moments(thetas, lh, n, 0, m, seed, 64, workspace=ws).cpu().numpy()
    assert not P.workspace_status(ws) & STATUS_COMPRESSED
    for r, th in enumerate(thetas):
        A = W.grid_gmrf(37, th)
        want = orc.moments(orc.Op("csr", A), lh[r, 0], lh[r, 1], n, seed, range(m), workers=4)
        assert np.abs(mu[r] - want).max() <= 1e-11 * A.n_rows
