"""GPU parity of the moment-doubling schedule (cheb_set_doubling; reading G25).

With doubling the library applies Ã only ceil(n/2) times per probe and forms
  mu_{2j} = 2 w_j^T w_j - mu_0,   mu_{2j-1} = 2 w_j^T w_{j-1} - mu_1
(T_{2j} = 2T_j^2 - I, T_{2j+1} = 2T_{j+1}T_j - T_1 for symmetric Ã).  The oracle is NOT
changed: it still runs Algorithm 1's recurrence for all n steps and takes mu_j = v^T w_j
directly, so these tests check the identity end to end against an independent
computation, with the same tolerances as the plain path (1e-11 d on moments, 1e-10
relative on Gamma).
"""
import numpy as np
import pytest

import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_1503_06394_b200 as P  # noqa: E402

GAMMA_RTOL = 1e-10


@pytest.fixture
def doubling():
    P.set_doubling(True)
    yield
    P.set_doubling(False)
    P.set_persistent(1)


def _dev_op(kind, A, At=None, c=0.0, u=None):
    return P.Operator(kind, P.DeviceCSR.from_host(A),
                      P.DeviceCSR.from_host(At) if At is not None else None, c,
                      torch.from_numpy(u).cuda() if u is not None else None)


def _check(mu_gpu, mu_orc, d):
    mu_gpu = np.asarray(mu_gpu)
    assert mu_gpu.shape == mu_orc.shape
    assert np.all(np.isfinite(mu_gpu))
    err = np.abs(mu_gpu - mu_orc).max()
    assert err <= 1e-11 * d, err


@pytest.mark.parametrize("name", ["gmrf32", "gmrf_s", "torus_s", "btb_s", "spd_s"])
@pytest.mark.parametrize("k", [8, 16, 64, 128])
@pytest.mark.parametrize("persist", [0, 2])
def test_doubling_moments_and_gamma_small(orc, doubling, name, k, persist):
    P.set_persistent(persist)
    wl = W.get_workload(name)
    A, At = wl.matrices()
    op = _dev_op(wl.mode, A, At, wl.r1_c)
    a, b = (wl.a, wl.b) if wl.a is not None else P.bounds_btb(op)
    m = wl.num_probes
    r = P.logdet(op, a, b, wl.degree, m, seed=wl.seed, k=k, want_moments=True)
    mu = orc.moments(orc.Op(wl.mode, A, wl.r1_c), a, b, wl.degree, wl.seed, range(m), workers=4)
    _check(r.moments, mu, wl.d)
    g, gp, se = orc.gamma_from_moments(orc.coeffs_log(a, b, wl.degree), mu)
    assert abs(r.logdet - g) <= GAMMA_RTOL * abs(g)
    assert np.all(np.abs(r.gamma_p - gp) <= 1e-10 * np.abs(gp) + 1e-12 * wl.d)


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5, 8, 41])
@pytest.mark.parametrize("persist", [0, 2])
def test_doubling_degrees_odd_even(orc, doubling, n, persist):
    """Every degree parity: the last step writes mu_{2j-1} and (if 2j <= n) mu_{2j}."""
    P.set_persistent(persist)
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    op = _dev_op("csr", A)
    n0 = P.launch_count()
    r = P.logdet(op, wl.a, wl.b, n, 9, seed=2, k=8, want_moments=True)
    nl = P.launch_count() - n0
    steps = (n + 1) // 2
    blocks = 2
    if persist == 0:
        # prep (count + scatter), compressed copy (values + encode), (init + ceil(n/2) steps) per
        # block, status epilogue, finalize
        assert nl == 2 + 2 + blocks * (1 + steps) + 1 + 1
    mu = orc.moments(orc.Op("csr", A), wl.a, wl.b, n, 2, range(9))
    _check(r.moments, mu, wl.d)


def test_doubling_rank1_explicit_u(orc, doubling):
    T = W.torus_laplacian(21)
    u = np.linspace(0.5, 1.5, T.n_rows)
    op = _dev_op("rank1", T, None, 1e-3, u)
    a, b = 1e-3, 8.5
    for persist in (0, 2):
        P.set_persistent(persist)
        r = P.logdet(op, a, b, 50, 10, seed=3, k=16, want_moments=True)
        mu = orc.moments(orc.Op("rank1", T, 1e-3, u), a, b, 50, 3, range(10))
        _check(r.moments, mu, T.n_rows)


@pytest.mark.parametrize("name", ["gmrf32", "torus_s", "gmrf_s"])
def test_doubling_persistent_bit_identical_to_per_step(doubling, name):
    wl = W.get_workload(name)
    A, _ = wl.matrices()
    op = _dev_op(wl.mode, A, None, wl.r1_c)
    out = {}
    for mode in (0, 2):
        P.set_persistent(mode)
        out[mode] = P.moments(op, wl.a, wl.b, wl.degree, 0, 24, 5, 16).cpu().numpy()
    assert np.array_equal(out[0], out[2])


def test_doubling_shards_and_determinism(doubling):
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    op = _dev_op("csr", A)
    full = P.moments(op, wl.a, wl.b, 13, 0, 32, 9, 16).cpu().numpy()
    part = P.moments(op, wl.a, wl.b, 13, 5, 21, 9, 16).cpu().numpy()
    assert np.array_equal(full[5:21], part)
    assert np.array_equal(full, P.moments(op, wl.a, wl.b, 13, 0, 32, 9, 16).cpu().numpy())


def test_doubling_off_restores_algorithm1(orc):
    """Default schedule is Algorithm 1 (n applications)."""
    assert not P.get_doubling()
    wl = W.get_workload("gmrf32")
    A, _ = wl.matrices()
    op = _dev_op("csr", A)
    P.set_persistent(0)
    try:
        n0 = P.launch_count()
        P.logdet(op, wl.a, wl.b, 10, 16, k=16)
        assert P.launch_count() - n0 == 2 + 2 + 1 + 10 + 1 + 1  # prep, compressed copy, init, steps, status, finalize
        P.set_doubling(True)
        n0 = P.launch_count()
        P.logdet(op, wl.a, wl.b, 10, 16, k=16)
        assert P.launch_count() - n0 == 2 + 2 + 1 + 5 + 1 + 1
    finally:
        P.set_doubling(False)
        P.set_persistent(1)

# Full-size doubling parity (every probe of configs[0..4] vs the oracle's tables) lives in
# tests/test_parity_full_gpu.py.
