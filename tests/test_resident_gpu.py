"""GPU parity of the shared-memory-resident multi-step kernel (cheb_resident_kernel)
against the pinned CPU oracle on identical seeded inputs: one cluster of 16 or 8 CTAs (halos and
reductions over DSMEM), the flat grid (one CTA per SM, halos through exported global rows, one
grid counter per step), the unstaged-matrix fallback, rank-1 with ones and explicit u, the power
basis, CTAs without rows, determinism and the timeout status.  Tolerances as
tests/test_parity_gpu.py (north_star: Gamma 1e-10 relative).
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


def _dev_op(kind, A, c=0.0, u=None):
    return P.Operator(kind, P.DeviceCSR.from_host(A), None, c,
                      torch.from_numpy(u).cuda() if u is not None else None)


@pytest.fixture
def env():
    """Set CHEB_* tuning variables for one test (read by the library at every plan)."""
    saved = {}

    def set_(**kw):
        for k, v in kw.items():
            saved.setdefault(k, os.environ.get(k))
            os.environ[k] = str(v)
    yield set_
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    P.set_persistent(1)
    P.set_resident(1)


class _SPD:
    """The paper's §5.1 random SPD matrix (G23) as a plain CSR operator: irregular columns,
    so most gathers leave the CTA and the cluster.  [a,b] = [10^-3, Gershgorin max]."""
    def __init__(self, d=4099, seed=3):
        self.S = W.random_spd(d, seed)
        rows = np.repeat(np.arange(self.S.n_rows), np.diff(self.S.row_ptr))
        self.d, self.mode, self.r1_c, self.degree, self.num_probes, self.seed = d, "csr", 0.0, 25, 20, 11
        self.a = 1e-3
        self.b = float(np.bincount(rows, np.abs(self.S.val), d).max()) * 1.001

    def matrices(self):
        return self.S, None


def _run(orc, wl_name, k, m=None, seed=None):
    wl = _SPD() if wl_name == "spd_csr" else W.get_workload(wl_name)
    A, _ = wl.matrices()
    op = _dev_op(wl.mode, A, wl.r1_c)
    m = m or wl.num_probes
    seed = wl.seed if seed is None else seed
    r = P.logdet(op, wl.a, wl.b, wl.degree, m, seed=seed, k=k, want_moments=True)
    sched = P.last_schedule()
    mu = orc.moments(orc.Op(wl.mode, A, wl.r1_c), wl.a, wl.b, wl.degree, seed, range(m), workers=4)
    g, gp, se = orc.gamma_from_moments(orc.coeffs_log(wl.a, wl.b, wl.degree), mu)
    return wl, r, sched, mu, g, gp, se


def _check(wl, r, mu, g, gp, se):
    assert np.all(np.isfinite(r.moments))
    assert np.abs(r.moments - mu).max() <= 1e-11 * wl.d
    assert abs(r.logdet - g) <= 1e-10 * abs(g), (r.logdet, g)
    assert np.all(np.abs(r.gamma_p - gp) <= 1e-10 * np.abs(gp) + 1e-12 * wl.d)
    assert abs(r.stderr - se) <= 1e-8 * se


# one cluster: gmrf32 at every k, torus_s (rank-1) and gmrf_s at k <= 16
@pytest.mark.parametrize("name,k", [("gmrf32", 8), ("gmrf32", 16), ("gmrf32", 32), ("gmrf32", 64),
                                    ("torus_s", 8), ("torus_s", 16), ("gmrf_s", 16), ("spd_csr", 8)])
def test_resident_one_cluster(orc, env, name, k):
    wl, r, sched, mu, g, gp, se = _run(orc, name, k)
    assert sched == "resident"
    _check(wl, r, mu, g, gp, se)


@pytest.mark.parametrize("rg", [8, 16])
@pytest.mark.parametrize("name,k", [("gmrf32", 16), ("torus_s", 8), ("spd_csr", 8)])
def test_resident_cluster_sizes(orc, env, rg, name, k):
    env(CHEB_RG=rg)
    wl, r, sched, mu, g, gp, se = _run(orc, name, k)
    assert sched == "resident"
    _check(wl, r, mu, g, gp, se)


# the flat grid (the single-cluster shortcut disabled)
@pytest.mark.parametrize("name,k", [("gmrf_s", 16), ("torus_s", 32), ("gmrf32", 64), ("spd_csr", 16),
                                    ("torus_s", 8), ("gmrf_s", 64), ("torus_s", 16), ("torus_s", 64)])
def test_resident_flat_grid(orc, env, name, k):
    env(CHEB_RES_SINGLE_MAX=0)
    wl, r, sched, mu, g, gp, se = _run(orc, name, k)
    assert sched == "resident"
    _check(wl, r, mu, g, gp, se)


@pytest.mark.parametrize("single", [True, False])
@pytest.mark.parametrize("name,k", [("gmrf_s", 16), ("torus_s", 16), ("gmrf32", 64), ("spd_csr", 8)])
def test_resident_moment_doubling(orc, env, single, name, k):
    """Moment doubling (reading G25) on the resident kernel: ceil(n/2) steps give mu_0..mu_n."""
    if not single:
        env(CHEB_RES_SINGLE_MAX=0)
    P.set_doubling(True)
    try:
        wl, r, sched, mu, g, gp, se = _run(orc, name, k)
    finally:
        P.set_doubling(False)
    assert sched == "resident"
    _check(wl, r, mu, g, gp, se)


@pytest.mark.parametrize("single", [True, False])
def test_resident_unstaged_matrix(orc, env, single):
    """A CTA whose matrix rows exceed the staged capacity gathers col/val from global memory."""
    env(CHEB_RES_CAP=0, **({} if single else {"CHEB_RES_SINGLE_MAX": 0}))
    wl, r, sched, mu, g, gp, se = _run(orc, "torus_s", 16)
    assert sched == "resident"
    _check(wl, r, mu, g, gp, se)


@pytest.mark.parametrize("single", [True, False])
def test_resident_rank1_explicit_u(orc, env, single):
    if not single:
        env(CHEB_RES_SINGLE_MAX=0)
    T = W.torus_laplacian(21)
    u = np.linspace(0.5, 1.5, T.n_rows)
    op = _dev_op("rank1", T, 1e-3, u)
    a, b = 1e-3, 8.5
    r = P.logdet(op, a, b, 50, 10, seed=3, k=16, want_moments=True)
    assert P.last_schedule() == "resident"
    mu = orc.moments(orc.Op("rank1", T, 1e-3, u), a, b, 50, 3, range(10))
    assert np.abs(r.moments - mu).max() <= 1e-11 * T.n_rows


@pytest.mark.parametrize("single", [True, False])
def test_resident_power_basis(orc, env, single):
    """Taylor baseline (power recurrence) on the resident kernel: w_j = (I - M/s) w_{j-1}."""
    if not single:
        env(CHEB_RES_SINGLE_MAX=0)
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    op = _dev_op("csr", A)
    s = wl.a + wl.b
    mu_g = P.power_moments(op, s, 12, 0, 16, 5, 16).cpu().numpy()
    assert P.last_schedule() == "resident"
    mu = orc.moments(orc.Op("csr", A), s, 0.0, 12, 5, range(16), power=True)
    assert np.abs(mu_g - mu).max() <= 1e-11 * wl.d


@pytest.mark.parametrize("d", [1, 7, 40])
def test_resident_tiny_operators(orc, env, d):
    """d smaller than the grid: CTAs without rows still take part in every barrier."""
    S = W.random_spd(max(d, 2), 5) if d > 1 else W.csr.from_coo(1, 1, [0], [0], [0.7])
    if d > 1:
        S = W.csr.from_coo(d, d, *_coo_head(S, d))
    lam = float(np.abs(S.val).max()) * 20 + 1.0
    op = _dev_op("csr", S)
    for single in (8192, 0):
        env(CHEB_RES_SINGLE_MAX=single)
        mu_g = P.moments(op, 1e-3, lam, 9, 0, 3, 4, 8).cpu().numpy()
        assert P.last_schedule() == "resident"
        mu = orc.moments(orc.Op("csr", S), 1e-3, lam, 9, 4, range(3))
        scale = np.maximum(np.abs(mu).max(axis=0), d)
        assert np.all(np.abs(mu_g - mu) <= 1e-11 * scale)


def _coo_head(S, d):
    """The leading d x d block of a CSR (symmetric when S is)."""
    rows = np.repeat(np.arange(S.n_rows), np.diff(S.row_ptr))
    keep = (rows < d) & (S.col_idx < d)
    return rows[keep], S.col_idx[keep], S.val[keep]


def test_resident_deterministic_and_equal_to_other_schedules(env):
    """Bit-identical run to run; equal to the persistent and per-step schedules up to the
    summation order of the dot products (w_j itself is computed identically)."""
    wl = W.get_workload("torus_s")
    A, _ = wl.matrices()
    op = _dev_op("rank1", A, wl.r1_c)
    out = []
    for _ in range(2):
        out.append(P.moments(op, wl.a, wl.b, wl.degree, 0, 24, 5, 16).cpu().numpy())
        assert P.last_schedule() == "resident"
    assert np.array_equal(out[0], out[1])
    for pers in (2, 0):
        P.set_persistent(pers)
        other = P.moments(op, wl.a, wl.b, wl.degree, 0, 24, 5, 16).cpu().numpy()
        assert P.last_schedule() == ("persistent" if pers == 2 else "per_step")
        assert np.abs(other - out[0]).max() <= 1e-13 * np.abs(out[0]).max()


def test_resident_off_switch(env):
    wl = W.get_workload("gmrf32")
    A, _ = wl.matrices()
    op = _dev_op("csr", A)
    P.set_resident(0)
    P.moments(op, wl.a, wl.b, 5, 0, 8, 1, 8)
    assert P.last_schedule() == "persistent"
    P.set_resident(1)
    P.moments(op, wl.a, wl.b, 5, 0, 8, 1, 8)
    assert P.last_schedule() == "resident"


@pytest.mark.parametrize("single", [True, False])
def test_resident_timeout_status(env, single):
    """The injected timeout bit poisons the resident call's moments like any other schedule."""
    env(CHEB_INJECT_TIMEOUT=1, **({} if single else {"CHEB_RES_SINGLE_MAX": 0}))
    wl = W.get_workload("gmrf32")
    A, _ = wl.matrices()
    op = _dev_op("csr", A)
    with pytest.raises(P.ChebError):
        P.logdet(op, wl.a, wl.b, wl.degree, 16, seed=1, k=16)
    assert P.last_schedule() == "resident"


# several probe blocks in one launch (single-cluster geometry: one cluster per block, up to the
# co-resident cluster count per launch; CHEB_RES_MULTI=0 runs one block per launch)
@pytest.mark.parametrize("dbl", [False, True])
@pytest.mark.parametrize("name,k,p0,p1", [("gmrf32", 16, 0, 64), ("gmrf32", 8, 3, 203),
                                          ("torus_s", 8, 5, 46), ("spd_csr", 8, 0, 37)])
def test_resident_multi_block(orc, env, dbl, name, k, p0, p1):
    """Blocks sharing a launch give the moments of one block per launch bit for bit, and the
    oracle's: ragged last block, a global probe offset, several launches (> the clusters that fit)."""
    wl = _SPD() if name == "spd_csr" else W.get_workload(name)
    A, _ = wl.matrices()
    op = _dev_op(wl.mode, A, wl.r1_c)
    P.set_doubling(dbl)
    try:
        out = {}
        for multi in (1, 0):
            env(CHEB_RES_MULTI=multi)
            out[multi] = P.moments(op, wl.a, wl.b, wl.degree, p0, p1, wl.seed, k).cpu().numpy()
            assert P.last_schedule() == "resident"
    finally:
        P.set_doubling(False)
    assert np.array_equal(out[1], out[0])
    mu = orc.moments(orc.Op(wl.mode, A, wl.r1_c), wl.a, wl.b, wl.degree, wl.seed, range(p0, p1), workers=4)
    assert np.abs(out[1] - mu).max() <= 1e-11 * wl.d


def test_resident_multi_block_explicit_u(orc, env):
    T = W.torus_laplacian(21)
    u = np.linspace(0.5, 1.5, T.n_rows)
    op = _dev_op("rank1", T, 1e-3, u)
    out = {}
    for multi in (1, 0):
        env(CHEB_RES_MULTI=multi)
        out[multi] = P.moments(op, 1e-3, 8.5, 40, 0, 40, 3, 8).cpu().numpy()
        assert P.last_schedule() == "resident"
    assert np.array_equal(out[1], out[0])
    mu = orc.moments(orc.Op("rank1", T, 1e-3, u), 1e-3, 8.5, 40, 3, range(40))
    assert np.abs(out[1] - mu).max() <= 1e-11 * T.n_rows
