"""GPU parity: the CUDA path (through the C ABI) against the pinned CPU oracle on
identical seeded inputs.

Tolerances (BASELINE north_star):
  * probes: bit-exact (integer/bit work);
  * Gamma: |Gamma_gpu - Gamma_oracle| <= 1e-10 |Gamma_oracle|;
  * diagnostics: |d mu_{p,j}| <= 1e-11 * d, per-probe |d Gamma_p| <= 1e-10 |Gamma_p| + 1e-12 d.
"""
import math

import numpy as np
import pytest

import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes only with -m gpu
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_1503_06394_b200 as P  # noqa: E402

GAMMA_RTOL = 1e-10


def _mats(wl):
    A, At = wl.matrices()
    return A, At


def _dev_op(kind, A, At=None, c=0.0, u=None):
    return P.Operator(kind, P.DeviceCSR.from_host(A),
                      P.DeviceCSR.from_host(At) if At is not None else None, c,
                      torch.from_numpy(u).cuda() if u is not None else None)


def _check_moments(mu_gpu, mu_orc, d):
    mu_gpu = np.asarray(mu_gpu)
    assert mu_gpu.shape == mu_orc.shape
    assert np.all(np.isfinite(mu_gpu))
    err = np.abs(mu_gpu - mu_orc).max()
    assert err <= 1e-11 * d, err


def _check_gamma(g_gpu, g_orc):
    assert abs(g_gpu - g_orc) <= GAMMA_RTOL * abs(g_orc), (g_gpu, g_orc)


# ------------------------------------------------------------------ probes (a2)
@pytest.mark.parametrize("d,p0,k", [(1, 0, 8), (1000, 0, 8), (1027, 5, 16), (4099, 33, 32),
                                    (65536, 64, 64), (3, 1 << 40, 64), (5000, 7, 128)])
def test_probes_bit_identical(orc, d, p0, k):
    v = P.probes(d, 0x1234, p0, k).cpu().numpy()
    for j in range(k):
        assert np.array_equal(v[:, j], orc.rademacher(0x1234, p0 + j, d)), (j,)


# ------------------------------------------------------------------ small configs, every k
SMALL = ["gmrf32", "gmrf_s", "torus_s", "btb_s", "spd_s"]


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("k", [8, 16, 32, 64, 128])
@pytest.mark.parametrize("persist", [0, 2])
def test_moments_and_gamma_small(orc, persistent_mode, name, k, persist):
    """Per-step launches (persist=0) and the persistent multi-step kernel (persist=2,
    csr/rank-1) against the oracle."""
    persistent_mode(persist)
    wl = W.get_workload(name)
    A, At = _mats(wl)
    op = _dev_op(wl.mode, A, At, wl.r1_c)
    a, b = (wl.a, wl.b) if wl.a is not None else P.bounds_btb(op)
    m = wl.num_probes  # 12/20/64: ragged last block for most k
    r = P.logdet(op, a, b, wl.degree, m, seed=wl.seed, k=k, want_moments=True)
    mu = orc.moments(orc.Op(wl.mode, A, wl.r1_c), a, b, wl.degree, wl.seed, range(m), workers=4)
    _check_moments(r.moments, mu, wl.d)
    g, gp, se = orc.gamma_from_moments(orc.coeffs_log(a, b, wl.degree), mu)
    _check_gamma(r.logdet, g)
    assert np.all(np.abs(r.gamma_p - gp) <= 1e-10 * np.abs(gp) + 1e-12 * wl.d)
    assert abs(r.stderr - se) <= 1e-8 * se


@pytest.fixture
def persistent_mode():
    """Restore the default persistent-kernel mode after a test."""
    yield P.set_persistent
    P.set_persistent(1)


def test_rank1_explicit_u(orc):
    T = W.torus_laplacian(21)
    u = np.linspace(0.5, 1.5, T.n_rows)
    op = _dev_op("rank1", T, None, 1e-3, u)
    a, b = 1e-3, 8.5
    r = P.logdet(op, a, b, 50, 10, seed=3, k=16, want_moments=True)
    mu = orc.moments(orc.Op("rank1", T, 1e-3, u), a, b, 50, 3, range(10))
    _check_moments(r.moments, mu, T.n_rows)


@pytest.mark.parametrize("dbl", [False, True])
@pytest.mark.parametrize("persist", [0, 2])
def test_general_csr_without_diagonal_entries(orc, persistent_mode, dbl, persist):
    """Rows without a stored diagonal and empty rows (the -beta*w term must still apply): the prep
    adds an (i, -beta) entry at the head of such a row, and the doubling kernels read w_{j-1}[i]
    from that first gather; per-step and persistent schedules."""
    persistent_mode(persist)
    P.set_doubling(dbl)
    try:
        _csr_without_diagonal(orc)
    finally:
        P.set_doubling(False)


def _csr_without_diagonal(orc):
    S = W.random_spd(3000, 4)
    rows = np.repeat(np.arange(S.n_rows), np.diff(S.row_ptr))
    keep = (rows != S.col_idx) | (rows % 7 != 0)
    # some rows (and, to keep the operator symmetric -- moment doubling assumes it -- their
    # columns) become empty
    keep &= ~((rows % 101) == 5) & ~((S.col_idx % 101) == 5)
    C = W.csr.from_coo(S.n_rows, S.n_cols, rows[keep], S.col_idx[keep], S.val[keep])
    lam = 1.0 + np.abs(C.val).max() * 40
    op = _dev_op("csr", C)
    mu_g = P.moments(op, 0.05, lam, 25, 0, 9, 11, 8).cpu().numpy()
    mu = orc.moments(orc.Op("csr", C), 0.05, lam, 25, 11, range(9))
    # the spectrum leaves [a,b] (no stored diagonal in some rows): compare relative
    scale = np.maximum(np.abs(mu).max(axis=0), C.n_rows)
    assert np.all(np.abs(mu_g - mu) <= 1e-11 * scale)


@pytest.mark.parametrize("n", [0, 1, 2])
def test_degenerate_degrees(orc, n):
    wl = W.get_workload("gmrf_s")
    A, _ = _mats(wl)
    op = _dev_op("csr", A)
    r = P.logdet(op, wl.a, wl.b, n, 5, seed=2, k=8, want_moments=True)
    mu = orc.moments(orc.Op("csr", A), wl.a, wl.b, n, 2, range(5))
    _check_moments(r.moments, mu, wl.d)
    if n == 0:
        assert np.all(r.moments[:, 0] == wl.d)
        assert r.logdet == coeffs0(wl) * wl.d


def coeffs0(wl):
    return P.coeffs_log(wl.a, wl.b, 0)[0]


def test_single_row_and_single_probe(orc):
    A = W.csr.from_coo(1, 1, [0], [0], [0.7])
    op = _dev_op("csr", A)
    r = P.logdet(op, 0.5, 1.0, 10, 1, seed=4, k=8, want_moments=True)
    mu = orc.moments(orc.Op("csr", A), 0.5, 1.0, 10, 4, [0])
    _check_moments(r.moments, mu, 1)
    assert r.stderr == 0.0
    assert abs(r.logdet - math.log(0.7)) < 1e-6


def test_shard_offsets_do_not_change_probes(orc):
    """Global probe addressing: moments of probes [5, 21) computed as a shard equal
    the same rows of a [0, 32) run bit for bit (fixed k)."""
    wl = W.get_workload("gmrf_s")
    A, _ = _mats(wl)
    op = _dev_op("csr", A)
    full = P.moments(op, wl.a, wl.b, 12, 0, 32, 9, 16).cpu().numpy()
    part = P.moments(op, wl.a, wl.b, 12, 5, 21, 9, 16).cpu().numpy()
    assert np.array_equal(full[5:21], part)
    again = P.moments(op, wl.a, wl.b, 12, 0, 32, 9, 16).cpu().numpy()
    assert np.array_equal(full, again)  # deterministic reductions


def test_host_entry_point_matches_device(orc):
    wl = W.get_workload("torus_s")
    A, _ = _mats(wl)
    rd = P.logdet(_dev_op("rank1", A, None, wl.r1_c), wl.a, wl.b, wl.degree, wl.num_probes, seed=5,
                  k=8, want_moments=True)
    rh = P.logdet_host("rank1", A, wl.a, wl.b, wl.degree, wl.num_probes, seed=5, k=8, c=wl.r1_c,
                       want_moments=True)
    assert np.array_equal(rd.moments, rh.moments) and rd.logdet == rh.logdet


def test_bounds_btb_match_oracle(orc):
    for d, seed in ((5003, 3), (20000, 8)):
        B = W.random_nonsingular(d, seed)
        op = _dev_op("btb", B, W.transpose(B))
        a, b = P.bounds_btb(op)
        oa, ob = orc.bounds_btb(B)
        assert abs(a - oa) <= 1e-13 * oa and abs(b - ob) <= 1e-13 * ob


def test_nonfinite_detected():
    """b below lambda_max: |T_j| grows geometrically and overflows -> CL_ENONFINITE."""
    A = W.csr.from_coo(50, 50, np.arange(50), np.arange(50), np.full(50, 1e6))
    op = _dev_op("csr", A)
    with pytest.raises(P.ChebError) as ei:
        P.logdet(op, 0.5, 1.0, 200, 8, seed=1, k=8)
    assert ei.value.code == -5


def test_launch_count_increases(persistent_mode):
    wl = W.get_workload("gmrf32")
    A, _ = _mats(wl)
    op = _dev_op("csr", A)
    persistent_mode(0)
    n0 = P.launch_count()
    P.logdet(op, wl.a, wl.b, 10, 16, k=16)
    # prep (count + scatter) + compressed copy (values + encode) + init + 10 steps + status epilogue
    # + finalize
    assert P.launch_count() - n0 == 2 + 2 + 1 + 10 + 1 + 1
    persistent_mode(2)
    n0 = P.launch_count()
    P.logdet(op, wl.a, wl.b, 10, 16, k=16)
    assert P.launch_count() - n0 == 2 + 1 + 1 + 1 + 1  # prep (2) + init + persistent + status + finalize


@pytest.mark.parametrize("name", ["gmrf32", "torus_s", "gmrf_s"])
def test_persistent_bit_identical_to_per_step(persistent_mode, name):
    """Same grid, same tile schedule, same reduction order: identical moments."""
    wl = W.get_workload(name)
    A, _ = _mats(wl)
    op = _dev_op(wl.mode, A, None, wl.r1_c)
    out = {}
    for mode in (0, 2):
        persistent_mode(mode)
        out[mode] = P.moments(op, wl.a, wl.b, wl.degree, 0, 24, 5, 16).cpu().numpy()
    assert np.array_equal(out[0], out[2])


# ------------------------------------------------------------------ estimate vs truth
def test_config0_estimate_vs_closed_form():
    from oracle import closed_forms as cf
    wl = W.get_workload("gmrf32")
    A, _ = _mats(wl)
    r = P.logdet(_dev_op("csr", A), wl.a, wl.b, wl.degree, wl.num_probes, seed=wl.seed, k=64)
    assert abs(r.logdet - cf.grid_logdet(32, 0.2)) <= 4 * r.stderr


# ------------------------------------------------------------------ BASELINE full sizes, sampled
def _full_size(orc, name, k, sample, workers=None):
    wl = W.get_workload(name)
    A, At = _mats(wl)
    op = _dev_op(wl.mode, A, At, wl.r1_c)
    a, b = (wl.a, wl.b) if wl.a is not None else P.bounds_btb(op)
    est = P.Estimator(op, a, b, wl.degree, wl.num_probes, k, seed=wl.seed)
    gp, stats = est.run()
    torch.cuda.synchronize()
    mu = est.mu.cpu().numpy()
    st = stats.cpu().numpy()
    assert st[2] == 1.0
    omu = orc.moments(orc.Op(wl.mode, A, wl.r1_c), a, b, wl.degree, wl.seed, sample,
                      workers=workers or len(sample))
    _check_moments(mu[list(sample)], omu, wl.d)
    c = orc.coeffs_log(a, b, wl.degree)
    gpn = gp.cpu().numpy()
    for i, p in enumerate(sample):
        og = orc.gamma_from_moments(c, omu[i:i + 1])[0]
        assert abs(gpn[p] - og) <= GAMMA_RTOL * abs(og) + 1e-12 * wl.d
    return wl, st, a, b


def test_full_config1_torus256(orc):
    from oracle import closed_forms as cf
    wl, st, a, b = _full_size(orc, "torus256", 32, [0, 31])
    log_tau = P.log_tau_from_rank1(st[0], wl.r1_c, wl.d)
    assert abs(log_tau - cf.torus_log_tau(256)) <= 4 * st[1]


def test_full_config2_gmrf1000(orc):
    from oracle import closed_forms as cf
    wl, st, a, b = _full_size(orc, "gmrf1000", 64, [0, 37, 63])
    assert abs(st[0] - cf.grid_logdet(1000, 0.24)) <= 4 * st[1]


@pytest.mark.slow
def test_full_config3_gmrf5000_bench_launch(orc):
    """The bench launch configuration (k = 64, m = 128, two probe blocks)."""
    from oracle import closed_forms as cf
    wl, st, a, b = _full_size(orc, "gmrf5000", 64, [0, 127])
    assert abs(st[0] - cf.grid_logdet(5000, 0.24)) <= 4 * st[1]


@pytest.mark.slow
def test_full_config4_btb4m(orc):
    _full_size(orc, "btb4m", 64, [0, 63])


# ------------------------------------------------------------------ Taylor baseline
@pytest.mark.parametrize("name", ["gmrf_s", "torus_s", "btb_s", "spd_s"])
@pytest.mark.parametrize("persist", [0, 2])
def test_taylor_power_moments_parity(orc, persistent_mode, name, persist):
    """Power-basis moments v^T (I - M/s)^j v through the same fused kernels vs the oracle."""
    persistent_mode(persist)
    wl = W.get_workload(name)
    A, At = _mats(wl)
    op = _dev_op(wl.mode, A, At, wl.r1_c)
    a, b = (wl.a, wl.b) if wl.a is not None else P.bounds_btb(op)
    s = a + b
    n, m = 25, 11
    mu = P.power_moments(op, s, n, 0, m, wl.seed, 16).cpu().numpy()
    want = orc.moments(orc.Op(wl.mode, A, wl.r1_c), s, 0.0, n, wl.seed, range(m), workers=4, power=True)
    _check_moments(mu, want, wl.d)
    g, se, _ = P.taylor_logdet(op, s, n, m, wl.seed, 16)
    og = orc.taylor_logdet(orc.Op(wl.mode, A, wl.r1_c), s, n, m, wl.seed, workers=4)
    _check_gamma(g, og["gamma"])


def test_chebyshev_beats_taylor_config2():
    """Fig. 1(d) claim on the GPU path, matched (m, n, seed), BASELINE configs[2]:
    the Chebyshev estimate is within 4 stderr of the exact log det and closer to it than
    the Taylor estimate."""
    from oracle import closed_forms as cf
    wl = W.get_workload("gmrf1000")
    A, _ = _mats(wl)
    op = _dev_op("csr", A)
    n, m = 30, 64
    r = P.logdet(op, wl.a, wl.b, n, m, seed=wl.seed, k=64)
    gt, _, _ = P.taylor_logdet(op, wl.a + wl.b, n, m, wl.seed, 64)
    exact = cf.grid_logdet(1000, 0.24)
    assert abs(r.logdet - exact) <= 4 * r.stderr
    assert abs(r.logdet - exact) < abs(gt - exact)


# ------------------------------------------------------------------ spectral bounds
@pytest.mark.parametrize("name", ["gmrf_s", "torus_s", "btb_s"])
def test_affine_power_moments_parity(orc, name):
    wl = W.get_workload(name)
    A, At = _mats(wl)
    op = _dev_op(wl.mode, A, At, wl.r1_c)
    s = P.norm_bound(op)
    for alpha, beta in ((1.0 / s, 0.0), (-1.0 / s, -1.0)):
        mu = P.affine_power_moments(op, alpha, beta, 30, 0, 9, 5, 16).cpu().numpy()
        want = orc.affine_power_moments(orc.Op(wl.mode, A, wl.r1_c), alpha, beta, 30, 5, range(9))
        assert np.all(np.abs(mu - want) <= 1e-11 * np.maximum(np.abs(want), wl.d))


def test_norm_bounds_match_oracle(orc):
    G = W.grid_gmrf(40, 0.23)
    assert P.norm_bound(_dev_op("csr", G)) == orc.gershgorin(G)
    B = W.random_nonsingular(3000, 4)
    ob = orc.bounds_btb(B)[1]
    assert abs(P.norm_bound(_dev_op("btb", B, W.transpose(B))) - ob) <= 1e-13 * ob


def _dense_spectrum(kind, A, c=0.0):
    """Extreme eigenvalues of the (small) operator from a dense symmetric eigensolver (cuSOLVER)."""
    D = torch.from_numpy(W.to_dense(A)).cuda()
    if kind == "btb":
        D = D.T @ D
    elif kind == "rank1":
        D = D + c
    lam = torch.linalg.eigvalsh(D)
    return float(lam[0]), float(lam[-1])


@pytest.mark.parametrize("name", ["gmrf_s", "torus_s", "btb_s", "spd_s"])
def test_spectrum_bounds_match_oracle_lanczos(orc, name):
    """f4: the device Lanczos runs (one per probe, on M) produce the oracle's Lanczos tridiagonals
    (explicit vectors, full re-orthogonalisation, mapped from Ã-space to M-space) over the first 20
    steps -- before the extreme Ritz values converge, where the two agree to rounding -- and, after
    80 steps, the same extreme Ritz values, which lie inside the dense spectrum; [a, b] encloses it."""
    wl = W.get_workload(name)
    A, At = _mats(wl)
    op = _dev_op(wl.mode, A, At, wl.r1_c)
    oop = orc.Op(wl.mode, A, wl.r1_c)
    l0, l1 = _dense_spectrum(wl.mode, A, wl.r1_c)
    lo, hi = 0.0, 1.1 * l1  # the oracle's Ã map (Lanczos is affine invariant)
    al_, be_ = 2.0 / (hi - lo), (hi + lo) / (hi - lo)
    probes, seed = 4, 21
    sb = P.spectrum_bounds(op, 20, probes, seed=seed, want_jacobi=True)
    assert sb["lanczos_steps"] == 20
    for p, (ga, gb) in enumerate(sb["jacobi"]):
        oa, ob = orc.lanczos(oop, lo, hi, 20, seed=seed, p=p)
        assert np.max(np.abs(ga - (oa + be_) / al_)) <= 1e-9 * l1, np.max(np.abs(ga - (oa + be_) / al_))
        assert np.max(np.abs(gb - ob / al_)) <= 1e-9 * l1, np.max(np.abs(gb - ob / al_))
    # after 80 steps: extreme Ritz values inside the dense spectrum and within their residual bound
    # of its ends (Kahan); the oracle's (re-orthogonalised) run obeys the same
    sb = P.spectrum_bounds(op, 80, probes, seed=seed)
    ob = orc.spectrum_bounds(oop, lo, hi, 80, seed, range(probes))
    tol = 1e-10 * l1
    for r in (sb, ob):
        assert l0 - tol <= r["lambda_min"] <= l0 + r["res_min"] + tol, (r, l0)
        assert l1 - r["res_max"] - tol <= r["lambda_max"] <= l1 + tol, (r, l1)
    assert sb["a"] <= l0 and sb["b"] >= l1 and sb["b"] <= sb["hi_bound"]


def test_spectrum_bounds_grid_closed_form():
    """Device Lanczos recovers the grid's closed-form extreme eigenvalues; [a, b] encloses the
    spectrum; hi defaults to the device norm bound."""
    from oracle import closed_forms as cf
    N, theta = 20, 0.2
    op = _dev_op("csr", W.grid_gmrf(N, theta))
    sb = P.spectrum_bounds(op, 80, 4, seed=5)
    lam = cf.grid_eigs(N, theta)
    assert sb["lanczos_steps"] == 80
    assert abs(sb["lambda_min"] - lam.min()) < 1e-9 and abs(sb["lambda_max"] - lam.max()) < 1e-9
    assert sb["a"] <= lam.min() and lam.max() <= sb["b"] <= sb["hi_bound"]
    assert sb["hi_bound"] == P.norm_bound(op)


@pytest.mark.slow
def test_spectrum_bounds_config3_estimate(orc):
    """configs[3] without a caller-supplied interval: device Lanczos bounds enclose the closed-form
    spectrum [1 - 4 theta cos(pi/5001), 1 + 4 theta cos(pi/5001)], and the estimate on them equals
    the closed-form-interval estimate (same probes) within its standard error."""
    wl = W.get_workload("gmrf5000")
    A, _ = _mats(wl)
    op = _dev_op("csr", A)
    sb = P.spectrum_bounds(op, 100, 8, seed=77)
    c = math.cos(math.pi / 5001)
    lmin, lmax = 1 - 4 * 0.24 * c, 1 + 4 * 0.24 * c
    assert 0 < sb["a"] <= lmin and lmax <= sb["b"], sb
    ra = P.logdet(op, sb["a"], sb["b"], wl.degree, wl.num_probes, seed=wl.seed, k=64)
    rc = P.logdet(op, wl.a, wl.b, wl.degree, wl.num_probes, seed=wl.seed, k=64)
    assert abs(ra.logdet - rc.logdet) <= rc.stderr, (ra.logdet, rc.logdet, rc.stderr, sb)


# ------------------------------------------------------------------ GMRF likelihood scan
def _grid_family(N):
    import paper_1503_06394_b200.gmrf as G
    base = W.grid_gmrf(N, 1.0)  # I - Adj: D = I, O = -Adj
    return G, G.PrecisionFamily(P.DeviceCSR.from_host(base)), base


def test_quadform_and_gershgorin_parity(orc):
    G, fam, base = _grid_family(37)
    J = fam.at(-0.22)
    Jh = W.grid_gmrf(37, -0.22)
    x = np.random.default_rng(3).standard_normal(J.n_rows)
    q = G.quadform(J, torch.from_numpy(x).cuda())
    oq = orc.quadform(Jh, x)
    assert abs(q - oq) <= 1e-13 * abs(oq)
    lo, hi = G.gershgorin(J)
    assert abs(lo - (1 - 4 * 0.22)) < 1e-15 and abs(hi - (1 + 4 * 0.22)) < 1e-15


def test_family_moments_batched_parity(orc):
    """f2: R = 5 members J(theta) = I - theta Adj in the columns of one probe block (padded to 8
    members, kp = 8 probes each at k = 64; 13 probes: a ragged second block), every member's moments
    vs the oracle on its own matrix and interval; Gershgorin intervals of the family kernel vs the
    closed form; common probes (member r's probe p is the oracle's probe p)."""
    G, fam, base = _grid_family(37)
    thetas = [-0.24, -0.1, 0.05, 0.2, 0.23]
    lh = fam.gershgorin(thetas)
    for (lo, hi), th in zip(lh, thetas):
        assert abs(lo - (1 - 4 * abs(th))) < 1e-15 and abs(hi - (1 + 4 * abs(th))) < 1e-15
    n, m, seed = 30, 13, 4
    for k in (64, 128):
        mu = fam.moments(thetas, lh, n, 0, m, seed, k).cpu().numpy()
        assert mu.shape == (5, m, n + 1)
        for r, th in enumerate(thetas):
            A = W.grid_gmrf(37, th)
            want = orc.moments(orc.Op("csr", A), lh[r, 0], lh[r, 1], n, seed, range(m), workers=4)
            _check_moments(mu[r], want, A.n_rows)
    with pytest.raises(P.ChebError):  # 5 members need k >= 16 (8 x 2 probes)
        fam.moments(thetas, lh, n, 0, m, seed, 8)


def test_quadform_split_parity(orc):
    G, fam, base = _grid_family(29)
    x = np.random.default_rng(5).standard_normal(base.n_rows)
    qd, qo = G.quadform_split(fam.base, torch.from_numpy(x).cuda())
    for th in (-0.2, 0.15):
        oq = orc.quadform(W.grid_gmrf(29, th), x)
        assert abs(qd + th * qo - oq) <= 1e-13 * abs(oq)


def test_likelihood_scan_parity(orc):
    """Scan values vs the oracle's (same probes, same formula, P:670 with reading G16)."""
    import math
    G, fam, base = _grid_family(30)
    rng = np.random.default_rng(8)
    xs = [rng.standard_normal(900) for _ in range(2)]
    thetas = [-0.24, -0.2, 0.1]
    res = G.likelihood_scan(fam, thetas, [torch.from_numpy(x).cuda() for x in xs], 40, 16, seed=4, batched=True)
    res2 = G.likelihood_scan(fam, thetas, [torch.from_numpy(x).cuda() for x in xs], 40, 16, seed=4)
    assert np.allclose(res.loglik, res2.loglik, rtol=1e-12, atol=0)  # batched = separate estimates
    for th, ll in zip(thetas, res.loglik):
        A = W.grid_gmrf(30, th)
        a, b = 1 - 4 * abs(th), 1 + 4 * abs(th)
        og = orc.logdet(orc.Op("csr", A), a, b, 40, 16, 4, workers=4)["gamma"]
        oq = sum(orc.quadform(A, x) for x in xs)
        oll = 0.5 * 2 * og - 0.5 * oq - 0.5 * 2 * 900 * math.log(2 * math.pi)
        assert abs(ll - oll) <= 1e-10 * abs(oll)


def test_likelihood_scan_recovers_rho():
    """§5.2 at desk scale: exact samples x ~ N(0, J(rho*)^-1) (dense Cholesky)
    of a 64x64 grid GMRF with rho* = -0.22; the scan's argmax lands next to rho*."""
    G, fam, base = _grid_family(64)
    rho = -0.22
    Jd = W.to_dense(W.grid_gmrf(64, rho))
    L = np.linalg.cholesky(Jd)
    rng = np.random.default_rng(11)
    xs = [np.linalg.solve(L.T, rng.standard_normal(Jd.shape[0])) for _ in range(8)]
    thetas = np.round(np.arange(-0.245, -0.1949, 0.005), 4)
    res = G.likelihood_scan(fam, thetas, [torch.from_numpy(x).cuda() for x in xs], 80, 64, seed=2)
    assert abs(res.argmax - rho) <= 0.0151, (res.argmax, res.loglik)


# ------------------------------------------------------------------ multi-GPU sharding on the GPU path
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_estimators_sum_to_single_run(world):
    """dist.ShardedEstimator's math on the real kernels: the zero-padded moment tables of
    `world` shards (rank r computes probes shard_range(m, world, r)) sum -- the NCCL
    all_reduce -- to exactly the single-GPU table, so Gamma is bit-identical for any G."""
    from paper_1503_06394_b200.dist import shard_range
    wl = W.get_workload("gmrf_s")
    A, _ = _mats(wl)
    op = _dev_op("csr", A)
    m, k = 24, 8
    full = P.Estimator(op, wl.a, wl.b, 30, m, k, seed=3)
    full.run()
    total = torch.zeros_like(full.mu)
    for r in range(world):
        b0, b1 = shard_range(m, world, r)
        est = P.Estimator(op, wl.a, wl.b, 30, m, k, seed=3, probe_begin=b0, probe_end=b1)
        est.enqueue_moments()
        total += est.mu
    assert torch.equal(total, full.mu)
    _, st_full = P.finalize(full.mu, full.c)
    _, st_sum = P.finalize(total, full.c)
    assert torch.equal(st_full, st_sum)


@pytest.mark.parametrize("name", ["gmrf32", "torus_s", "btb_s", "gmrf_s"])
def test_cuda_graph_replay_identical(name):
    """A captured estimate replays to the bit-identical result of an eager run."""
    wl = W.get_workload(name)
    A, At = _mats(wl)
    op = _dev_op(wl.mode, A, At, wl.r1_c)
    a, b = (wl.a, wl.b) if wl.a is not None else P.bounds_btb(op)
    m = wl.num_probes
    k = next(kk for kk in (8, 16, 32, 64, 128) if kk >= min(m, 64))
    est = P.Estimator(op, a, b, wl.degree, m, k, seed=wl.seed)
    gp0, st0 = est.run()
    torch.cuda.synchronize()
    gp0, st0 = gp0.clone(), st0.clone()
    replay, gp, st = est.capture()
    for _ in range(3):
        replay()
    torch.cuda.synchronize()
    assert torch.equal(st, st0) and torch.equal(gp, gp0)


def test_rank1_ones_general_path_when_rows_do_not_sum_to_zero(orc, persistent_mode):
    """u = 1 on an operator whose rows do not sum to zero (a GMRF: S 1 != 0) must take the
    general u^T w reduction path (the eigenvector shortcut only applies when S 1 = 0 exactly)."""
    wl = W.get_workload("gmrf_s")
    A, _ = _mats(wl)
    c = 1e-4
    op = _dev_op("rank1", A, None, c)
    a, b = wl.a, wl.b + c * A.n_rows
    for persist in (0, 2):
        persistent_mode(persist)
        r = P.logdet(op, a, b, 30, 12, seed=6, k=16, want_moments=True)
        mu = orc.moments(orc.Op("rank1", A, c), a, b, 30, 6, range(12), workers=4)
        _check_moments(r.moments, mu, A.n_rows)


def test_host_entry_arena_reuse_across_operators(orc):
    """cheb_logdet_host reuses (and grows) its per-thread device arenas across calls with
    operators of different sizes and modes; every result equals the device-operator call."""
    P.release_cache()
    cases = [("gmrf32", 8), ("btb_s", 8), ("gmrf32", 16), ("torus_s", 8)]
    for name, k in cases:
        wl = W.get_workload(name)
        A, At = _mats(wl)
        op = _dev_op(wl.mode, A, At, wl.r1_c)
        a, b = (wl.a, wl.b) if wl.a is not None else P.bounds_btb(op)
        rd = P.logdet(op, a, b, 12, 9, seed=3, k=k, want_moments=True)
        rh = P.logdet_host(wl.mode, A, a, b, 12, 9, seed=3, k=k, At=At, c=wl.r1_c, want_moments=True)
        assert np.array_equal(rd.moments, rh.moments) and rd.logdet == rh.logdet, name
    P.release_cache()


# ------------------------------------------------------------------ instantiations no other test reaches
def test_rank1_standard_tile_geometry_per_step(orc, persistent_mode):
    """Rank-1 on the standard tile geometry (cheb_step_kernel<64, RANK1, ..., RP = 0>): a 1024^2
    torus + c 11^T at k = 64 has a working set above half of L2, so neither the small-tile rule nor
    the persistent kernel applies.  Every probe against the oracle."""
    persistent_mode(1)
    N = 1024
    T = W.torus_laplacian(N)
    lam2 = 2.0 - 2.0 * math.cos(2.0 * math.pi / N)
    c = lam2 / (N * N)
    op = _dev_op("rank1", T, None, c)
    n, m = 24, 64
    P.profile_begin()
    r = P.logdet(op, lam2, 8.0, n, m, seed=13, k=64, want_moments=True)
    prof = P.profile_end()
    assert prof["persistent"][1] == 0 and prof["single"][1] == n  # per-step launches
    mu = orc.moments(orc.Op("rank1", T, c), lam2, 8.0, n, 13, range(m), workers=8)
    _check_moments(r.moments, mu, T.n_rows)
    g, _, _ = orc.gamma_from_moments(orc.coeffs_log(lam2, 8.0, n), mu)
    _check_gamma(r.logdet, g)


@pytest.fixture
def small_tiles_mode():
    yield P.set_small_tiles
    P.set_small_tiles(1)


@pytest.mark.parametrize("name", ["gmrf32", "gmrf_s", "torus_s"])
@pytest.mark.parametrize("k", [8, 64])
@pytest.mark.parametrize("dbl", [False, True])
def test_persistent_standard_geometry(orc, persistent_mode, small_tiles_mode, name, k, dbl):
    """cheb_persist_kernel<..., RP = 0> (persistent forced, small tiles off): vs the oracle and
    bit-identical to per-step launches on the same geometry."""
    small_tiles_mode(0)
    wl = W.get_workload(name)
    A, _ = _mats(wl)
    op = _dev_op(wl.mode, A, None, wl.r1_c)
    m = wl.num_probes
    P.set_doubling(dbl)
    try:
        out = {}
        for mode in (0, 2):
            persistent_mode(mode)
            out[mode] = P.moments(op, wl.a, wl.b, wl.degree, 0, m, wl.seed, k).cpu().numpy()
    finally:
        P.set_doubling(False)
    assert np.array_equal(out[0], out[2])
    mu = orc.moments(orc.Op(wl.mode, A, wl.r1_c), wl.a, wl.b, wl.degree, wl.seed, range(m), workers=4)
    _check_moments(out[2], mu, wl.d)


# ------------------------------------------------------------------ device errors on the async path
def test_timeout_status_poisons_and_raises(persistent_mode, monkeypatch):
    """A timed-out spin wait (injected: CHEB_INJECT_TIMEOUT raises the status bit the persistent
    kernel's bailout sets) must never come back as a normal value: cheb_moments' status epilogue
    turns the call's moments into NaN, the status word reports it, Estimator.run(check=True),
    ShardedEstimator.run() and cheb_logdet raise."""
    from paper_1503_06394_b200.dist import ShardedEstimator
    wl = W.get_workload("gmrf_s")
    A, _ = _mats(wl)
    op = _dev_op("csr", A)
    monkeypatch.setenv("CHEB_INJECT_TIMEOUT", "1")
    est = P.Estimator(op, wl.a, wl.b, 12, 16, 16, seed=3)
    gp, stats = est.run()
    assert P.workspace_status(est.workspace) & 1
    assert np.all(np.isnan(est.mu.cpu().numpy()))
    assert stats.cpu().numpy()[2] == 0.0
    with pytest.raises(P.ChebError) as ei:
        est.run(check=True)
    assert ei.value.code == -4
    with pytest.raises(P.ChebError) as ei:
        ShardedEstimator(op, wl.a, wl.b, 12, 16, 16, seed=3).run()
    assert ei.value.code == -4
    with pytest.raises(P.ChebError) as ei:
        P.logdet(op, wl.a, wl.b, 12, 16, seed=3, k=16)
    assert ei.value.code == -4
    monkeypatch.delenv("CHEB_INJECT_TIMEOUT")
    gp, stats = est.run(check=True)  # status word is per call: clean again
    assert P.workspace_status(est.workspace) & 3 == 0


def test_nonfinite_status_on_async_path():
    """b below lambda_max on the asynchronous path: status bit 1, check raises CL_ENONFINITE."""
    from paper_1503_06394_b200.dist import ShardedEstimator
    A = W.csr.from_coo(50, 50, np.arange(50), np.arange(50), np.full(50, 1e6))
    op = _dev_op("csr", A)
    est = P.Estimator(op, 0.5, 1.0, 200, 8, 8, seed=1)
    est.run()
    assert P.workspace_status(est.workspace) & 2
    with pytest.raises(P.ChebError) as ei:
        est.run(check=True)
    assert ei.value.code == -5
    with pytest.raises(P.ChebError):
        ShardedEstimator(op, 0.5, 1.0, 200, 8, 8, seed=1).run()


def test_dist_entry_point_one_rank_torchrun(orc):
    """`torchrun --nproc-per-node 1 -m paper_1503_06394_b200.dist` (the multi-GPU driver's launch
    path, NCCL process group of one rank): its estimate equals the oracle's on the same probes."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", "--master-port=29517", "-m", "paper_1503_06394_b200.dist",
           "--workload", "gmrf_s", "--k", "8"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    wl = W.get_workload("gmrf_s")
    A, _ = _mats(wl)
    og = orc.logdet(orc.Op("csr", A), wl.a, wl.b, wl.degree, wl.num_probes, wl.seed, workers=4)["gamma"]
    assert out["world"] == 1 and out["num_probes"] == wl.num_probes
    _check_gamma(out["logdet"], og)


@pytest.mark.parametrize("workload", ["gmrf32", "gmrf1000"])
def test_bench_two_ranks_functional(workload):
    """bench.py's N > 1 path (torchrun, probe shards, all-reduce of the moment table, max-over-ranks
    timing, e2e through cheb_moments_host) run as two ranks sharing cuda:0 over gloo
    (BENCH_SHARE_GPU=1: a functional check, not a measurement): the estimate is bit-identical to the
    one-rank line (adding the zero rows of the other shard is exact)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    flags = ["--workload", workload, "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-alt",
             "--no-weak"]
    out = {}
    for n in (1, 2):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr=127.0.0.1", f"--master-port={29530 + n}", "bench.py", "--gpus", str(n)] + flags
        env = dict(os.environ, BENCH_SHARE_GPU="1")
        r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600, env=env)
        assert r.returncode == 0, r.stderr[-2000:]
        out[n] = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert out[2]["n_gpus"] == 2 and out[2]["config"]["parallelism"] == "probe-dp2"
    assert out[2]["config"]["probes_per_gpu"] * 2 == out[1]["config"]["num_probes"]
    assert out[2]["config"]["gamma"] == out[1]["config"]["gamma"]
    assert out[2]["e2e"]["value"] > 0 and "functional_check_shared_gpu" in out[2]
