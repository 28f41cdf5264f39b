"""Pins of the CPU oracle against facts fixed by the paper and by mathematics
(closed forms, brute force, textbook identities) -- never against itself.

Each test names the part of oracle/cheb_oracle.c it pins and the passage it
follows.  A plausible mistake (dropped term, wrong sign/index, transposed
operand, missing factor 2, missing affine map) fails at least one of them.
"""
import math
import os

import numpy as np
import pytest

import workloads as W
from oracle import closed_forms as cf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_hex(name):
    out = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                out.append(int(line, 16))
    return out


# ---------------------------------------------------------------- generator (G6)
def test_splitmix64_published_stream(orc):
    """Flat counter t = p*d + i + 1 at p = 0 reproduces the published SplitMix64
    stream for seed 0 (tests/golden/splitmix64_seed0.txt)."""
    want = _golden_hex("splitmix64_seed0.txt")
    got = [orc.splitmix64(0, t) for t in (1, 2, 3)]
    assert got == want


def test_rademacher_entries_layout_balance(orc):
    """entries are +-1, balanced, deterministic; probe p row i uses
    bit 63 of the output at counter p*d+i+1."""
    d = 100_000
    v = orc.rademacher(5, 0, d)
    assert set(np.unique(v)) == {-1.0, 1.0}
    assert abs(v.mean()) <= 0.02
    assert np.array_equal(v, orc.rademacher(5, 0, d))
    # probe 3 of a d=17 problem: counter 3*17 + i + 1
    v3 = orc.rademacher(9, 3, 17)
    for i in range(17):
        z = orc.splitmix64(9, 3 * 17 + i + 1)
        assert v3[i] == (-1.0 if z >> 63 else 1.0)
    # distinct probes are (nearly) orthogonal: |v_p . v_q| ~ sqrt(d)
    w = orc.rademacher(5, 1, d)
    assert abs(v @ w) < 6 * math.sqrt(d)


# ---------------------------------------------------------------- §2.1 coefficients
def test_nodes(orc):
    """P:153 x_k = cos(pi(k+1/2)/(n+1)); S:207-210 examples."""
    assert abs(orc.cheb_nodes(0)[0]) < 1e-15
    x1 = orc.cheb_nodes(1)
    assert np.allclose(x1, [math.sqrt(2) / 2, -math.sqrt(2) / 2], atol=1e-15)
    x = orc.cheb_nodes(7)
    assert np.allclose(np.cos(8 * np.arccos(x)), 0.0, atol=1e-14)  # roots of T_{n+1}


@pytest.mark.parametrize("f,n,want", [
    (lambda x: x, 1, [0, 1]),
    (lambda x: np.ones_like(x), 3, [1, 0, 0, 0]),
    (lambda x: 2 * x * x - 1, 2, [0, 0, 1]),
    (lambda x: 4 * x ** 3 - 3 * x + 0.5, 5, [0.5, 0, 0, 1, 0, 0]),
])
def test_coeffs_reproduce_polynomials(orc, f, n, want):
    """interpolation at n+1 Chebyshev nodes reproduces polynomials of
    degree <= n exactly (catches a wrong c_0 halving or T recurrence)."""
    x = orc.cheb_nodes(n)
    c = orc.coeffs_from_values(f(x))
    assert np.allclose(c, want, atol=1e-13)


@pytest.mark.parametrize("a,b,n", [(0.2, 1.8, 30), (0.04, 1.96, 100),
                                   (6.023626e-4, 8.0, 1000), (4.0, 17.0, 50)])
def test_coeffs_log_equal_aliased_series(orc, a, b, n):
    """c_j of log on [a,b] (P:143-153 + G1/G4) equal the closed-form Chebyshev
    series a_j of log plus the first-kind-node aliasing terms:
    c_j = a_j + sum_q (-1)^q (a_{2q(n+1)-j} + a_{2q(n+1)+j}),  c_0 = a_0 + sum_q (-1)^q a_{2q(n+1)}."""
    c = orc.coeffs_log(a, b, n)
    qmax = 60
    A = cf.log_series_coeffs(a, b, 2 * qmax * (n + 1) + n + 1)
    want = A[: n + 1].copy()
    for q in range(1, qmax):
        for j in range(n + 1):
            hi = A[2 * q * (n + 1) + j]
            lo = 0.0 if j == 0 else A[2 * q * (n + 1) - j]
            want[j] += (-1) ** q * (hi + lo)
    # fp64 floor of an (n+1)-term sum of f(x_k) T_j(x_k): (n+1) eps max|f|
    fmax = max(abs(math.log(a)), abs(math.log(b)))
    assert np.abs(c - want).max() <= 2 * (n + 1) * 2.2e-16 * fmax


def test_coeffs_interpolate_at_nodes(orc):
    """p_n(x_k) = f(x_k) at every node (1e-10)."""
    a, b, n = 0.04, 1.96, 100
    c = orc.coeffs_log(a, b, n)
    for xk in orc.cheb_nodes(n):
        assert abs(orc.cheb_eval(c, xk) - math.log(((b - a) * xk + (b + a)) / 2)) < 1e-10


@pytest.mark.parametrize("delta", [0.05, 0.1, 0.2, 0.4])
@pytest.mark.parametrize("n", [5, 10, 20, 40])
def test_theorem3_envelope(orc, delta, n):
    """Theorem 3 / P:487: max |log(1-x) - p_n(x)| <= 20 log(2(1/d-1))/((K-1)K^n)
    on [delta, 1-delta]; equivalently our [a,b]=[delta,1-delta] form on [-1,1]."""
    c = orc.coeffs_log(delta, 1 - delta, n)
    xs = np.linspace(-1, 1, 2001)
    err = max(abs(orc.cheb_eval(c, x) - math.log(((1 - 2 * delta) * x + 1) / 2)) for x in xs)
    floor = 4 * (n + 1) * 2.2e-16 * abs(math.log(delta))  # fp64 evaluation floor
    assert err <= cf.theorem3_bound(delta, n) + floor


@pytest.mark.parametrize("a,b", [(0.2, 1.8), (0.04, 1.96), (3.0, 11.0)])
def test_delta_form_sign_identity(orc, a, b):
    """Reading G4: the paper's delta-form coefficients (Alg. 1 line 4, P:226:
    Chebyshev coefficients of log(1 - ((1-2 delta)x+1)/2)) with s = a+b,
    delta = a/s, satisfy c^delta_j = (-1)^j c_j, after moving log s into c_0."""
    n = 25
    s = a + b
    delta = a / s
    x = orc.cheb_nodes(n)
    cd = orc.coeffs_from_values(np.log(1 - ((1 - 2 * delta) * x + 1) / 2))
    c = orc.coeffs_log(a, b, n)
    sign = (-1.0) ** np.arange(n + 1)
    want = sign * cd
    want[0] += math.log(s)
    fmax = max(abs(math.log(a)), abs(math.log(b)), abs(math.log(delta)))
    assert np.abs(c - want).max() <= 2 * (n + 1) * 2.2e-16 * fmax


def test_cheb_eval_matches_trig_form(orc):
    """T_j(x) = cos(j arccos x): recurrence evaluation == closed form."""
    rng = np.random.default_rng(0)
    c = rng.standard_normal(40)
    for x in np.linspace(-1, 1, 23):
        assert abs(orc.cheb_eval(c, x) - cf.cheb_poly_closed(c, [x])[0]) < 1e-12


# ---------------------------------------------------------------- operator modes
def _dense_M(op):
    A = W.to_dense(op.A)
    if op.kind == "csr":
        return A
    if op.kind == "rank1":
        u = np.ones(op.d) if op.u is None else op.u
        return A + op.c * np.outer(u, u)
    return A.T @ A


def _ops_small():
    rng = np.random.default_rng(3)
    return [
        W.grid_gmrf(7, 0.2, 5),
        ("rank1", W.torus_laplacian(5), 0.3, None),
        ("rank1", W.torus_laplacian(4), 0.7, rng.standard_normal(16)),
        ("btb", W.random_nonsingular(30, 4)),
    ]


def _op(orc, spec):
    if isinstance(spec, tuple):
        if spec[0] == "rank1":
            return orc.Op("rank1", spec[1], spec[2], spec[3])
        return orc.Op("btb", spec[1])
    return orc.Op("csr", spec)


def test_apply_tilde_matches_dense(orc):
    """Ã x = (2/(b-a)) M x - ((b+a)/(b-a)) x for each operator mode, against a
    dense numpy product (catches a transposed B, a missing rank-1 term, a wrong
    affine map)."""
    rng = np.random.default_rng(1)
    for spec in _ops_small():
        op = _op(orc, spec)
        M = _dense_M(op)
        a, b = 0.3, 9.0
        x = rng.standard_normal(op.d)
        want = (2 / (b - a)) * (M @ x) - ((b + a) / (b - a)) * x
        got = orc.apply_tilde(op, a, b, x)
        assert np.allclose(got, want, rtol=1e-13, atol=1e-13)


def _tilde_eigs(eigs, a, b):
    return (2 * eigs - (b + a)) / (b - a)


def _basis_trace_moments(orc, op, a, b, n):
    mu = np.zeros(n + 1)
    e = np.zeros(op.d)
    for i in range(op.d):
        e[:] = 0
        e[i] = 1
        mu += orc.moments_vec(op, a, b, n, e)
    return mu


def test_basis_probes_grid_closed_form(orc):
    """Probes e_1..e_d turn the estimator into the exact trace:
    sum_i e_i^T T_j(Ã) e_i = sum_lambda T_j(lambda~) with closed-form grid
    eigenvalues and T_j in trigonometric form -- pins the recurrence, the
    factor 2, the w_{j-1} term and the affine map for every j (config 0)."""
    N, theta, n = 32, 0.2, 30
    a, b = 1 - 4 * theta, 1 + 4 * theta
    op = orc.Op("csr", W.grid_gmrf(N, theta))
    mu = _basis_trace_moments(orc, op, a, b, n)
    lt = _tilde_eigs(cf.grid_eigs(N, theta), a, b)
    want = np.array([cf.cheb_T(j, lt).sum() for j in range(n + 1)])
    assert np.abs(mu - want).max() < 1e-11 * op.d
    c = orc.coeffs_log(a, b, n)
    got = orc.gamma_from_moments(c, mu[None, :])[0]
    exact_poly = cf.cheb_poly_closed(c, lt).sum()
    assert abs(got - exact_poly) < 6e-13 * abs(exact_poly)


def test_basis_probes_torus_rank1_closed_form(orc):
    """Rank-1 mode: M = L + c 11^T on a 12x12 torus has the torus spectrum with
    the zero mode moved to c*N^2 (closed form)."""
    N, n = 12, 60
    lam2 = 2 - 2 * math.cos(2 * math.pi / N)
    c1 = lam2 / (N * N)
    a, b = lam2, 8.0
    op = orc.Op("rank1", W.torus_laplacian(N), c1)
    mu = _basis_trace_moments(orc, op, a, b, n)
    lt = _tilde_eigs(cf.torus_rank1_eigs(N, c1), a, b)
    want = np.array([cf.cheb_T(j, lt).sum() for j in range(n + 1)])
    assert np.abs(mu - want).max() < 1e-10 * op.d


@pytest.mark.parametrize("kind", ["csr", "rank1", "btb"])
def test_rademacher_quadratic_form_dense(orc, kind):
    """per-probe mu_j = v^T T_j(Ã) v with T_j(Ã) = Q T_j(Λ~) Q^T formed
    densely from an eigendecomposition and the trigonometric T_j."""
    if kind == "csr":
        op = orc.Op("csr", W.random_spd(60, 2))
    elif kind == "rank1":
        op = orc.Op("rank1", W.torus_laplacian(6), 0.05, np.linspace(0.5, 1.5, 36))
    else:
        op = orc.Op("btb", W.random_nonsingular(50, 5))
    M = _dense_M(op)
    lam, Q = np.linalg.eigh(M)
    a, b = lam.min() * 0.9, lam.max() * 1.1
    n = 24
    v = orc.rademacher(11, 2, op.d)
    mu = orc.moments_vec(op, a, b, n, v)
    lt = _tilde_eigs(lam, a, b)
    qv = Q.T @ v
    want = np.array([(qv * qv * cf.cheb_T(j, lt)).sum() for j in range(n + 1)])
    assert np.allclose(mu, want, rtol=1e-11, atol=1e-11 * op.d)


def test_degree_zero(orc):
    """n = 0 gives Gamma = c_0 * d exactly."""
    A = W.grid_gmrf(9, 0.1)
    r = orc.logdet(orc.Op("csr", A), 0.6, 1.4, 0, 5, 1)
    assert r["mu"].shape == (5, 1)
    assert np.all(r["mu"][:, 0] == 81.0)
    assert r["gamma"] == r["c"][0] * 81.0


def test_tilde_zero(orc):
    """M = ((a+b)/2) I gives Ã = 0, so mu_j = d T_j(0) = d cos(j pi/2) and
    Gamma_p = d (c_0 - c_2 + c_4 - ...)."""
    d, a, b, n = 50, 0.5, 2.5, 12
    I = W.csr.from_coo(d, d, np.arange(d), np.arange(d), np.full(d, (a + b) / 2))
    r = orc.logdet(orc.Op("csr", I), a, b, n, 3, 4)
    want_mu = d * np.round(np.cos(np.arange(n + 1) * np.pi / 2))
    assert np.all(r["mu"] == want_mu)
    c = r["c"]
    assert abs(r["gamma"] - d * sum(c[j] * (-1) ** (j // 2) for j in range(0, n + 1, 2))) < 1e-12 * d


def test_scalar_operator(orc):
    """M = sI: Gamma_p = d p_n((2s-(a+b))/(b-a)) ~ d log s (Theorem 3 bias)."""
    d, a, b, n, s = 40, 0.5, 3.0, 40, 1.7
    I = W.csr.from_coo(d, d, np.arange(d), np.arange(d), np.full(d, s))
    r = orc.logdet(orc.Op("csr", I), a, b, n, 2, 9)
    c = r["c"]
    xt = (2 * s - (a + b)) / (b - a)
    assert abs(r["gamma"] - d * cf.cheb_poly_closed(c, [xt])[0]) < 1e-12 * d
    assert abs(r["gamma"] - d * math.log(s)) < d * cf.theorem3_bound(a / (a + b), n)


def test_cayley_rank1(orc):
    """Rank-1 spanning-tree route (BJ configs[1]): K_n Laplacian + 1*11^T = nI, so
    log tau = logdet M - log(c n^2) = (n-2) log n (Cayley)."""
    n_v = 7
    op = orc.Op("rank1", W.complete_graph_laplacian(n_v), 1.0)
    r = orc.logdet(op, n_v - 1.0, n_v + 1.0, 30, 4, 2)
    log_tau = r["gamma"] - math.log(1.0 * n_v * n_v)
    assert abs(log_tau - (n_v - 2) * math.log(n_v)) < 1e-12


# ---------------------------------------------------------------- closed forms themselves
def test_grid_closed_form_equals_cholesky():
    """log det = 2 sum log L_ii on a 12x9 grid equals the closed form;
    theta -> -theta leaves it unchanged (bipartite grid, reading G15)."""
    A = W.to_dense(W.grid_gmrf(12, 0.23, 9))
    L = np.linalg.cholesky(A)
    chol = 2 * np.log(np.diag(L)).sum()
    assert abs(chol - cf.grid_logdet(12, 0.23, 9)) < 1e-12 * abs(chol)
    assert abs(cf.grid_logdet(12, 0.23, 9) - cf.grid_logdet(12, -0.23, 9)) < 1e-12
    assert abs(cf.grid_logdet(32, 0.2) - (-99.7972847113791)) < 1e-11


@pytest.mark.parametrize("N,tau", [(3, 11664), (4, 42467328)])
def test_torus_matrix_tree(N, tau):
    """Matrix-tree theorem: det of the reduced Laplacian == closed form."""
    L = W.to_dense(W.torus_laplacian(N))
    det = np.linalg.det(L[1:, 1:])
    assert abs(det - tau) < 1e-6 * tau
    assert abs(cf.torus_log_tau(N) - math.log(tau)) < 1e-12


def test_rank1_route_matches_reduced_laplacian():
    """log tau = logdet(L + c 11^T) - log(c N^2) == log det L(i*) (6x6 torus)."""
    N = 6
    L = W.to_dense(W.torus_laplacian(N))
    c = 0.37
    s1, ld = np.linalg.slogdet(L + c * np.ones_like(L))
    assert s1 > 0
    red = np.linalg.slogdet(L[1:, 1:])[1]
    assert abs((ld - math.log(c * N ** 4)) - red) < 1e-10


# ---------------------------------------------------------------- estimator statistics
def test_estimate_config0_vs_exact(orc):
    """Config 0 (BJ.configs[0]): Gamma with m = 64 probes lies within 4 stderr of
    the exact log det; polynomial bias <= Lemma 1 bound."""
    wl = W.get_workload("gmrf32")
    A, _ = wl.matrices()
    r = orc.logdet(orc.Op("csr", A), wl.a, wl.b, wl.degree, wl.num_probes, wl.seed, workers=4)
    exact = cf.grid_logdet(32, 0.2)
    assert abs(r["gamma"] - exact) <= 4 * r["stderr"]
    lt = _tilde_eigs(cf.grid_eigs(32, 0.2), wl.a, wl.b)
    bias = abs(cf.cheb_poly_closed(r["c"], lt).sum() - exact)
    assert bias <= wl.d * cf.theorem3_bound(wl.a / (wl.a + wl.b), wl.degree)


def test_variance_law(orc):
    """P:187-190 (reading G8): per-sample Var[v^T P v] = 2(||P||_F^2 - sum P_ii^2),
    E = tr P, with P = p_n(Ã) formed densely.  1280 probes on a 16x16 grid."""
    N, theta, n, m = 16, 0.22, 20, 1280
    a, b = 1 - 4 * theta, 1 + 4 * theta
    A = W.grid_gmrf(N, theta)
    op = orc.Op("csr", A)
    r = orc.logdet(op, a, b, n, m, 3, workers=4)
    lam, Q = np.linalg.eigh(W.to_dense(A))
    P = (Q * cf.cheb_poly_closed(r["c"], _tilde_eigs(lam, a, b))) @ Q.T
    var = 2 * ((P * P).sum() - (np.diag(P) ** 2).sum())
    sd = math.sqrt(var)
    gp = r["gamma_p"]
    assert abs(gp.mean() - np.trace(P)) < 4 * sd / math.sqrt(m)
    ratio = gp.std(ddof=1) / sd
    assert 0.9 < ratio < 1.1  # chi^2 band for 1279 dof is ~ +-4%
    # the oracle's reported standard error is the estimator's sd, i.e. the per-sample sd of the
    # variance law over sqrt(m) (P:187-190 with G8's 1/m): stderr * sqrt(m) ~ sqrt(2(|P|_F^2 - sum P_ii^2))
    assert 0.9 < r["stderr"] * math.sqrt(m) / sd < 1.1
    assert 0.9 < r["stderr"] / (sd / math.sqrt(m)) < 1.1


def test_stderr_two_probes_closed_form(orc):
    """m = 2: the sample sd of {x, y} is |x - y|/sqrt(2), so the standard error of the mean is
    |x - y|/2 exactly; m = 1 reports 0 (a single probe has no spread estimate)."""
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    r = orc.logdet(orc.Op("csr", A), wl.a, wl.b, 15, 2, 5, workers=2)
    x, y = r["gamma_p"]
    assert abs(r["stderr"] - abs(x - y) / 2) <= 1e-15 * abs(x - y)
    assert abs(r["gamma"] - (x + y) / 2) <= 1e-15 * abs(x + y)
    assert orc.logdet(orc.Op("csr", A), wl.a, wl.b, 15, 1, 5)["stderr"] == 0.0


# ---------------------------------------------------------------- Alg. 2 setup bounds
def test_bounds_btb_diagonal(orc):
    """Diagonal B: Johnson bound = min |b_ii|, ||B||_1||B||_inf = max |b_ii|^2."""
    d = np.array([1.5, -3.0, 2.0, 0.7])
    B = W.csr.from_coo(4, 4, np.arange(4), np.arange(4), d)
    a, b = orc.bounds_btb(B)
    assert a == 0.7 ** 2 and b == 9.0


def test_bounds_btb_enclose_singular_values(orc):
    """[a,b] encloses sigma(B)^2, checked by SVD; values vs brute force."""
    B = W.random_nonsingular(200, 9)
    a, b = orc.bounds_btb(B)
    D = W.to_dense(B)
    s = np.linalg.svd(D, compute_uv=False)
    assert a <= s.min() ** 2 and s.max() ** 2 <= b
    off = np.abs(D - np.diag(np.diag(D)))
    jb = (np.abs(np.diag(D)) - 0.5 * (off.sum(1) + off.sum(0))).min()
    assert abs(a - jb ** 2) < 1e-13 and abs(b - np.abs(D).sum(0).max() * np.abs(D).sum(1).max()) < 1e-12


def test_btb_triangular_logabsdet(orc):
    """Alg. 2: log|det B| = 1/2 log det B^T B; for triangular B it is
    d log 3 exactly.  Basis-probe trace of p_n(B^T B~) within Lemma 1's bias."""
    d, n = 120, 40
    B = W.triangular_b(d)
    a, b = orc.bounds_btb(B)
    op = orc.Op("btb", B)
    mu = _basis_trace_moments(orc, op, a, b, n)
    c = orc.coeffs_log(a, b, n)
    half = 0.5 * orc.gamma_from_moments(c, mu[None, :])[0]
    assert abs(half - d * math.log(3)) <= 0.5 * d * cf.theorem3_bound(a / (a + b), n) + 1e-10 * d


# ---------------------------------------------------------------- Taylor baseline
def test_taylor_scalar_operator_closed_form(orc):
    """M = sigma I: mu_k = d (1 - sigma/s)^k, and the estimate obeys the truncated-series
    bound |Gamma/d - log sigma| <= x^(n+1) / ((n+1)(1-x)), x = 1 - sigma/s."""
    d, sig, s, n = 30, 0.7, 2.0, 25
    I = W.csr.from_coo(d, d, np.arange(d), np.arange(d), np.full(d, sig))
    r = orc.taylor_logdet(orc.Op("csr", I), s, n, 3, 5)
    x = 1 - sig / s
    want = d * x ** np.arange(n + 1)
    assert np.allclose(r["mu"], want, rtol=1e-13, atol=0)
    assert abs(r["gamma"] / d - math.log(sig)) <= x ** (n + 1) / ((n + 1) * (1 - x)) + 1e-14
    assert r["c"][0] == math.log(s) and r["c"][3] == -1.0 / 3


def test_taylor_basis_probes_grid_closed_form(orc):
    """Standard-basis probes: sum_i e_i^T A^k e_i = sum_lambda (1 - lambda/s)^k with
    closed-form grid eigenvalues, every k (pins the power recurrence and the 1/s scaling)."""
    N, theta, n = 12, 0.2, 20
    s = 2.0  # = a + b for [0.2, 1.8]
    op = orc.Op("csr", W.grid_gmrf(N, theta))
    mu = np.zeros(n + 1)
    e = np.zeros(op.d)
    for i in range(op.d):
        e[:] = 0
        e[i] = 1
        mu += orc.power_moments_vec(op, s, n, e)
    lam = cf.grid_eigs(N, theta)
    want = np.array([((1 - lam / s) ** k).sum() for k in range(n + 1)])
    assert np.abs(mu - want).max() < 1e-12 * op.d


def test_chebyshev_beats_taylor_exact_traces(orc):
    """Fig. 1(d), noise-free form: with exact traces (basis probes) the
    Chebyshev polynomial's log-det error is far below the Taylor series' at equal degree."""
    N, theta, n = 16, 0.22, 20
    a, b = 1 - 4 * theta, 1 + 4 * theta
    A = W.grid_gmrf(N, theta)
    exact = cf.grid_logdet(N, theta)
    lt = (2 * cf.grid_eigs(N, theta) - (a + b)) / (b - a)
    cheb = cf.cheb_poly_closed(orc.coeffs_log(a, b, n), lt).sum()
    x = 1 - cf.grid_eigs(N, theta) / (a + b)
    taylor = (N * N) * math.log(a + b) + sum(-(x ** k).sum() / k for k in range(1, n + 1))
    assert abs(cheb - exact) < 0.01 * abs(taylor - exact)


# ---------------------------------------------------------------- power iteration
def test_affine_power_moments_diagonal_closed_form(orc):
    """M = diag(lam): v^T (alpha M - beta I)^j v = sum_i (alpha lam_i - beta)^j exactly (v_i^2 = 1)."""
    lam = np.linspace(0.3, 2.9, 41)
    d = lam.size
    M = W.csr.from_coo(d, d, np.arange(d), np.arange(d), lam)
    alpha, beta, n = 0.31, -0.2, 12
    v = orc.rademacher(4, 1, d)
    mu = orc.affine_power_moments_vec(orc.Op("csr", M), alpha, beta, n, v)
    want = np.array([((alpha * lam - beta) ** j).sum() for j in range(n + 1)])
    assert np.allclose(mu, want, rtol=1e-13)


def test_power_iteration_grid_extremes_and_gershgorin(orc):
    """Block power iteration recovers the closed-form extreme eigenvalues of the grid
    precision, and the Gershgorin bound equals 1 + 4 theta (interior rows)."""
    N, theta = 14, 0.21
    A = W.grid_gmrf(N, theta)
    s = orc.gershgorin(A)
    assert abs(s - (1 + 4 * theta)) < 1e-15
    op = orc.Op("csr", A)
    hi = orc.affine_power_moments(op, 1 / s, 0.0, 400, 7, range(6)).sum(axis=0)
    lo = orc.affine_power_moments(op, -1 / s, -1.0, 400, 7, range(6)).sum(axis=0)
    lam = cf.grid_eigs(N, theta)
    assert abs(s * hi[-1] / hi[-2] - lam.max()) < 2e-3
    assert abs(s * (1 - lo[-1] / lo[-2]) - lam.min()) < 2e-3


# ---------------------------------------------------------------- GMRF likelihood
def test_quadform_matches_dense(orc):
    A = W.grid_gmrf(9, 0.2, 7)
    x = np.random.default_rng(5).standard_normal(63)
    D = W.to_dense(A)
    assert abs(orc.quadform(A, x) - x @ D @ x) < 1e-12 * abs(x @ D @ x)


# ---------------------------------------------------------------- Lanczos spectral interval (f4, G26)
def _tridiag_csr(diag, off):
    d = diag.size
    r = np.concatenate([np.arange(d), np.arange(d - 1), np.arange(1, d)])
    c = np.concatenate([np.arange(d), np.arange(1, d), np.arange(d - 1)])
    v = np.concatenate([diag, off, off])
    return W.csr.from_coo(d, d, r, c, v)


def test_lanczos_reproduces_tridiagonal_from_e1(orc):
    """Textbook identity: Lanczos on a symmetric tridiagonal matrix with positive off-diagonal,
    started at e_1, returns that matrix (here Ã = alpha T - beta I of it)."""
    rng = np.random.default_rng(4)
    d = 30
    diag, off = rng.uniform(1.0, 3.0, d), rng.uniform(0.1, 0.5, d - 1)
    T = _tridiag_csr(diag, off)
    a, b = 0.5, 4.5
    al, be = orc.lanczos(orc.Op("csr", T), a, b, 12, v=np.eye(d)[0])
    alpha, beta = 2 / (b - a), (b + a) / (b - a)
    assert np.allclose(al, alpha * diag[:12] - beta, rtol=0, atol=1e-14)
    assert np.allclose(be, alpha * off[:12], rtol=0, atol=1e-14)


def test_lanczos_finds_distinct_eigenvalues_exactly(orc):
    """M diagonal with 6 distinct eigenvalues (each repeated): the Krylov space of any start vector
    has dimension 6, so after 6 steps the Ritz values are exactly those eigenvalues and the process
    stops (beta_6 = 0)."""
    vals = np.array([0.3, 0.7, 1.1, 2.0, 2.9, 3.5])
    diag = np.repeat(vals, 17)
    D = W.csr.from_coo(diag.size, diag.size, np.arange(diag.size), np.arange(diag.size), diag)
    a, b = 0.0, 4.0
    al, be = orc.lanczos(orc.Op("csr", D), a, b, 6, seed=3, p=0)
    th, r = orc.ritz(al, be)
    lam = (th + (b + a) / (b - a)) * (b - a) / 2
    assert np.allclose(lam, vals, atol=1e-12)
    assert be[5] < 1e-12 and np.all(r < 1e-12)


def test_lanczos_gauss_quadrature_matches_moments(orc):
    """Gauss quadrature from T_N (nodes theta_i, weights s_{1,i}^2) integrates polynomials of degree
    <= 2N-1 exactly against the probe's spectral measure: sum_i w_i T_j(theta_i) = mu_j / mu_0 with
    mu_j = v^T T_j(Ã) v from the (independently pinned) moment routine."""
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    op = orc.Op("csr", A)
    N = 12
    v = orc.rademacher(7, 0, wl.d)
    al, be = orc.lanczos(op, wl.a, wl.b, N, v=v)
    T = np.diag(al) + np.diag(be[:-1], 1) + np.diag(be[:-1], -1)
    th, S = np.linalg.eigh(T)
    w = S[0, :] ** 2
    mu = orc.moments_vec(op, wl.a, wl.b, 2 * N - 1, v)
    quad = np.array([np.sum(w * np.cos(j * np.arccos(np.clip(th, -1, 1)))) for j in range(2 * N)])
    assert np.allclose(quad * mu[0], mu, rtol=0, atol=1e-11 * wl.d)


def test_lanczos_grid_extremes_and_interval(orc):
    """20x20 GMRF grid (closed-form spectrum): the extreme Ritz values converge to lambda_min /
    lambda_max, each residual bound covers the distance to the eigenvalue, and the interval
    spectrum_bounds returns encloses the whole spectrum."""
    N, theta = 20, 0.2
    A = W.grid_gmrf(N, theta)
    lam = cf.grid_eigs(N, theta)
    lo, hi = 0.0, orc.gershgorin(A)
    sb = orc.spectrum_bounds(orc.Op("csr", A), lo, hi, 80, 5, range(4))
    assert abs(sb["lambda_min"] - lam.min()) < 1e-9 and abs(sb["lambda_max"] - lam.max()) < 1e-9
    assert sb["lambda_min"] >= lam.min() - 1e-12 and sb["lambda_max"] <= lam.max() + 1e-12  # Ritz: inside
    assert sb["a"] <= lam.min() and sb["b"] >= lam.max() and sb["b"] <= hi
    al, be = sb["jacobi"][0]
    th, r = orc.ritz(al, be)
    lt = 2 / hi * lam - 1
    for t, rr in zip(th, r):  # Kahan: some eigenvalue within each residual bound
        assert np.min(np.abs(lt - t)) <= rr + 1e-12
