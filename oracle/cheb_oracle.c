/*
 * cheb_oracle.c -- plain, slow, fp64 CPU ORACLE for the Chebyshev-Hutchinson
 * log-determinant estimator (arXiv 1503.06394).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_1503_06394_b200/csrc); neither includes the other.
 *
 * Compiled with plain `gcc -O2 -ffp-contract=off` (no FMA contraction, no
 * SIMD intrinsics).  Every routine cites the PAPER.md passage it follows
 * ("P:n" = line n of PAPER.md) and the DESIGN.md reading ("G#") where the
 * paper is garbled or silent.
 *
 * Parity pins: every function here is pinned by tests/test_oracle_pins.py
 * (closed forms, brute force, textbook identities); none is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ENOMEM (-3)
#define ORC_ENONFINITE (-5)

#define ORC_OP_CSR 0
#define ORC_OP_RANK1 1
#define ORC_OP_BTB 2

typedef struct {
    int64_t n_rows, n_cols;
    const int64_t *row_ptr;
    const int32_t *col_idx;
    const double *val;
} orc_csr;

typedef struct {
    int32_t kind;      /* ORC_OP_* */
    orc_csr A;         /* A (csr, rank1) or B (btb) */
    double r1_c;       /* rank-1 weight c */
    const double *r1_u;/* rank-1 vector u, NULL = all ones */
} orc_op;

/* ---------------------------------------------------------------------- */
/* §2.1 Chebyshev approximation                                 */
/* ---------------------------------------------------------------------- */

/* Nodes x_k = cos(pi (k + 1/2) / (n + 1)), k = 0..n. */
void orc_cheb_nodes(int32_t n, double *x)
{
    for (int32_t k = 0; k <= n; k++)
        x[k] = cos(M_PI * ((double)k + 0.5) / ((double)n + 1.0));
}

/* c_i = 1/(n+1) sum_k f(x_k) T_0(x_k)          (i = 0)
 * c_i = 2/(n+1) sum_k f(x_k) T_i(x_k)          (i >= 1)
 * with T_0 = 1, T_1 = x, T_{i+1} = 2x T_i - T_{i-1}.
 * fx[k] = f(x_k) at the nodes of orc_cheb_nodes. */
void orc_cheb_coeffs_from_values(int32_t n, const double *fx, double *c)
{
    double *x = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    orc_cheb_nodes(n, x);
    for (int32_t i = 0; i <= n; i++) {
        double s = 0.0;
        for (int32_t k = 0; k <= n; k++) {
            /* T_i(x_k) by the three-term recurrence */
            double t0 = 1.0, t1 = x[k], ti;
            if (i == 0) ti = t0;
            else if (i == 1) ti = t1;
            else {
                for (int32_t q = 1; q < i; q++) {
                    double t2 = 2.0 * x[k] * t1 - t0;
                    t0 = t1;
                    t1 = t2;
                }
                ti = t1;
            }
            s += fx[k] * ti;
        }
        c[i] = (i == 0 ? 1.0 : 2.0) / ((double)n + 1.0) * s;
    }
    free(x);
}

/* Coefficients of f(x) = log( ((b-a) x + (b+a)) / 2 ), x in [-1,1]:
 * log evaluated on [a,b] through the affine map g(x) = ((b-a)x+(b+a))/2.
 * This is Algorithm 1's line "c_i <- i-th coefficient of ... log(1 - ((1-2d)x+1)/2)"
 * in the [a,b] parameterisation (readings G1, G3, G4). */
int32_t orc_cheb_coeffs_log(double a, double b, int32_t n, double *c)
{
    if (!(a > 0.0) || !(b > a) || !isfinite(a) || !isfinite(b) || n < 0 || !c)
        return ORC_EINVAL;
    double *x = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *fx = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    orc_cheb_nodes(n, x);
    for (int32_t k = 0; k <= n; k++)
        fx[k] = log(((b - a) * x[k] + (b + a)) / 2.0);
    orc_cheb_coeffs_from_values(n, fx, c);
    free(x);
    free(fx);
    return ORC_OK;
}

/* p_n(x) = sum_j c_j T_j(x), T_j by the recurrence. */
double orc_cheb_eval(int32_t n, const double *c, double x)
{
    double t0 = 1.0, t1 = x, s = c[0];
    if (n >= 1) s += c[1] * t1;
    for (int32_t j = 2; j <= n; j++) {
        double t2 = 2.0 * x * t1 - t0;
        s += c[j] * t2;
        t0 = t1;
        t1 = t2;
    }
    return s;
}

/* ---------------------------------------------------------------------- */
/* §2.2 Rademacher probes, P:184-186 (generator unspecified: reading G6)   */
/* ---------------------------------------------------------------------- */

/* SplitMix64 output at flat counter t of the stream seeded `seed`:
 * z = seed + t*0x9E3779B97F4A7C15; two xor-shift-multiply rounds; final xor-shift. */
uint64_t orc_splitmix64(uint64_t seed, uint64_t t)
{
    uint64_t z = seed + t * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Probe p, entry i: counter t = p*d + i + 1; v = -1 if bit 63 set, else +1. */
void orc_rademacher(uint64_t seed, int64_t p, int64_t d, double *v)
{
    for (int64_t i = 0; i < d; i++) {
        uint64_t z = orc_splitmix64(seed, (uint64_t)p * (uint64_t)d + (uint64_t)i + 1ULL);
        v[i] = (z >> 63) ? -1.0 : 1.0;
    }
}

/* ---------------------------------------------------------------------- */
/* Operator application ("relies on matrix-vector multiplications",       */
/* P:191-198)                                         */
/* ---------------------------------------------------------------------- */

/* y = A x, A in CSR. */
static void csr_mv(const orc_csr *A, const double *x, double *y)
{
    for (int64_t i = 0; i < A->n_rows; i++) {
        double s = 0.0;
        for (int64_t e = A->row_ptr[i]; e < A->row_ptr[i + 1]; e++)
            s += A->val[e] * x[A->col_idx[e]];
        y[i] = s;
    }
}

/* y = A^T x by scattering over the rows of A (no transpose needed). */
static void csr_tmv(const orc_csr *A, const double *x, double *y)
{
    for (int64_t j = 0; j < A->n_cols; j++) y[j] = 0.0;
    for (int64_t i = 0; i < A->n_rows; i++)
        for (int64_t e = A->row_ptr[i]; e < A->row_ptr[i + 1]; e++)
            y[A->col_idx[e]] += A->val[e] * x[i];
}

/* Compensated (Neumaier) sum of x[i]*y[i]: a plain dot product whose rounding
 * error does not grow with d (SURVEY §8(c) "rounding noise from the dot
 * products"). */
static double dot(const double *x, const double *y, int64_t d)
{
    double s = 0.0, comp = 0.0;
    for (int64_t i = 0; i < d; i++) {
        double t = x[i] * y[i];
        double u = s + t;
        if (fabs(s) >= fabs(t)) comp += (s - u) + t;
        else comp += (t - u) + s;
        s = u;
    }
    return s + comp;
}

static int64_t op_dim(const orc_op *op) { return op->A.n_cols; }

/* y = M x for the three operator modes (SURVEY §8 preamble):
 *   csr:   M = A
 *   rank1: M = A + c u u^T               (BASELINE configs[1])
 *   btb:   M = B^T B, applied as B^T (B x), never formed (Alg. 2)
 * tmp: scratch of length d (btb only). */
void orc_apply_M(const orc_op *op, const double *x, double *y, double *tmp)
{
    int64_t d = op_dim(op);
    if (op->kind == ORC_OP_BTB) {
        csr_mv(&op->A, x, tmp);
        csr_tmv(&op->A, tmp, y);
        return;
    }
    csr_mv(&op->A, x, y);
    if (op->kind == ORC_OP_RANK1) {
        double s = 0.0, comp = 0.0;  /* u^T x, compensated */
        for (int64_t k = 0; k < d; k++) {
            double t = (op->r1_u ? op->r1_u[k] : 1.0) * x[k];
            double u = s + t;
            if (fabs(s) >= fabs(t)) comp += (s - u) + t;
            else comp += (t - u) + s;
            s = u;
        }
        s += comp;
        for (int64_t i = 0; i < d; i++)
            y[i] += op->r1_c * (op->r1_u ? op->r1_u[i] : 1.0) * s;
    }
}

/* y = Ã x with Ã = alpha M - beta I, alpha = 2/(b-a), beta = (b+a)/(b-a):
 * the affine map g^{-1} of [a,b] onto [-1,1] applied to M (reading G1/G3,
 * Lemma 1 "p_n denotes p_n o g^{-1}"). */
int32_t orc_apply_tilde(const orc_op *op, double a, double b, const double *x, double *y)
{
    int64_t d = op_dim(op);
    double alpha = 2.0 / (b - a), beta = (b + a) / (b - a);
    double *mx = (double *)malloc(sizeof(double) * (size_t)d);
    double *tmp = (double *)malloc(sizeof(double) * (size_t)d);
    if (!mx || !tmp) { free(mx); free(tmp); return ORC_ENOMEM; }
    orc_apply_M(op, x, mx, tmp);
    for (int64_t i = 0; i < d; i++) y[i] = alpha * mx[i] - beta * x[i];
    free(mx);
    free(tmp);
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* Algorithm 1 inner loop for ONE probe vector v:              */
/*   w_0 = v, w_1 = Ã v, w_{j+1} = 2 Ã w_j - w_{j-1} */
/*   mu_j = v^T w_j  (scalar moments; reading G7)                           */
/* Reading G2: the c_1 term is included whenever n >= 1.                    */
/* ---------------------------------------------------------------------- */
int32_t orc_moments_vec(const orc_op *op, double a, double b, int32_t n,
                        const double *v, double *mu)
{
    if (!(a > 0.0) || !(b > a) || n < 0) return ORC_EINVAL;
    int64_t d = op_dim(op);
    double alpha = 2.0 / (b - a), beta = (b + a) / (b - a);
    double *w0 = (double *)malloc(sizeof(double) * (size_t)d);
    double *w1 = (double *)malloc(sizeof(double) * (size_t)d);
    double *mx = (double *)malloc(sizeof(double) * (size_t)d);
    double *tmp = (double *)malloc(sizeof(double) * (size_t)d);
    if (!w0 || !w1 || !mx || !tmp) {
        free(w0); free(w1); free(mx); free(tmp);
        return ORC_ENOMEM;
    }
    /* w_0 = v; mu_0 = v^T v */
    for (int64_t i = 0; i < d; i++) w0[i] = v[i];
    mu[0] = dot(v, w0, d);
    if (n >= 1) {
        /* w_1 = Ã v */
        orc_apply_M(op, w0, mx, tmp);
        for (int64_t i = 0; i < d; i++) w1[i] = alpha * mx[i] - beta * w0[i];
        mu[1] = dot(v, w1, d);
        for (int32_t j = 2; j <= n; j++) {
            /* w_2 = 2 Ã w_1 - w_0, stored over w_0; then (w_0, w_1) <- (w_1, w_2) */
            orc_apply_M(op, w1, mx, tmp);
            for (int64_t i = 0; i < d; i++)
                w0[i] = 2.0 * (alpha * mx[i] - beta * w1[i]) - w0[i];
            mu[j] = dot(v, w0, d);
            double *t = w0; w0 = w1; w1 = t;
        }
    }
    int32_t rc = ORC_OK;
    for (int32_t j = 0; j <= n; j++)
        if (!isfinite(mu[j])) rc = ORC_ENONFINITE;
    free(w0); free(w1); free(mx); free(tmp);
    return rc;
}

/* Moments of Rademacher probe p (global index) -- Algorithm 1 line
 * "Draw a Rademacher random vector v" with the G6 generator. */
int32_t orc_moments_probe(const orc_op *op, double a, double b, int32_t n,
                          uint64_t seed, int64_t p, double *mu)
{
    int64_t d = op_dim(op);
    double *v = (double *)malloc(sizeof(double) * (size_t)d);
    if (!v) return ORC_ENOMEM;
    orc_rademacher(seed, p, d, v);
    int32_t rc = orc_moments_vec(op, a, b, n, v, mu);
    free(v);
    return rc;
}

/* Gamma_p = sum_{j=0}^{n} c_j mu_j, ascending j (reading G7). */
double orc_gamma_probe(int32_t n, const double *c, const double *mu)
{
    double s = 0.0;
    for (int32_t j = 0; j <= n; j++) s += c[j] * mu[j];
    return s;
}

/* ---------------------------------------------------------------------- */
/* Spectral interval of B^T B for Algorithm 2:                  */
/*   sigma_max^2 <= ||B||_1 ||B||_inf                          */
/*   sigma_min >= min_i (|b_ii| - (r_i + c_i)/2)  (Johnson's lower bound,   */
/*   for diagonally dominant B, "diagonal-dominant matrices")    */
/*   r_i / c_i = off-diagonal absolute row / column sums.                   */
/* Returns ORC_EINVAL if the Johnson bound is not positive.                 */
/* ---------------------------------------------------------------------- */
int32_t orc_bounds_btb(const orc_csr *B, double *a_out, double *b_out)
{
    int64_t d = B->n_rows;
    if (B->n_cols != d) return ORC_EINVAL;
    double *diag = (double *)calloc((size_t)d, sizeof(double));
    double *roff = (double *)calloc((size_t)d, sizeof(double));
    double *coff = (double *)calloc((size_t)d, sizeof(double));
    double *rabs = (double *)calloc((size_t)d, sizeof(double));
    double *cabs = (double *)calloc((size_t)d, sizeof(double));
    if (!diag || !roff || !coff || !rabs || !cabs) {
        free(diag); free(roff); free(coff); free(rabs); free(cabs);
        return ORC_ENOMEM;
    }
    for (int64_t i = 0; i < d; i++) {
        for (int64_t e = B->row_ptr[i]; e < B->row_ptr[i + 1]; e++) {
            int64_t j = B->col_idx[e];
            double x = fabs(B->val[e]);
            rabs[i] += x;
            cabs[j] += x;
            if (j == i) diag[i] = x;
            else { roff[i] += x; coff[j] += x; }
        }
    }
    double norm1 = 0.0, norminf = 0.0, smin = INFINITY;
    for (int64_t i = 0; i < d; i++) {
        if (cabs[i] > norm1) norm1 = cabs[i];
        if (rabs[i] > norminf) norminf = rabs[i];
        double s = diag[i] - 0.5 * (roff[i] + coff[i]);
        if (s < smin) smin = s;
    }
    free(diag); free(roff); free(coff); free(rabs); free(cabs);
    if (!(smin > 0.0)) return ORC_EINVAL;
    *a_out = smin * smin;
    *b_out = norm1 * norminf;
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* Taylor baseline: "other polynomial approximations, e.g.  */
/* Taylor, can also be used", the comparison of Fig. 1(d)       */
/* (P:633-638).  log det M = d log s + tr log(I - A), A = I - M/s, with     */
/* log(1 - x) = -sum_{k>=1} x^k / k truncated at k = n; the traces come     */
/* from the power recurrence w_k = A w_{k-1} (reading G24: s = a + b).      */
/* ---------------------------------------------------------------------- */
int32_t orc_taylor_coeffs(double s, int32_t n, double *c)
{
    if (!(s > 0.0) || n < 0 || !c) return ORC_EINVAL;
    c[0] = log(s);
    for (int32_t k = 1; k <= n; k++) c[k] = -1.0 / (double)k;
    return ORC_OK;
}

/* mu_k = v^T A^k v, k = 0..n, A = I - M/s. */
int32_t orc_power_moments_vec(const orc_op *op, double s, int32_t n, const double *v, double *mu)
{
    if (!(s > 0.0) || n < 0) return ORC_EINVAL;
    int64_t d = op_dim(op);
    double *w = (double *)malloc(sizeof(double) * (size_t)d);
    double *mx = (double *)malloc(sizeof(double) * (size_t)d);
    double *tmp = (double *)malloc(sizeof(double) * (size_t)d);
    if (!w || !mx || !tmp) { free(w); free(mx); free(tmp); return ORC_ENOMEM; }
    for (int64_t i = 0; i < d; i++) w[i] = v[i];
    mu[0] = dot(v, w, d);
    for (int32_t k = 1; k <= n; k++) {
        orc_apply_M(op, w, mx, tmp);
        for (int64_t i = 0; i < d; i++) w[i] = w[i] - mx[i] / s;  /* w <- (I - M/s) w */
        mu[k] = dot(v, w, d);
    }
    int32_t rc = ORC_OK;
    for (int32_t k = 0; k <= n; k++)
        if (!isfinite(mu[k])) rc = ORC_ENONFINITE;
    free(w); free(mx); free(tmp);
    return rc;
}

int32_t orc_power_moments_probe(const orc_op *op, double s, int32_t n, uint64_t seed, int64_t p, double *mu)
{
    int64_t d = op_dim(op);
    double *v = (double *)malloc(sizeof(double) * (size_t)d);
    if (!v) return ORC_ENOMEM;
    orc_rademacher(seed, p, d, v);
    int32_t rc = orc_power_moments_vec(op, s, n, v, mu);
    free(v);
    return rc;
}

/* ---------------------------------------------------------------------- */
/* Spectral bounds by power iteration ("one can  */
/* run the power iteration to estimate a better bound").                   */
/*   mu_j = v^T (alpha M - beta I)^j v  (unnormalised block power moments)  */
/*   Gershgorin: lambda_max(M) <= max_i sum_j |m_ij| for csr.               */
/* ---------------------------------------------------------------------- */
int32_t orc_affine_power_moments_vec(const orc_op *op, double alpha, double beta, int32_t n,
                                     const double *v, double *mu)
{
    if (n < 0) return ORC_EINVAL;
    int64_t d = op_dim(op);
    double *w = (double *)malloc(sizeof(double) * (size_t)d);
    double *mx = (double *)malloc(sizeof(double) * (size_t)d);
    double *tmp = (double *)malloc(sizeof(double) * (size_t)d);
    if (!w || !mx || !tmp) { free(w); free(mx); free(tmp); return ORC_ENOMEM; }
    for (int64_t i = 0; i < d; i++) w[i] = v[i];
    mu[0] = dot(v, w, d);
    for (int32_t j = 1; j <= n; j++) {
        orc_apply_M(op, w, mx, tmp);
        for (int64_t i = 0; i < d; i++) w[i] = alpha * mx[i] - beta * w[i];
        mu[j] = dot(v, w, d);
    }
    free(w); free(mx); free(tmp);
    return ORC_OK;
}

int32_t orc_affine_power_moments_probe(const orc_op *op, double alpha, double beta, int32_t n,
                                       uint64_t seed, int64_t p, double *mu)
{
    int64_t d = op_dim(op);
    double *v = (double *)malloc(sizeof(double) * (size_t)d);
    if (!v) return ORC_ENOMEM;
    orc_rademacher(seed, p, d, v);
    int32_t rc = orc_affine_power_moments_vec(op, alpha, beta, n, v, mu);
    free(v);
    return rc;
}

double orc_gershgorin(const orc_csr *A)
{
    double best = 0.0;
    for (int64_t i = 0; i < A->n_rows; i++) {
        double s = 0.0;
        for (int64_t e = A->row_ptr[i]; e < A->row_ptr[i + 1]; e++) s += fabs(A->val[e]);
        if (s > best) best = s;
    }
    return best;
}

/* x^T A x (compensated), for the GMRF log-likelihood scan:
 *   log p(x | rho) = 1/2 log det J(rho) - 1/2 x^T J(rho) x - d/2 log(2 pi)  (reading G16). */
double orc_quadform(const orc_csr *A, const double *x)
{
    double *ax = (double *)malloc(sizeof(double) * (size_t)A->n_rows);
    if (!ax) return NAN;
    csr_mv(A, x, ax);
    double r = dot(x, ax, A->n_rows);
    free(ax);
    return r;
}

/* ---------------------------------------------------------------------- */
/* Spectral interval by Lanczos (sigma_max "by the    */
/* power iteration", sigma_min "by the inverse power iteration"; reading    */
/* G26 replaces both by the Lanczos process, which contains the power       */
/* iteration's Krylov space and converges first at both ends of the         */
/* spectrum).  Plain Lanczos on Ã = alpha*M - beta*I ([a,b] map, reading    */
/* G1) with FULL re-orthogonalisation (classical Gram-Schmidt, twice):      */
/*   q_1 = v/|v|,  w = Ã q_j - beta_{j-1} q_{j-1},  alpha_j = q_j.w,        */
/*   w -= alpha_j q_j, w -= sum_i (q_i.w) q_i (twice),                      */
/*   beta_j = |w|,  q_{j+1} = w / beta_j,                j = 1..N.           */
/* alpha_out[j-1] = alpha_j (diagonal of the Jacobi matrix T_N),            */
/* beta_out[j-1] = beta_j (off-diagonal; beta_N is the residual factor:     */
/* |Ã y - theta y| = beta_N |s_N| for a Ritz pair (theta, y = Q s)).        */
/* Returns ORC_OK, or the number of completed steps as -(100+j) when w      */
/* vanished at step j (invariant subspace found).                           */
/* ---------------------------------------------------------------------- */
int32_t orc_lanczos_tilde(const orc_op *op, double a, double b, int32_t N, const double *v,
                          double *alpha_out, double *beta_out)
{
    int64_t d = op_dim(op);
    double *Q = (double *)malloc(sizeof(double) * (size_t)d * (size_t)(N + 1));
    double *w = (double *)malloc(sizeof(double) * (size_t)d);
    if (!Q || !w) { free(Q); free(w); return ORC_ENOMEM; }
    double nv = sqrt(dot(v, v, d));
    for (int64_t i = 0; i < d; i++) Q[i] = v[i] / nv;
    int32_t rc = ORC_OK;
    for (int32_t j = 0; j < N; j++) {
        double *q = Q + (size_t)j * d;
        int32_t e = orc_apply_tilde(op, a, b, q, w);
        if (e) { rc = e; break; }
        if (j > 0) {
            const double *qm = Q + (size_t)(j - 1) * d;
            for (int64_t i = 0; i < d; i++) w[i] -= beta_out[j - 1] * qm[i];
        }
        double al = dot(q, w, d);
        alpha_out[j] = al;
        for (int64_t i = 0; i < d; i++) w[i] -= al * q[i];
        for (int pass = 0; pass < 2; pass++) {
            for (int32_t t = 0; t <= j; t++) {
                const double *qt = Q + (size_t)t * d;
                double h = dot(qt, w, d);
                for (int64_t i = 0; i < d; i++) w[i] -= h * qt[i];
            }
        }
        double be = sqrt(dot(w, w, d));
        beta_out[j] = be;
        if (!(be > 0.0)) { rc = -(100 + j + 1); break; }
        double *qn = Q + (size_t)(j + 1) * d;
        for (int64_t i = 0; i < d; i++) qn[i] = w[i] / be;
    }
    free(Q);
    free(w);
    return rc;
}

int32_t orc_lanczos_probe(const orc_op *op, double a, double b, int32_t N, uint64_t seed, int64_t p,
                          double *alpha_out, double *beta_out)
{
    int64_t d = op_dim(op);
    double *v = (double *)malloc(sizeof(double) * (size_t)d);
    if (!v) return ORC_ENOMEM;
    orc_rademacher(seed, p, d, v);
    int32_t rc = orc_lanczos_tilde(op, a, b, N, v, alpha_out, beta_out);
    free(v);
    return rc;
}
