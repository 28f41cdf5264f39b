/*
 * cheb_logdet.h -- C ABI of the B200-native Chebyshev-Hutchinson log-determinant
 * hot path (arXiv 1503.06394).  Library: paper_1503_06394_b200/libchebld.so.
 *
 * What it computes (PAPER.md, "P:n" = line n):
 *   Gamma ~= log det M for a symmetric positive-definite operator M whose
 *   spectrum lies in [a, b]:
 *     alpha = 2/(b-a), beta = (b+a)/(b-a), Ã = alpha*M - beta*I          (G1/G3)
 *     c_j   = Chebyshev interpolation coefficients of log on [a,b]
 *     v_p   = Rademacher probes, v_p[i] = -1 iff bit 63 of
 *             splitmix64(seed, p*d + i + 1) is set                        (G6)
 *     w_0 = v, w_1 = Ã v, w_{j+1} = 2 Ã w_j - w_{j-1}                    (Alg. 1)
 *     mu_{p,j} = v_p^T w_j ;  Gamma_p = sum_j c_j mu_{p,j} ;
 *     Gamma = (1/m) sum_p Gamma_p                                         (G7)
 *   Operator modes:
 *     CL_OP_CSR        M = A
 *     CL_OP_CSR_RANK1  M = A + c u u^T   (u = all ones if r1_u == NULL;
 *                      spanning trees: log tau = Gamma - log(c N^2))      (BASELINE configs[1])
 *     CL_OP_BTB        M = B^T B applied as B^T (B w), never formed;
 *                      log|det B| = Gamma / 2                             (Alg. 2)
 *
 * Conventions
 *   - All functions return 0 (CL_OK) on success or a negative CL_E* code, never
 *     throw, and set a thread-local message readable with cheb_last_error().
 *   - All validation runs before any device work; outputs are written only on
 *     success (device outputs of the asynchronous calls: on successful launch).
 *   - The caller owns every buffer passed in; the library never frees or keeps
 *     a pointer past the call.  Only cheb_logdet / cheb_logdet_host (per-thread
 *     arenas, see cheb_release_cache) and cheb_probes / cheb_bounds_btb /
 *     cheb_norm_bound / cheb_gershgorin / cheb_quadform allocate device memory.
 *   - Matrices are canonical CSR: row_ptr int64[n_rows+1] (row_ptr[0] = 0),
 *     col_idx int32[nnz] sorted & unique within a row, val fp64[nnz].
 *   - Probe-block layout on the device: W[d][k] fp64 row-major, the k probes of a
 *     block contiguous; k in {8, 16, 32, 64, 128}.
 */
#ifndef CHEB_LOGDET_H
#define CHEB_LOGDET_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CL_OK 0
#define CL_EINVAL (-1)     /* bad scalar argument / NULL pointer / bad k          */
#define CL_EDIM (-2)       /* non-square M, B^T not the transpose shape, d >= 2^31 */
#define CL_ENOMEM (-3)     /* workspace too small or cudaMalloc failed             */
#define CL_ECUDA (-4)      /* CUDA runtime error (message has the CUDA string)     */
#define CL_ENONFINITE (-5) /* a moment / estimate is not finite: [a,b] does not
                              enclose the spectrum (|T_j| blow-up)     */

typedef struct {
    int64_t n_rows, n_cols, nnz;
    const int64_t *row_ptr; /* [n_rows+1] */
    const int32_t *col_idx; /* [nnz]      */
    const double *val;      /* [nnz]      */
} cl_csr;

typedef enum { CL_OP_CSR = 0, CL_OP_CSR_RANK1 = 1, CL_OP_BTB = 2, CL_OP_FAMILY = 3 } cl_op_kind;

typedef struct {
    int32_t kind;      /* cl_op_kind (FAMILY: only for cheb_workspace_bytes, see      */
                       /* cheb_family_moments)                                       */
    cl_csr A;          /* A (CSR, RANK1), B (BTB) or the family base; d = A.n_cols  */
    cl_csr At;         /* BTB only: exact CSR of B^T (n_rows = B.n_cols)          */
    double r1_c;       /* RANK1 only: weight c                                    */
    const double *r1_u;/* RANK1 only: u[d], NULL = all ones                       */
} cl_operator;

typedef struct {
    double logdet;        /* Gamma: estimate of log det M (BTB: of B^T B)         */
    double stderr_;       /* sample sd(Gamma_p) / sqrt(m)                          */
    int64_t num_probes;   /* m                                                      */
    int32_t degree;       /* n                                                      */
    int32_t probe_block;  /* k actually used                                        */
    double *per_probe;    /* caller-owned HOST array [m] or NULL: Gamma_p           */
    double *moments;      /* caller-owned HOST array [m*(n+1)] or NULL: mu_{p,j}    */
    double elapsed_s;     /* wall time of the call                                  */
} cl_result;

typedef struct {
    double lambda_min, lambda_max; /* extreme Ritz values over the probes (inside the spectrum)  */
    double res_min, res_max;       /* their Lanczos residual bounds |M y - lambda y| (Kahan: an  */
                                   /* eigenvalue of M lies within res of each)                   */
    double a, b;                   /* interval for cheb_logdet: max(lambda_min - res_min, 0),    */
                                   /* min(lambda_max + res_max, hi_bound)                        */
    double hi_bound;               /* guaranteed upper bound of the spectrum (cheb_norm_bound)   */
    int32_t lanczos_steps;         /* Lanczos steps used (min over probes; fewer than requested  */
                                   /* when a run reached an invariant subspace)                  */
    int32_t num_probes;
} cl_spectrum;

/* Chebyshev interpolation coefficients c_0..c_n of f(x) = log(((b-a)x+(b+a))/2)
 * on [-1,1] at the n+1 first-kind nodes x_k = cos(pi(k+1/2)/(n+1))
 * (Alg. 1 line 4 P:225-227 in [a,b] form).  Host fp64 routine; c_out
 * is a HOST array of degree+1 doubles.  CL_EINVAL if !(0 < a < b), non-finite, or
 * degree < 0. */
int cheb_coeffs_log(double a, double b, int32_t degree, double *c_out);

/* Device workspace bytes cheb_moments needs for operator `op` and probe block k
 * on the current device.  Returns 0 on invalid input (see cheb_last_error). */
size_t cheb_workspace_bytes(const cl_operator *op, int32_t probe_block);

/* Shard-level, stream-ordered, ASYNCHRONOUS moments: for global probes
 * p in [probe_begin, probe_end) writes mu_out[(p-probe_begin)*(degree+1) + j]
 * = v_p^T T_j(Ã) v_p, j = 0..degree (DEVICE array).  All CSR / u pointers are
 * DEVICE pointers.  Probes are addressed by global index, so sharding never
 * changes a probe.  `stream` is a cudaStream_t (NULL = legacy default).
 * Allocates nothing; `workspace` must hold cheb_workspace_bytes(op, k) bytes and may be used
 * by one call at a time (calls on different streams need separate workspaces).
 * Errors found on the device are reported without a host synchronisation: the call ends with a
 * status epilogue that records them in the workspace status word (cheb_workspace_status) and,
 * for a timed-out spin wait of the persistent kernel, overwrites every moment of the call with
 * NaN, so cheb_finalize's stats[2] (all-finite flag) is 0 for any estimate that saw either. */
int cheb_moments(const cl_operator *op, double a, double b, int32_t degree,
                 int64_t probe_begin, int64_t probe_end, uint64_t seed,
                 int32_t probe_block, void *workspace, size_t ws_bytes,
                 double *mu_out, void *stream);

/* Taylor baseline (Fig. 1(d)): power moments
 *   mu_{p,j} = v_p^T A^j v_p,  A = I - M/s  (s > 0; s >= lambda_max(M) keeps spec(A) in [0,1)),
 * by the power recurrence w_j = A w_{j-1} on the same fused SpMM kernels.  Arguments, layout,
 * workspace and stream semantics as cheb_moments.  With c = cheb_taylor_coeffs(s, n)
 * (c_0 = log s, c_k = -1/k: log det M = d log s + tr log(I - A), log(1-x) = -sum_k x^k/k),
 * cheb_finalize gives the Taylor estimate of log det M. */
int cheb_power_moments(const cl_operator *op, double s, int32_t degree, int64_t probe_begin,
                       int64_t probe_end, uint64_t seed, int32_t probe_block, void *workspace,
                       size_t ws_bytes, double *mu_out, void *stream);
int cheb_taylor_coeffs(double s, int32_t degree, double *c_out);

/* Device-side spectral bounds ("one can run the power iteration to estimate a
 * better bound"):
 *   cheb_affine_power_moments: mu_{p,j} = v_p^T (alpha M - beta I)^j v_p (power recurrence on
 *     the fused kernels; cheb_power_moments is alpha = -1/s, beta = -1).  Block power
 *     iteration: mu_{j+1}/mu_j -> the dominant eigenvalue of alpha M - beta I.
 *   cheb_norm_bound: s >= lambda_max(M) from the matrix, on the device: Gershgorin
 *     max_i sum_j |a_ij| (+ |c| max|u|^2 d for rank-1) or ||B||_1 ||B||_inf for B^T B
 *     (P:301-302).  s_out is a HOST double; synchronous on `stream`.
 * Python's spectrum_estimate() combines them into (lambda_min, lambda_max) estimates. */
int cheb_affine_power_moments(const cl_operator *op, double alpha, double beta, int32_t degree,
                              int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                              void *workspace, size_t ws_bytes, double *mu_out, void *stream);
int cheb_norm_bound(const cl_operator *op, double *s_out, void *stream);

/* x^T A x for a DEVICE CSR A (square) and DEVICE vector x[d]; result to the HOST double
 * *out; deterministic (fixed reduction order); synchronous on `stream`.  The GMRF
 * log-likelihood scan (§5.2) is
 *   log p(x | rho) = 1/2 log det J(rho) - 1/2 x^T J(rho) x - d/2 log(2 pi). */
int cheb_quadform(const cl_csr *A, const double *x, double *out, void *stream);

/* x^T D x and x^T O x for a DEVICE CSR A = D + O (D its diagonal entries, O the rest): out2[0],
 * out2[1] (HOST).  For the family M(theta) = D + theta O, x^T M(theta) x = out2[0] + theta out2[1].
 * Deterministic; synchronous on `stream`. */
int cheb_quadform_split(const cl_csr *A, const double *x, double *out2, void *stream);

/* One-parameter operator family for the GMRF likelihood scan (§5.2):
 * M_r = D + theta_r O, r < R, from a DEVICE base CSR = D + O (D its diagonal entries, O the rest;
 * the grid GMRF: base = I - Adj, M_r = I - theta_r Adj).
 *   cheb_family_gershgorin: lo_hi[2r], lo_hi[2r+1] = the Gershgorin interval of M_r (HOST array
 *     [R][2]); synchronous.
 *   cheb_family_moments: the R members in the COLUMNS of one probe block, so all R share every pass
 *     over the matrix: with R_pad = R rounded up to a power of two and kp = probe_block / R_pad
 *     (>= 2), column c of a block carries member c / kp and probe p0 + c % kp (common random
 *     numbers: every member sees the same probes).  Per column the step applies
 *     Ã_r = alpha_r M_r - beta_r I for the member's interval ab[2r], ab[2r+1] (HOST [R][2]):
 *     (alpha_r d_i - beta_r) w_i + alpha_r theta_r (O w)_i.  mu_out (DEVICE) receives
 *     mu[r][p - probe_begin][j] = v_p^T T_j(Ã_r) v_p, layout [R][probe_end-probe_begin][degree+1].
 *     Workspace: cheb_workspace_bytes of an operator {kind = CL_OP_FAMILY, A = base}.  Algorithm 1,
 *     per-step launches; asynchronous like cheb_moments (same status word / NaN poisoning).
 *     CL_EINVAL for probe_block < 16 or < 2 R_pad, or an invalid interval. */
int cheb_family_gershgorin(const cl_csr *base, int32_t R, const double *theta, double *lo_hi, void *stream);
int cheb_family_moments(const cl_csr *base, int32_t R, const double *theta, const double *ab, int32_t degree,
                        int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                        void *workspace, size_t ws_bytes, double *mu_out, void *stream);

/* Gershgorin interval of a DEVICE CSR: lo_hi[0] = min_i (a_ii - sum_{j!=i} |a_ij|),
 * lo_hi[1] = max_i sum_j |a_ij| (HOST array[2]); for a symmetric A it encloses spec(A)
 * (the GMRF configs' [1-4theta, 1+4theta]).  Synchronous on `stream`. */
int cheb_gershgorin(const cl_csr *A, double *lo_hi, void *stream);

/* ASYNCHRONOUS device accumulation (reading G7):
 *   gamma_p[p] = sum_{j=0..n} c[j] mu[p*(n+1)+j] (ascending j),
 *   stats[0] = Gamma = (sum_p gamma_p, ascending p)/m,
 *   stats[1] = sample sd(gamma_p)/sqrt(m) (0 if m == 1),
 *   stats[2] = 1.0 if every gamma_p is finite else 0.0.
 * mu, c, gamma_p, stats are DEVICE arrays. */
int cheb_finalize(const double *mu, const double *c, int64_t m, int32_t degree,
                  double *gamma_p, double *stats, void *stream);

/* Device status of the last cheb_moments / cheb_power_moments / cheb_affine_power_moments call
 * that used `workspace` (DEVICE pointer; the word sits at a fixed offset of every workspace):
 *   bit 0 (1) = a grid-wide spin wait of the persistent kernel gave up after ~seconds without
 *               progress (CTAs not co-resident); that call's moments were set to NaN;
 *   bit 1 (2) = a moment of that call is not finite ([a,b] does not enclose the spectrum);
 *   bit 8 (0x100, informational, not an error) = the per-step kernels of that call read the
 *               compressed matrix copy (uniform padded rows, int16 column deltas, <= 128 distinct
 *               values: 3 bytes per entry instead of 12); moments are bit-identical
 *               to the plain copy.  Env CHEB_CV=0 disables the compressed copy.
 * *status is a HOST uint32; synchronises `stream` (enqueue after the call, same stream). */
int cheb_workspace_status(const void *workspace, uint32_t *status, void *stream);

/* Synchronous single-GPU estimate in BASELINE's shape; operator pointers are
 * DEVICE pointers.  probe_block = 0 picks k automatically.  Allocates its own
 * workspace.  CL_ENONFINITE if any estimate is not finite. */
int cheb_logdet(const cl_operator *op, double a, double b, int32_t degree,
                int32_t num_probes, uint64_t seed, int32_t probe_block,
                cl_result *out);

/* As cheb_logdet, but every operator pointer is a HOST pointer: the call copies
 * the matrix (and u) to the device, runs, copies the result back, and frees. */
int cheb_logdet_host(const cl_operator *op, double a, double b, int32_t degree,
                     int32_t num_probes, uint64_t seed, int32_t probe_block,
                     cl_result *out);

/* Spectral interval [a, b] of M for the estimator, computed from the matrix on the device
 * ("run the power iteration to estimate a better bound", "use the inverse
 * power iteration to estimate [sigma_min]"; reading G26 uses the Lanczos process instead, whose
 * Krylov space contains the power iterates and which converges first at both ends).
 * num_probes independent Lanczos runs on M, started at the Rademacher probes of `seed` (global
 * probes 0..num_probes-1; the path's splitmix64 generator), N = lanczos_steps steps each, without
 * re-orthogonalisation, run as blocks of k probes ([d][k] columns) on the device: the operator
 * products by the spmm kernel, the recurrence and its three reductions per step by
 * lanczos_vec_kernel; only the Jacobi matrices T_N (k x 2N doubles per block) return to the host,
 * whose QL eigen-solver gives the extreme Ritz values and their residual bounds (see cl_spectrum).
 * jacobi_out: NULL or a HOST array [num_probes][2N] receiving T_N per probe: diagonal
 * alpha_0..alpha_{N-1}, then beta_1..beta_N (off-diagonal, the last is the residual factor); NaN
 * beyond an early stop.  Synchronous; device memory from the calling thread's arena.
 * CL_EINVAL for N outside [1, 2000] or probes outside [1, 4096]. */
int cheb_spectrum_bounds(const cl_operator *op, int32_t lanczos_steps, int32_t num_probes, uint64_t seed,
                         cl_spectrum *out, double *jacobi_out);

/* Shard-level moments from a HOST operator (the end-to-end call of one rank of the multi-GPU
 * driver): copies the operator to the device (per-thread arena, see cheb_release_cache), runs
 * cheb_moments for global probes [probe_begin, probe_end) and copies the moments to the HOST
 * array mu_out[(probe_end-probe_begin)*(degree+1)].  Synchronous.  CL_ECUDA on a device
 * timeout, CL_ENONFINITE if a moment is not finite (mu_out is written in both cases). */
int cheb_moments_host(const cl_operator *op, double a, double b, int32_t degree, int64_t probe_begin,
                      int64_t probe_end, uint64_t seed, int32_t probe_block, double *mu_out);

/* Spectral interval of B^T B for Algorithm 2, computed on the device
 * from B and B^T (DEVICE CSRs in op, kind must be CL_OP_BTB):
 *   ab_out[0] = a = (min_i |b_ii| - (r_i + c_i)/2)^2   (Johnson lower bound on
 *               sigma_min; r_i, c_i off-diagonal absolute row/column sums)
 *   ab_out[1] = b = ||B||_1 ||B||_inf
 * ab_out is a HOST array[2]; synchronous on `stream`.  CL_EINVAL if the Johnson
 * bound is not positive (B not diagonally dominant enough). */
int cheb_bounds_btb(const cl_operator *op, double *ab_out, void *stream);

/* The probes the path uses: writes v_p[i] (+1.0 / -1.0) for p in
 * [probe_begin, probe_begin+k), into v_out[i*k + (p-probe_begin)] (DEVICE, d*k
 * doubles), running the same probe-initialisation kernel as cheb_moments. */
int cheb_probes(int64_t d, uint64_t seed, int64_t probe_begin, int32_t probe_block,
                double *v_out, void *stream);

/* Kernel accounting for benchmarks.  cheb_launch_count(): cumulative number of
 * this library's kernel launches in the process.  cheb_profile_begin(): start
 * recording CUDA events around every Chebyshev-step launch on its stream;
 * cheb_profile_end(): synchronise, return the summed step-kernel milliseconds,
 * the number of step launches, and stop recording. */
int64_t cheb_launch_count(void);
int cheb_profile_begin(void);
int cheb_profile_end(double *step_ms, int64_t *step_launches);
/* After cheb_profile_end(): summed milliseconds and launch count of the B^T B spmm kernel
 * (Y = B w_{j-1}, the first half of every B^T B application; one launch per step). */
int cheb_profile_spmm(double *ms, int64_t *launches);
/* After cheb_profile_end(): milliseconds and launches of the persistent kernel (each launch
 * = all n Chebyshev steps of one probe block). */
int cheb_profile_persistent(double *ms, int64_t *launches);

/* Persistent multi-step schedule for CL_OP_CSR / CL_OP_CSR_RANK1 (process-wide):
 *   0 = off (one launch per step);
 *   1 = auto (default): all n steps of a probe block in one cooperative launch with a grid
 *       barrier per step when the working set (two probe blocks + matrix) fits in half of
 *       L2 -- there the per-step launch/drain gaps, not bandwidth, bound the step;
 *   2 = always.
 * Moments are bit-identical to per-step launches when both use the same grid size. */
int cheb_set_persistent(int32_t mode);

/* Tile geometry of the Algorithm-1 kernels (process-wide):
 *   1 = auto (default): operators whose working set fits in half of L2 use 16-row tiles (at
 *       k = 64; 256*4/k rows) in both the per-step and the persistent kernel -- more tiles per
 *       step shorten the critical path of a latency-bound step; so do Algorithm-1 runs with
 *       probe blocks k <= 16 (64-row instead of 128-row tiles at k = 16);
 *   0 = always the standard geometry (32-row tiles at k = 64).
 * Moments are bit-identical between schedules that use the same geometry and grid.
 * CL_EINVAL for other values. */
int cheb_set_small_tiles(int32_t mode);
int cheb_get_small_tiles(void);

/* Moment-doubling schedule for cheb_moments / cheb_logdet / cheb_logdet_host (process-wide;
 * default 0; env CHEB_DOUBLING sets the initial value).  DESIGN.md reading G25:
 *   0 = Algorithm 1 as written: n applications of Ã per probe, mu_j = v^T w_j;
 *   1 = ceil(n/2) applications: for a SYMMETRIC Ã the Chebyshev identities
 *       T_{2j} = 2 T_j^2 - I and T_{2j+1} = 2 T_{j+1} T_j - T_1 give
 *         mu_{2j}   = 2 w_j^T w_j     - mu_0,
 *         mu_{2j-1} = 2 w_j^T w_{j-1} - mu_1   (mu_1 = w_1^T w_0 = v^T Ã v),
 *       i.e. the same moments mu_0..mu_n (equal in exact arithmetic, rounding differs) from half
 *       the matrix passes.  Requires M symmetric (A symmetric; B^T B always is).  Not applied
 *       to the power-basis entry points.  CL_EINVAL for other values. */
int cheb_set_doubling(int32_t on);
int cheb_get_doubling(void);

/* Shared-memory-resident schedule for CL_OP_CSR / CL_OP_CSR_RANK1 (process-wide; default 1; env
 * CHEB_RESIDENT sets the initial value).  Applies only in the automatic persistent mode
 * (cheb_set_persistent(1)), to Algorithm 1, moment doubling and the power basis, k <= 64:
 *   1 = auto: when one probe block (two d x k fp64 buffers + the CTAs' matrix rows) fits in the
 *       shared memory of one CTA per SM, all n steps run in one launch in which every CTA keeps
 *       its rows of w_{j-1}, w_{j-2} on chip: small operators in one thread-block cluster
 *       (other CTAs' rows over DSMEM, one cluster barrier per step), larger ones on a flat
 *       cooperative grid (other CTAs' rows from a global copy of the rows they need, one grid
 *       counter per step) (cheb_resident_kernel); w_j is bit-identical to the other
 *       schedules, the dot products follow this kernel's fixed order (deterministic run to run);
 *   0 = off (the L2-resident persistent kernel or per-step launches).
 * CL_EINVAL for other values. */
int cheb_set_resident(int32_t mode);
int cheb_get_resident(void);

/* Schedule the calling thread's last cheb_moments-family call ran (set when it returns CL_OK):
 * 0 = one launch per step, 1 = L2-resident persistent kernel, 2 = shared-memory-resident kernel;
 * -1 before any call.  Diagnostics (tests, bench). */
int cheb_last_schedule(void);

/* cheb_logdet / cheb_logdet_host keep their device workspace (and cheb_logdet_host the device
 * copy of the operator) in grow-only per-thread arenas, so repeated estimates do not pay a
 * multi-GB cudaMalloc/cudaFree per call.  cheb_release_cache() frees the calling thread's
 * arenas (they are also freed when the thread exits). */
int cheb_release_cache(void);

/* Thread-local message for the last failing call on this thread. */
const char *cheb_last_error(void);

/* ABI version (major*10000 + minor*100 + patch). */
int cheb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CHEB_LOGDET_H */
