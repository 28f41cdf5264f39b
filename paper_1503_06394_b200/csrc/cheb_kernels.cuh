// cheb_kernels.cuh -- sm_100a device kernels of the Chebyshev-Hutchinson hot path.
//
// Layout:
//   W[d][K]  fp64, the K probes of a block contiguous per row (row = 8K bytes);
//   each row is handled by a "group" of L = K/2 lanes, lane l owning probes
//   2l, 2l+1 as one 16-byte double2 (fully coalesced 8K-byte row accesses).
//   S[d][WORDS] uint32 packed probe signs (bit p%32 of word p/32 = 1 <=> v_p[i] = -1).
//
// Kernels
//   probe_init_kernel<K,MODE>       K1: v -> W_cur, S; mu_0 = v^T v; rank-1 s_0 = u^T v
//   cheb_step_kernel<K,MODE,FIRST>  K2: fused CSR-SpMM x K probes + three-term
//                                   recurrence + Ã scaling + rank-1 term + per-probe
//                                   dot v^T w_j, deterministic last-CTA reduction (K4)
//   spmm_kernel<K>                  K3: Y = B W (first half of a B^T B application)
//   finalize_kernel                 Gamma_p, Gamma, stderr
//   bounds_btb_kernel               Johnson / norm bounds of B^T B
//
// Every kernel is a persistent grid (a multiple of the SM count) walking row
// tiles t = blockIdx.x, blockIdx.x + gridDim.x, ... in increasing order, so the
// rows being processed chip-wide form one narrow moving window: the W_cur halo
// rows i +- N of a stencil are re-read from L2, not HBM (SURVEY §7 "hard parts").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace chebld {

constexpr int kThreads = 256;
constexpr int kUnroll = 2;  // rows per group processed concurrently (memory-level parallelism)
#ifndef CHEB_MIN_CTAS
#define CHEB_MIN_CTAS 3     // resident CTAs per SM the step kernel is register-budgeted for
#endif

enum { MODE_CSR = 0, MODE_RANK1 = 1, MODE_BTB = 2 };

template <int K>
struct Geo {
    static_assert(K == 8 || K == 16 || K == 32 || K == 64, "K in {8,16,32,64}");
    static constexpr int L = K / 2;               // lanes per row
    static constexpr int GROUPS = kThreads / L;   // row groups per CTA
    static constexpr int WORDS = K >= 32 ? K / 32 : 1;
    static constexpr int TILE = GROUPS * kUnroll; // rows per tile
    static constexpr int RED_T = kThreads / K;    // threads per probe in the final reduction
};

// SplitMix64 at flat counter t of the stream seeded `seed` (reading G6).
__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t t) {
    uint64_t z = seed + t * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double2 ld_nc2(const double* p) {
    return __ldg(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double2 ld_cs2(const double* p) {
    return __ldcs(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ void st2(double* p, double2 v) {
    *reinterpret_cast<double2*>(p) = v;
}

struct StepArgs {
    int64_t d;          // rows of the gather matrix (= dimension of M)
    int64_t ntiles;
    const int64_t* rp;  // gather matrix: A (csr/rank1) or B^T (btb)
    const int32_t* ci;
    const double* va;
    const double* xg;   // gather source: W_cur (csr/rank1) or Y = B W_cur (btb)
    const double* wcur; // W_cur (the -beta*w term)
    double* wnext;      // in: W_prev (unless FIRST); out: W_next (in place)
    const uint32_t* sbits;
    double alpha, beta;
    double r1c;          // rank-1 weight
    const double* r1u;   // rank-1 u (nullptr = ones)
    const double* s_cur; // [K] u^T w_{j-1}
    double* s_next;      // [K] u^T w_j
    double* part_mu;     // [gridDim.x][K]
    double* part_s;      // [gridDim.x][K]
    unsigned int* ticket;
    double* mu_out;      // mu_out[p*mu_stride + mu_col]
    int64_t mu_stride;
    int32_t mu_col;
    int32_t kvalid;      // probes of this block that exist (<= K)
};

// ---------------------------------------------------------------------------
// Deterministic CTA + grid reduction of two per-thread double2 accumulators
// (probes 2l, 2l+1).  Order: fixed shuffle tree inside a warp, warps in index
// order, CTAs in a fixed strided order -- independent of timing.  The last CTA
// to finish (atomic ticket) produces the final sums.
// ---------------------------------------------------------------------------
template <int K, bool HAS_S>
__device__ __forceinline__ void grid_reduce_finish(double2 mu, double2 s, const StepArgs& a) {
    using G = Geo<K>;
    __shared__ double red_mu[kThreads / 32][K];
    __shared__ double red_s[HAS_S ? kThreads / 32 : 1][K];
    __shared__ double fin_mu[G::RED_T][K];
    __shared__ double fin_s[HAS_S ? G::RED_T : 1][K];
    __shared__ bool is_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lg = lane % G::L;
#pragma unroll
    for (int off = G::L; off < 32; off <<= 1) {
        mu.x += __shfl_xor_sync(0xffffffffu, mu.x, off);
        mu.y += __shfl_xor_sync(0xffffffffu, mu.y, off);
        if (HAS_S) {
            s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
            s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
        }
    }
    if (lane < G::L) {
        red_mu[warp][2 * lg] = mu.x;
        red_mu[warp][2 * lg + 1] = mu.y;
        if (HAS_S) {
            red_s[warp][2 * lg] = s.x;
            red_s[warp][2 * lg + 1] = s.y;
        }
    }
    __syncthreads();
    if (tid < K) {
        double m = 0.0, t = 0.0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; w++) {
            m += red_mu[w][tid];
            if (HAS_S) t += red_s[w][tid];
        }
        a.part_mu[(size_t)blockIdx.x * K + tid] = m;
        if (HAS_S) a.part_s[(size_t)blockIdx.x * K + tid] = t;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        unsigned int prev = atomicAdd(a.ticket, 1u);
        is_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    {
        const int p = tid % K, r = tid / K;
        double m = 0.0, t = 0.0;
        for (int c = r; c < (int)gridDim.x; c += G::RED_T) {
            m += __ldcg(a.part_mu + (size_t)c * K + p);
            if (HAS_S) t += __ldcg(a.part_s + (size_t)c * K + p);
        }
        fin_mu[r][p] = m;
        if (HAS_S) fin_s[r][p] = t;
    }
    __syncthreads();
    if (tid < K) {
        double m = 0.0, t = 0.0;
#pragma unroll
        for (int r = 0; r < G::RED_T; r++) {
            m += fin_mu[r][tid];
            if (HAS_S) t += fin_s[r][tid];
        }
        if (tid < a.kvalid) a.mu_out[(size_t)tid * a.mu_stride + a.mu_col] = m;
        if (HAS_S) a.s_next[tid] = t;
    }
    if (tid == 0) *a.ticket = 0u;  // re-arm for the next launch (stream-ordered)
}

// ---------------------------------------------------------------------------
// K1: probe initialisation.  W_cur[i][p] = v_p[i] = +-1 (global probe p0+p),
// sign bits, mu_0 = v^T v (= d exactly), rank-1 s_0 = u^T v.
// ---------------------------------------------------------------------------
template <int K, int MODE>
__global__ void __launch_bounds__(kThreads)
probe_init_kernel(StepArgs a, uint64_t seed, uint64_t p0, double* w0, uint32_t* sbits) {
    using G = Geo<K>;
    constexpr bool HAS_S = (MODE == MODE_RANK1);
    const int lg = threadIdx.x % G::L;
    const int group = threadIdx.x / G::L;
    const int p2 = 2 * lg;
    const uint64_t d = (uint64_t)a.d;
    double2 mu = make_double2(0.0, 0.0), s = make_double2(0.0, 0.0);
    const int64_t rows_per_iter = (int64_t)G::GROUPS;
    const int64_t niter = (a.d + rows_per_iter - 1) / rows_per_iter;
    for (int64_t t = blockIdx.x; t < niter; t += gridDim.x) {
        const int64_t i = t * rows_per_iter + group;
        const bool ok = i < a.d;
        uint32_t bits = 0;
        double v0 = 1.0, v1 = 1.0;
        if (ok) {
            const uint64_t z0 = splitmix64_at(seed, (p0 + p2) * d + (uint64_t)i + 1ull);
            const uint64_t z1 = splitmix64_at(seed, (p0 + p2 + 1) * d + (uint64_t)i + 1ull);
            const uint32_t b0 = (uint32_t)(z0 >> 63), b1 = (uint32_t)(z1 >> 63);
            v0 = b0 ? -1.0 : 1.0;
            v1 = b1 ? -1.0 : 1.0;
            bits = (b0 << (p2 & 31)) | (b1 << ((p2 + 1) & 31));
            st2(w0 + (size_t)i * K + p2, make_double2(v0, v1));
            mu.x += v0 * v0;
            mu.y += v1 * v1;
            if (HAS_S) {
                const double u = a.r1u ? __ldg(a.r1u + i) : 1.0;
                s.x += u * v0;
                s.y += u * v1;
            }
        }
        // OR the bits of the (up to) 16 lanes that share one 32-bit word
        constexpr int WL = G::L < 16 ? G::L : 16;
#pragma unroll
        for (int off = 1; off < WL; off <<= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, off);
        if (ok && (lg % 16) == 0) sbits[(size_t)i * G::WORDS + (p2 >> 5)] = bits;
    }
    grid_reduce_finish<K, HAS_S>(mu, s, a);
}

// ---------------------------------------------------------------------------
// K2: the fused Chebyshev step (w_j from w_{j-1}, w_{j-2}):
//   y    = alpha * (G xg)_i [+ alpha*c*u_i*s_cur] - beta * wcur_i
//   w_j  = FIRST ? y : 2y - w_{j-2}          (written over w_{j-2})
//   mu_j += v_i * w_j ; rank-1: s_j += u_i * w_j
// ---------------------------------------------------------------------------
template <int K, int MODE, bool FIRST>
__global__ void __launch_bounds__(kThreads, CHEB_MIN_CTAS)
cheb_step_kernel(StepArgs a) {
    using G = Geo<K>;
    constexpr bool HAS_S = (MODE == MODE_RANK1);
    constexpr int U = kUnroll;
    const int lg = threadIdx.x % G::L;
    const int group = threadIdx.x / G::L;
    const int p2 = 2 * lg;
    const int sh = p2 & 31, wsel = p2 >> 5;
    double2 mu = make_double2(0.0, 0.0), s = make_double2(0.0, 0.0);
    double2 r1 = make_double2(0.0, 0.0);
    if (HAS_S) {
        const double2 sc = *reinterpret_cast<const double2*>(a.s_cur + p2);
        r1 = make_double2(a.alpha * a.r1c * sc.x, a.alpha * a.r1c * sc.y);
    }
    for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        int64_t row[U], rs[U], len[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            row[u] = t * G::TILE + u * G::GROUPS + group;
            ok[u] = row[u] < a.d;
            rs[u] = ok[u] ? __ldg(a.rp + row[u]) : 0;
            len[u] = ok[u] ? __ldg(a.rp + row[u] + 1) - rs[u] : 0;
        }
        double2 wp[U];
        uint32_t sw[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            wp[u] = make_double2(0.0, 0.0);
            if (!FIRST && ok[u]) wp[u] = ld_cs2(a.wnext + (size_t)row[u] * K + p2);
            sw[u] = ok[u] ? __ldg(a.sbits + (size_t)row[u] * G::WORDS + wsel) : 0u;
        }
        double2 acc[U], xd[U];
        bool found[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            acc[u] = make_double2(0.0, 0.0);
            xd[u] = make_double2(0.0, 0.0);
            found[u] = false;
        }
        int64_t maxlen = len[0];
#pragma unroll
        for (int u = 1; u < U; u++) maxlen = len[u] > maxlen ? len[u] : maxlen;
        for (int64_t e0 = 0; e0 < maxlen; e0 += 4) {
            int c[U][4];
            double v[U][4];
            double2 x[U][4];
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const bool in = e0 + q < len[u];
                    c[u][q] = in ? __ldg(a.ci + rs[u] + e0 + q) : -1;
                    v[u][q] = in ? __ldg(a.va + rs[u] + e0 + q) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < 4; q++)
                    x[u][q] = c[u][q] >= 0 ? ld_nc2(a.xg + (size_t)c[u][q] * K + p2)
                                           : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    acc[u].x = fma(v[u][q], x[u][q].x, acc[u].x);
                    acc[u].y = fma(v[u][q], x[u][q].y, acc[u].y);
                    if (MODE != MODE_BTB && c[u][q] == row[u]) {
                        xd[u] = x[u][q];
                        found[u] = true;
                    }
                }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (!ok[u]) continue;
            if (MODE == MODE_BTB || !found[u]) xd[u] = ld_nc2(a.wcur + (size_t)row[u] * K + p2);
            double yx = a.alpha * acc[u].x - a.beta * xd[u].x;
            double yy = a.alpha * acc[u].y - a.beta * xd[u].y;
            double ui = 1.0;
            if (HAS_S) {
                ui = a.r1u ? __ldg(a.r1u + row[u]) : 1.0;
                yx = fma(ui, r1.x, yx);
                yy = fma(ui, r1.y, yy);
            }
            double2 wn;
            if (FIRST) {
                wn = make_double2(yx, yy);
            } else {
                wn = make_double2(2.0 * yx - wp[u].x, 2.0 * yy - wp[u].y);
            }
            __stcs(reinterpret_cast<double2*>(a.wnext + (size_t)row[u] * K + p2), wn);
            const uint32_t b = sw[u] >> sh;
            mu.x += (b & 1u) ? -wn.x : wn.x;
            mu.y += (b & 2u) ? -wn.y : wn.y;
            if (HAS_S) {
                s.x = fma(ui, wn.x, s.x);
                s.y = fma(ui, wn.y, s.y);
            }
        }
    }
    grid_reduce_finish<K, HAS_S>(mu, s, a);
}

// ---------------------------------------------------------------------------
// K3: Y = B W (first half of applying B^T B; Alg. 2 via P:312-314)
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(kThreads, CHEB_MIN_CTAS)
spmm_kernel(int64_t d, int64_t ntiles, const int64_t* __restrict__ rp,
            const int32_t* __restrict__ ci, const double* __restrict__ va,
            const double* __restrict__ x, double* __restrict__ y) {
    using G = Geo<K>;
    constexpr int U = kUnroll;
    const int lg = threadIdx.x % G::L;
    const int group = threadIdx.x / G::L;
    const int p2 = 2 * lg;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int64_t row[U], rs[U], len[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            row[u] = t * G::TILE + u * G::GROUPS + group;
            ok[u] = row[u] < d;
            rs[u] = ok[u] ? __ldg(rp + row[u]) : 0;
            len[u] = ok[u] ? __ldg(rp + row[u] + 1) - rs[u] : 0;
        }
        double2 acc[U];
#pragma unroll
        for (int u = 0; u < U; u++) acc[u] = make_double2(0.0, 0.0);
        int64_t maxlen = len[0];
#pragma unroll
        for (int u = 1; u < U; u++) maxlen = len[u] > maxlen ? len[u] : maxlen;
        for (int64_t e0 = 0; e0 < maxlen; e0 += 4) {
            int c[U][4];
            double v[U][4];
            double2 xx[U][4];
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const bool in = e0 + q < len[u];
                    c[u][q] = in ? __ldg(ci + rs[u] + e0 + q) : -1;
                    v[u][q] = in ? __ldg(va + rs[u] + e0 + q) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < 4; q++)
                    xx[u][q] = c[u][q] >= 0 ? ld_nc2(x + (size_t)c[u][q] * K + p2)
                                            : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    acc[u].x = fma(v[u][q], xx[u][q].x, acc[u].x);
                    acc[u].y = fma(v[u][q], xx[u][q].y, acc[u].y);
                }
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            if (ok[u]) st2(y + (size_t)row[u] * K + p2, acc[u]);
    }
}

// ---------------------------------------------------------------------------
// Accumulation (reading G7): one CTA.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
finalize_kernel(const double* __restrict__ mu, const double* __restrict__ c, int64_t m,
                int32_t n, double* __restrict__ gamma_p, double* __restrict__ stats) {
    for (int64_t p = threadIdx.x; p < m; p += blockDim.x) {
        const double* row = mu + (size_t)p * (n + 1);
        double g = 0.0;
        for (int32_t j = 0; j <= n; j++) g = fma(c[j], row[j], g);
        gamma_p[p] = g;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        bool finite = true;
        for (int64_t p = 0; p < m; p++) {
            const double g = gamma_p[p];
            finite = finite && isfinite(g);
            s += g;
        }
        const double gamma = s / (double)m;
        double var = 0.0;
        for (int64_t p = 0; p < m; p++) {
            const double dv = gamma_p[p] - gamma;
            var = fma(dv, dv, var);
        }
        stats[0] = gamma;
        stats[1] = m > 1 ? sqrt(var / (double)(m - 1)) / sqrt((double)m) : 0.0;
        stats[2] = finite ? 1.0 : 0.0;
    }
}

// ---------------------------------------------------------------------------
// Spectral interval of B^T B.  out[0] <- min_i s_i as an ordered
// key, out[1] <- max row abs sum, out[2] <- max column abs sum (bit patterns of
// non-negative doubles order like integers).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long order_key(double x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(kThreads)
bounds_btb_kernel(int64_t d, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                  const double* __restrict__ va, const int64_t* __restrict__ trp,
                  const int32_t* __restrict__ tci, const double* __restrict__ tva,
                  unsigned long long* out) {
    double smin = INFINITY, rmax = 0.0, cmax = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
         i += (int64_t)gridDim.x * blockDim.x) {
        double diag = 0.0, roff = 0.0, rabs = 0.0, coff = 0.0, cabs = 0.0;
        for (int64_t e = rp[i]; e < rp[i + 1]; e++) {
            const double x = fabs(va[e]);
            rabs += x;
            if (ci[e] == i) diag = x; else roff += x;
        }
        for (int64_t e = trp[i]; e < trp[i + 1]; e++) {
            const double x = fabs(tva[e]);
            cabs += x;
            if (tci[e] != i) coff += x;
        }
        smin = fmin(smin, diag - 0.5 * (roff + coff));
        rmax = fmax(rmax, rabs);
        cmax = fmax(cmax, cabs);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        smin = fmin(smin, __shfl_xor_sync(0xffffffffu, smin, off));
        rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
        cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, off));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out + 0, order_key(smin));
        atomicMax(out + 1, order_key(rmax));
        atomicMax(out + 2, order_key(cmax));
    }
}

}  // namespace chebld
