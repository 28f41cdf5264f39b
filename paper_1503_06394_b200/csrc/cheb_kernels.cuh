// cheb_kernels.cuh -- sm_100a device kernels of the Chebyshev-Hutchinson hot path.
//
// Layout:
//   W[d][K]  fp64, the K probes of a block contiguous per row (row = 8K bytes).
//   S[d][WORDS] uint32 packed probe signs (bit p%32 of word p/32 set <=> v_p[i] = -1).
//
// Kernels
//   prep_kernel<MODE>               per-estimate operator prep: Ã's alpha/beta folded into a
//                                   padded value copy, padded col/row_ptr copies for 16-byte
//                                   bulk copies, "row has no stored diagonal" bitmap
//   probe_init_kernel<K,MODE>       K1: v -> W_cur, S; mu_0 = v^T v; rank-1 s_0 = u^T v
//   cheb_step_kernel<K,MODE,FIRST>  K2: fused CSR-SpMM x K probes + three-term recurrence +
//                                   Ã scaling + rank-1 term + per-probe dot v^T w_j, with a
//                                   deterministic last-CTA reduction (K4)
//   spmm_kernel<K>                  K3: Y = B W (first half of a B^T B application)
//   finalize_kernel                 Gamma_p, Gamma, stderr
//   bounds_btb_kernel               Johnson / norm bounds of B^T B
//
// The step kernel is a persistent grid (SMs x resident CTAs) walking row tiles
// t = blockIdx.x + i*gridDim.x in increasing order, so the rows in flight chip-wide form one
// narrow window and the W_cur halo rows i +- N of a stencil are re-read from L2, not HBM.
// Each CTA double-buffers its tiles in shared memory: one thread issues TMA bulk copies
// (cp.async.bulk, mbarrier completion) of the NEXT tile's row_ptr slice, col/val range,
// W_prev rows and sign words while all warps gather W_cur rows for the current tile.
#pragma once
#include <cassert>
#include <cstdint>
#include <type_traits>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

// CHEB_CHECKS=1 builds (scripts/build_variants.py "checked") turn on device-side bounds
// asserts: compute-sanitizer is not available on the B200 pool, so out-of-range gathers,
// staging overflows and bad tile geometry trap here instead.
#ifndef CHEB_CHECKS
#define CHEB_CHECKS 0
#endif
#if CHEB_CHECKS
#define CHEB_ASSERT(x) assert(x)
#else
#define CHEB_ASSERT(x) ((void)0)
#endif

namespace chebld {

namespace cg = cooperative_groups;

constexpr int kThreads = 256;
#ifndef CHEB_MIN_CTAS
#define CHEB_MIN_CTAS 4  // resident CTAs per SM the step kernel is register-budgeted for
#endif
#ifndef CHEB_MIN_CTAS_DBL
#define CHEB_MIN_CTAS_DBL 3  // moment doubling carries two more accumulator channels
#endif
#ifndef CHEB_DBL_STAGE_WC
#define CHEB_DBL_STAGE_WC 0  // 1: moment doubling stages the tile's own W_cur rows (else: first gather)
#endif
#ifndef CHEB_RPG_DBL
#define CHEB_RPG_DBL 2  // rows per lane group of the moment-doubling kernels (32-row tiles at k=64)
#endif
#ifndef CHEB_RPG
#define CHEB_RPG 2  // rows per lane group per tile (tile = 256*RPG*4/K rows)
#endif
#ifndef CHEB_STAGES
#define CHEB_STAGES 2  // shared-memory pipeline depth of cheb_step_kernel
#endif
#ifndef CHEB_DECOUPLE
// per-stage "consumed" mbarriers instead of a CTA barrier after each tile of cheb_step_kernel:
// 0 never, 1 always, 2 (default) on the small-tile geometry (RP = 1: k <= 16 and L2-resident
// operators; configs[3] at k = 16: 1541 vs 1575 ms per estimate, at k = 64 with 32-row tiles
// 1276 vs 1253 ms, so not there)
#define CHEB_DECOUPLE 2
#endif
constexpr int kStepStages = CHEB_STAGES;
#ifndef CHEB_CAP_PER_ROW
#define CHEB_CAP_PER_ROW 8  // staged nonzeros per tile row (average)
#endif
#ifndef CHEB_NNZ_UNROLL
#define CHEB_NNZ_UNROLL 5  // nnz of a row whose gathers are in flight together (5-point stencil: 1 chunk)
#endif

// MODE_FAM: a one-parameter family M_r = D + theta_r O of a base CSR (D its diagonal, O the rest),
// R values of theta in the columns of one probe block (the rho-likelihood scan)
enum { MODE_CSR = 0, MODE_RANK1 = 1, MODE_BTB = 2, MODE_FAM = 3 };

__host__ __device__ constexpr int words_for(int K) { return K >= 32 ? K / 32 : 1; }

// Probes per lane of the step kernels: PPL/2 16-byte slots per gathered row (4: two slots, the
// probes {2l, 2l+1, K/2+2l, K/2+2l+1}; 8: four slots at stride K/4).  More probes per lane
// amortise the per-nonzero index work (column/value reads, address math) over more DFMAs.
#ifndef CHEB_PPL
#define CHEB_PPL 4
#endif
constexpr int kPPL = CHEB_PPL;
// 256-bit gathers and stores (sm_100 LDG/STG .ENL2.256): a lane's 4 probes are contiguous, so one
// 32-byte access per gathered row instead of two 16-byte ones at stride K/2 (CHEB_WIDE=0: the split
// layout {2l, 2l+1} + {K/2+2l, K/2+2l+1}).  Both cover whole 32-byte sectors per row.
// 0 never, 1 always, 2 (default) for probe blocks k <= CHEB_WIDE_MAXK (configs[3] per estimate:
// k = 16 1534 vs 1686 ms; k = 32 1386 vs 1334 ms and k = 64 1388 vs 1328 ms in favour of the split
// layout, whose 16-byte accesses already cover whole sectors of 2+ rows per warp instruction)
#ifndef CHEB_WIDE
#define CHEB_WIDE 2
#endif
#ifndef CHEB_WIDE_MAXK
#define CHEB_WIDE_MAXK 16
#endif
__host__ __device__ constexpr bool wide_k(int K) {
    return kPPL == 4 && (CHEB_WIDE == 1 || (CHEB_WIDE == 2 && K <= CHEB_WIDE_MAXK));
}
static_assert(kPPL == 4 || kPPL == 8, "CHEB_PPL must be 4 or 8");

// Geometry of the step / spmm kernels: each lane owns PPL probes in PPL/2 slots of two
// consecutive probes, L = K/PPL lanes own a row; RPG rows per group per tile.  The tile
// (rows) does not depend on PPL.
// R4: rows per lane group at PPL = 4 (CHEB_RPG; the moment-doubling kernels use CHEB_RPG_DBL).
template <int K, int R4 = CHEB_RPG>
struct Geo {
    static_assert(K == 8 || K == 16 || K == 32 || K == 64 || K == 128, "K in {8,...,128}");
    static constexpr int PPL = kPPL;
    static constexpr int NSL = PPL / 2;             // 16-byte slots per lane and row
    static constexpr int SS = K / NSL;              // probe stride between a lane's slots (split layout)
    static constexpr bool WIDE = wide_k(K);         // 256-bit accesses, a lane's probes contiguous
    // first probe of slot sl of lane lg: contiguous with 256-bit accesses, split otherwise
    __host__ __device__ static constexpr int lane_probe(int lg, int sl) {
        return WIDE ? PPL * lg + 2 * sl : 2 * lg + sl * SS;
    }
    static constexpr int L = K / PPL;               // lanes per row: 1..32
    static constexpr int GROUPS = kThreads / L;     // rows in flight per CTA
    static constexpr int RPG = R4 * 4 / PPL;        // rows per group per tile
    static_assert(RPG >= 1, "CHEB_RPG too small for CHEB_PPL");
    static constexpr int TILE = GROUPS * RPG;       // rows per tile: 256 .. 16
    static constexpr int WORDS = words_for(K);
    static constexpr int CAP = TILE * CHEB_CAP_PER_ROW;  // staged nnz capacity (rows of a tile with more
                                                        // nnz in total gather col/val from global)
    static constexpr int RED_T = kThreads / K;      // threads per probe in the final reduction
    // shared-memory stage layout (bytes, every field 16-byte aligned)
    static constexpr int WBYTES = TILE * K * 8;     // 16 KB
    static constexpr int RPBYTES = (TILE + 2) * 8;
    static constexpr int COLBYTES = (CAP + 8) * 4;
    static constexpr int VALBYTES = (CAP + 4) * 8;
    static constexpr int SGNBYTES = ((TILE * WORDS * 4 + 15) / 16) * 16;
    static constexpr int UBYTES = ((TILE * 8 + 15) / 16) * 16;
};

// WC: the tile's own W_cur rows are staged too (always for BTB; the per-step moment-doubling
// kernel needs w_{j-1}[i] for its w_j^T w_{j-1} dot).
// spmm_kernel: 4 probes per lane in two slots {2l, 2l+1, K/2+2l, K/2+2l+1}, K/4 lanes per row
template <int K>
struct SpmmGeo {
    static constexpr int L = K / 4;
    static constexpr int GROUPS = kThreads / L;
};

template <int K, int MODE, bool WC = false, int R4 = CHEB_RPG>
struct StageLayout {
    using G = Geo<K, R4>;
    static constexpr bool HAS_WC = (MODE == MODE_BTB) || WC;
    static constexpr int OFF_WPREV = 0;
    static constexpr int OFF_WCUR = OFF_WPREV + G::WBYTES;                       // HAS_WC only
    static constexpr int OFF_VAL = OFF_WCUR + (HAS_WC ? G::WBYTES : 0);
    static constexpr int OFF_RP = OFF_VAL + G::VALBYTES;
    static constexpr int OFF_COL = OFF_RP + G::RPBYTES;
    static constexpr int OFF_SGN = OFF_COL + G::COLBYTES;
    static constexpr int OFF_U = OFF_SGN + G::SGNBYTES;                          // RANK1 only
    static constexpr int BYTES = OFF_U + (MODE == MODE_RANK1 || MODE == MODE_FAM ? G::UBYTES : 0);  // u / D
    static constexpr int SMEM = 2 * BYTES;                                       // double buffer
};

// ---------------------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA bulk copy (cp.async.bulk, SASS UBLKCP)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {  // release.cta
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
#ifndef CHEB_MBAR_SUSPEND_NS
#define CHEB_MBAR_SUSPEND_NS 0  // try_wait suspend-time hint (0: the hardware default)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    do {
        if (CHEB_MBAR_SUSPEND_NS > 0) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(addr), "r"(phase), "r"((uint32_t)CHEB_MBAR_SUSPEND_NS)
                : "memory");
        } else {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(addr), "r"(phase)
                : "memory");
        }
    } while (!done);
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// global -> shared bulk copy, completion counted on `bar` (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
        "[%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// SplitMix64 at flat counter t of the stream seeded `seed` (reading G6).
__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t t) {
    uint64_t z = seed + t * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ int64_t imin64(int64_t x, int64_t y) { return x < y ? x : y; }

// +-1.0 from bit `b` of `w` (set -> -1.0, the probe convention)
__device__ __forceinline__ double pm1(uint32_t w, int b) {
    return __hiloint2double((int)(0x3FF00000u | (((w >> b) & 1u) << 31)), 0);
}

// x with its sign bit xor'ed by bit 31 of m (exactly -x or x)
// 8-byte global -> shared async copy (LDGSTS): the data never occupies a register
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ double signflip(double x, uint32_t m) {
    return __hiloint2double(__double2hiint(x) ^ (int)(m & 0x80000000u), __double2loint(x));
}

__device__ __forceinline__ double2 ldg2(const double* p) {
    return __ldg(reinterpret_cast<const double2*>(p));
}
// 32 contiguous bytes (32-byte aligned): read-only path / L1-allocating coherent path
__device__ __forceinline__ void ldg4(const double* p, double2& lo, double2& hi) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(lo.x), "=d"(lo.y), "=d"(hi.x), "=d"(hi.y) : "l"(p));
}
__device__ __forceinline__ void ldca4(const double* p, double2& lo, double2& hi) {
    asm volatile("ld.global.ca.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(lo.x), "=d"(lo.y), "=d"(hi.x), "=d"(hi.y) : "l"(p));
}
__device__ __forceinline__ void stcs4(double* p, double2 lo, double2 hi) {  // streaming store
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(lo.x), "d"(lo.y), "d"(hi.x),
                 "d"(hi.y)
                 : "memory");
}

struct StepArgs {
    int64_t d;            // rows of the gather matrix (= dimension of M)
    int64_t ntiles;
    const int64_t* rp;    // prepped gather matrix: padded row_ptr copy
    const int32_t* ci;    //   padded col copy
    const double* va;     //   padded scaled values (alpha*a, diagonal alpha*a_ii - beta)
    const double* xg;     // gather source: W_cur (csr/rank1) or Y = B W_cur (btb)
    const double* wcur;   // W_cur
    double* wnext;        // in: W_prev (unless FIRST); out: W_next (in place)
    const uint32_t* sbits;
    double beta;          // for rows without a stored diagonal (csr/rank1) and for btb
    double r1c_alpha;     // alpha * c (rank-1)
    const double* r1u;    // padded u copy (nullptr = ones)
    const double* s_cur;  // [K] u^T w_{j-1}
    double* s_next;       // [K] u^T w_j
    double* part;         // per-CTA partials [NCH][gridDim.x][K]
    double* gpart;        // reduction-group sums [NCH][ng][K] (persistent: [2][NCH][ng][K])
    int32_t fam_kp;       // MODE_FAM: probes per family member in a block (column c: member c / fam_kp,
                          // probe c % fam_kp); 0 otherwise
    int32_t fam_r;        // MODE_FAM: family members with output rows (columns of padding members skipped)
    int64_t fam_rstride;  // MODE_FAM: doubles between the mu rows of consecutive members
    const double* fam_coef;  // MODE_FAM: [3][K] per column: alpha_c, beta_c, alpha_c * theta_c
    int32_t rg;           // reduction group size (0: red_group(gridDim.x)); the persistent kernel's
                          // cluster size, so per-step launches of the same grid reduce identically
    unsigned int* ticket;
    double* mu_out;       // mu_out[p*mu_stride + mu_col]
    int64_t mu_stride;
    int32_t mu_col;
    int32_t kvalid;       // probes of this block that exist (<= K)
    // compressed gather matrix (csr / rank-1 per-step kernels; cv_prep_kernels): usable when
    // *cv_ok != 0 -- every prepped row has exactly CHEB_NNZ_UNROLL entries, entry e of row i is
    // (i + cv_dc[e], cv_tab[cv_vi[e]])
    const int32_t* cv_ok;
    const int16_t* cv_dc;
    const uint8_t* cv_vi;
    const double* cv_tab;  // [kCvSlots]
};

// ---------------------------------------------------------------------------------------
// Canonical (deterministic) reduction of the per-CTA partials part[c][p], c < G.
// Reduction groups of RG = red_group(G) consecutive CTAs: group q covers c in
// [q*RG, min(G, (q+1)*RG)).  For probe p:
//     S_q = (((0 + part[q*RG][p]) + part[q*RG+1][p]) + ...)      (ascending c)
//     mu  = the fixed tree of group_tree_sum over S_0 .. S_{ng-1}
// Every kernel that produces moments uses exactly this order, so the result depends only on
// the grid size G -- not on which kernel or CTA computed it.  The per-step kernels form the S_q
// in their last CTA from global partials; the persistent kernel runs each group as a thread-
// block cluster and forms S_q from its CTAs' shared memory (DSMEM), so one grid-wide barrier
// per step suffices (every CTA then sums the ng = ceil(G/RG) group sums itself).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum_xor(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

constexpr int kRedGroup = 8;      // portable cluster size: the default reduction group
constexpr int kMaxRedGroup = 16;  // largest (non-portable) cluster the persistent kernel may use
__host__ __device__ constexpr int red_group(int G, int rg = kRedGroup) { return G < rg ? (G < 1 ? 1 : G) : rg; }

// Second level of the canonical order for one channel: gp = that channel's group sums [ng][K].
// Thread t handles probe t / T and the groups q = t % T, t % T + T, ... (ascending), T = 256 / K
// consecutive lanes per probe; their partial sums are combined by the xor butterfly T/2, ..., 1,
// so every lane of the probe ends with the same value.  All kThreads threads must call it.
template <int K>
__device__ __forceinline__ double group_tree_sum(const double* gp, int ng) {
    constexpr int T = kThreads / K;
    const int p = threadIdx.x / T, u = threadIdx.x % T;
    double t = 0.0;
    constexpr int B = 16;  // loads in flight per batch (one L2 round trip for ng <= 16 T), then the adds in ascending q
    for (int q0 = u; q0 < ng; q0 += B * T) {
        double v[B];
#pragma unroll
        for (int r = 0; r < B; r++) v[r] = q0 + r * T < ng ? __ldcg(gp + (size_t)(q0 + r * T) * K + p) : 0.0;
#pragma unroll
        for (int r = 0; r < B; r++) t += v[r];
    }
#pragma unroll
    for (int off = T / 2; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    return t;
}

// All K probes of NCH channels by one CTA (last-CTA-done epilogue).  part: [NCH][G][K] (global,
// written by other CTAs); gpart: [NCH][ng][K] global scratch; out: shared [NCH][K].
template <int K, int NCH>
__device__ __forceinline__ void reduce_partials_grouped(const double* part, int G, int RG, double* gpart,
                                                        double (*out)[K]) {
    const int ng = (G + RG - 1) / RG;
    for (int x = threadIdx.x; x < NCH * ng * K; x += kThreads) {
        const int p = x % K, q = (x / K) % ng, ch = x / (K * ng);
        const int c0 = q * RG, cn = (G - c0) < RG ? (G - c0) : RG;
        const double* src = part + ((size_t)ch * G + c0) * K + p;
        double v[kMaxRedGroup], sq = 0.0;
#pragma unroll
        for (int r = 0; r < kMaxRedGroup; r++) v[r] = r < cn ? __ldcg(src + (size_t)r * K) : 0.0;
#pragma unroll
        for (int r = 0; r < kMaxRedGroup; r++) sq += v[r];
        gpart[((size_t)ch * ng + q) * K + p] = sq;
    }
    __syncthreads();  // block-level visibility of the gpart stores
#pragma unroll
    for (int ch = 0; ch < NCH; ch++) {
        const double t = group_tree_sum<K>(gpart + (size_t)ch * ng * K, ng);
        if (threadIdx.x % (kThreads / K) == 0) out[ch][threadIdx.x / (kThreads / K)] = t;
    }
    __syncthreads();
}

// Lane lg of a row group owns probes probe_of<K,PPL,SPLIT>(lg, q), q < PPL: contiguous
// (pl = PPL*lg + q) or, with SPLIT, PPL/2 pairs at stride K/(PPL/2): {2lg, 2lg+1} + s*K/(PPL/2)
// (PPL = 4: {2lg, 2lg+1, K/2+2lg, K/2+2lg+1}) so that every 16-byte access of a warp is contiguous.
template <int K, int PPL, bool SPLIT>
__device__ __forceinline__ int probe_of(int lg, int q) {
    return SPLIT ? 2 * lg + (q & 1) + (q >> 1) * (K / (PPL / 2)) : PPL * lg + q;
}

// Epilogues of the last CTA:
//   EPI_STEP  ch0 -> mu[p][col]                        (+ rank-1: ch1 -> s_next)
//   EPI_DBL   moment doubling, step j = col: ch0 = w_j^T w_j, ch1 = w_j^T w_{j-1}
//             mu[p][2j] = 2 ch0 - mu[p][0],  mu[p][2j-1] = 2 ch1 - mu[p][1]  (j = 1: mu[p][1] = ch1)
//             (indices > n = mu_stride - 1 are not written)   (+ rank-1: ch2 -> s_next)
enum { EPI_STEP = 0, EPI_DBL = 2 };

// Moment-doubling epilogue for one probe row (T_{2j} = 2 T_j^2 - I, T_{2j+1} = 2 T_{j+1} T_j - T_1
// for the symmetric Ã; reading G25).
__device__ __forceinline__ void dbl_write(double* row, int j, int64_t n, double q, double r) {
    if (j == 1) {
        if (n >= 1) row[1] = r;
    } else if (2 * (int64_t)j - 1 <= n) {
        row[2 * j - 1] = 2.0 * r - row[1];
    }
    if (2 * (int64_t)j <= n) row[2 * j] = 2.0 * q - row[0];
}

// Shared-memory scratch of grid_reduce_finish (aliases the callers' dynamic shared memory,
// which is idle once every tile is consumed): red[NCH][8][K], fin[NCH][K].
template <int K, int NCH>
__host__ __device__ constexpr int red_scratch_bytes() {
    return 8 * (NCH * (kThreads / 32) * K + NCH * K);
}

template <int K, int PPL, int NCH, int EPI, bool HAS_S, bool SPLIT = false>
__device__ __forceinline__ void grid_reduce_finish(double (&acc)[NCH][PPL], const StepArgs& a,
                                                   unsigned char* scratch) {
    constexpr int LG = K / PPL;
    auto red = reinterpret_cast<double(*)[kThreads / 32][K]>(scratch);
    auto fin = reinterpret_cast<double(*)[K]>(scratch + 8 * NCH * (kThreads / 32) * K);
    __shared__ bool is_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lg = lane % LG;
#pragma unroll
    for (int off = LG; off < 32; off <<= 1) {
#pragma unroll
        for (int ch = 0; ch < NCH; ch++)
#pragma unroll
            for (int q = 0; q < PPL; q++) acc[ch][q] += __shfl_xor_sync(0xffffffffu, acc[ch][q], off);
    }
    if (lane < LG && warp < kThreads / 32) {  // extra (producer) warps contribute nothing
#pragma unroll
        for (int q = 0; q < PPL; q++) {
            const int p = probe_of<K, PPL, SPLIT>(lg, q);
#pragma unroll
            for (int ch = 0; ch < NCH; ch++) red[ch][warp][p] = acc[ch][q];
        }
    }
    __syncthreads();
    if (tid < K) {
#pragma unroll
        for (int ch = 0; ch < NCH; ch++) {
            double m = 0.0;
#pragma unroll
            for (int w = 0; w < kThreads / 32; w++) m += red[ch][w][tid];
            a.part[((size_t)ch * gridDim.x + blockIdx.x) * K + tid] = m;
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned int prev = atomicAdd(a.ticket, 1u);
        is_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    reduce_partials_grouped<K, NCH>(a.part, (int)gridDim.x, a.rg > 0 ? a.rg : red_group((int)gridDim.x), a.gpart, fin);
    if (tid < K) {
        // MODE_FAM: column tid is probe tid % fam_kp of family member tid / fam_kp
        const int pc = a.fam_kp ? tid % a.fam_kp : tid, mc = a.fam_kp ? tid / a.fam_kp : 0;
        double* row = a.mu_out + (size_t)mc * a.fam_rstride + (size_t)pc * a.mu_stride;
        if (pc < a.kvalid && (!a.fam_kp || mc < a.fam_r)) {
            if (EPI == EPI_STEP) row[a.mu_col] = fin[0][tid];
            if (EPI == EPI_DBL) dbl_write(row, a.mu_col, a.mu_stride - 1, fin[0][tid], fin[1][tid]);
        }
        if (HAS_S) a.s_next[tid] = fin[NCH - 1][tid];
    }
    if (tid == 0) *a.ticket = 0u;  // re-arm for the next launch (stream-ordered)
}

// ---------------------------------------------------------------------------------------
// Operator prep (once per estimate): padded copies for 16-byte bulk copies and the Ã map
// folded into the values:  val'_e = alpha*a_e (- beta if e is row i's diagonal, csr/rank1).
// ---------------------------------------------------------------------------------------
// Padded row lengths: every row of the prepped gather matrix is padded to a multiple of the
// gather chunk U = CHEB_NNZ_UNROLL with entries (column i, value 0), so the step kernels' chunk
// loop needs no bounds checks.  cnt[i] = ceil(nnz_i / U) * U, cnt[d] = 0 (exclusive-scanned into
// the prepped row pointer).
__global__ void __launch_bounds__(kThreads)
prep_count_kernel(int64_t d, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int with_diag,
                  int64_t* __restrict__ cnt) {
    constexpr int U = CHEB_NNZ_UNROLL;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= d; i += (int64_t)gridDim.x * blockDim.x) {
        if (i == d) {
            cnt[i] = 0;
            continue;
        }
        int64_t len = rp[i + 1] - rp[i];
        if (with_diag) {  // csr / rank-1: one extra slot for the -beta entry of a row with no stored diagonal
            bool has = false;
            for (int64_t e = rp[i]; e < rp[i + 1]; e++) has |= (ci[e] == i);
            len += has ? 0 : 1;
        }
        cnt[i] = (len + U - 1) / U * U;
    }
}

// rp2: prepped row pointer (exclusive scan of the padded lengths, entries [0, d]); this kernel
// writes the scaled entries of row i at rp2[i].. and pads the row with (i, 0.0).  A csr / rank-1
// row's first entry is its diagonal (alpha a_ii - beta, or (i, -beta) in the slot prep_count_kernel
// reserved when none is stored), so every row of Ã = alpha M - beta I is a plain sparse row and the
// step kernels have no diagonal special case; padding (i, 0.0) adds exact zeros.
template <int MODE>
__global__ void __launch_bounds__(kThreads)
prep_kernel(int64_t d, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
            const double* __restrict__ va, double alpha, double beta, int64_t* __restrict__ rp2,
            int64_t rp2_len, int32_t* __restrict__ ci2, double* __restrict__ va2,
            const double* __restrict__ u, double* __restrict__ u2) {
    const int64_t total = rp2[d];  // padded nnz
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // multiple of 32
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < d; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        bool has = true;
        if (i < d) {
            const int64_t e0 = rp[i], e1 = rp[i + 1];
            const int64_t o0 = rp2[i], o1 = rp2[i + 1];
            has = (MODE == MODE_BTB);
            int64_t o = o0;
            if (MODE == MODE_FAM) {
                // family: raw off-diagonal values O (each member scales them by its alpha theta in
                // the kernel); the head slot (i, 0.0) gathers w_{j-1}[i], D_i goes to u2[i]
                double dv = 0.0;
                o = o0 + 1;
                for (int64_t e = e0; e < e1; e++) {
                    const int32_t c = ci[e];
                    if (c == i) {
                        dv = va[e];
                    } else {
                        ci2[o] = c;
                        va2[o] = va[e];
                        o++;
                    }
                }
                ci2[o0] = (int32_t)i;
                va2[o0] = 0.0;
                u2[i] = dv;
            } else if (MODE != MODE_BTB) {
                // csr / rank-1: the diagonal entry first (alpha a_ii - beta, or -beta when none is
                // stored), then the off-diagonal entries in CSR order: the doubling kernels take
                // w_{j-1}[i] from the row's first gather
                double dv = -beta;
                o = o0 + 1;
                for (int64_t e = e0; e < e1; e++) {
                    const int32_t c = ci[e];
                    if (c == i) {
                        dv = fma(alpha, va[e], -beta);
                        has = true;
                    } else {
                        ci2[o] = c;
                        va2[o] = alpha * va[e];
                        o++;
                    }
                }
                ci2[o0] = (int32_t)i;
                va2[o0] = dv;
            } else {
                for (int64_t e = e0; e < e1; e++, o++) {
                    const int32_t c = ci[e];
                    ci2[o] = c;
                    va2[o] = alpha * va[e];
                }
            }
            for (; o < o1; o++) {  // padding: (i, 0.0)
                ci2[o] = (int32_t)i;
                va2[o] = 0.0;
            }
            if (u2 && MODE != MODE_FAM) u2[i] = u ? u[i] : 1.0;
        }
    }
    if (blockIdx.x == 0) {
        for (int64_t k = d + 1 + threadIdx.x; k < rp2_len; k += blockDim.x) rp2[k] = total;
        if (threadIdx.x < 8) ci2[total + threadIdx.x] = 0;
        if (threadIdx.x < 4) va2[total + threadIdx.x] = 0.0;
        if (u2 && threadIdx.x < 2) u2[d + threadIdx.x] = 0.0;
    }
}

// ---------------------------------------------------------------------------------------
// Compressed gather matrix (the "CV" format: value-indexed, delta-coded columns -- the matrix
// compression of the SpMV literature).  When every prepped row has exactly U = CHEB_NNZ_UNROLL
// entries, every column is within int16 of its row and the prepped values take at most
// kCvMaxValues distinct bit patterns (stencil precisions, graph Laplacians: configs[0..3]), an
// entry costs 3 bytes (int16 column delta + uint8 value index) instead of 12, and the row pointer
// is implicit (row i = entries [U i, U i + U)): at configs[3], k = 16, 11.37 -> 10.05 GB per step.
// The decoded (column, value) pairs are bit-identical to the plain copy, so are the moments.
// The format check runs on the device (no host round trip): cv_ok stays 1 only if it holds.
// ---------------------------------------------------------------------------------------
#ifndef CHEB_CV_KERNEL
#define CHEB_CV_KERNEL 1  // 0: the step kernels never read the compressed copy (A/B builds)
#endif
constexpr int kCvSlots = 256;       // open-addressing table of value bit patterns
constexpr int kCvMaxValues = 128;   // at most half full: short probe chains
constexpr uint64_t kCvEmpty = ~0ull;

__device__ __forceinline__ int cv_hash(uint64_t k) { return (int)((k * 0x9E3779B97F4A7C15ull) >> 56); }

// Insert every prepped value into the table (tab: kCvSlots keys, set to kCvEmpty; meta[0] = ok,
// meta[1] = distinct count).  Each thread remembers its last 4 distinct values, so a matrix with
// a handful of values touches the table a handful of times per thread.
__global__ void __launch_bounds__(kThreads)
cv_values_kernel(int64_t total, const double* __restrict__ va2, unsigned long long* __restrict__ tab,
                 int32_t* __restrict__ meta) {
    uint64_t seen[4] = {kCvEmpty, kCvEmpty, kCvEmpty, kCvEmpty};
    int ns = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = (uint64_t)__double_as_longlong(va2[e]);
        if (k == seen[0] || k == seen[1] || k == seen[2] || k == seen[3]) continue;
        if (k == kCvEmpty || *(volatile int32_t*)meta == 0) {
            meta[0] = 0;
            return;
        }
        int h = cv_hash(k), n = 0;
        for (; n < kCvSlots; n++, h = (h + 1) & (kCvSlots - 1)) {
            const unsigned long long prev = atomicCAS(tab + h, (unsigned long long)kCvEmpty, (unsigned long long)k);
            if (prev == kCvEmpty) {  // inserted
                if (atomicAdd(meta + 1, 1) + 1 > kCvMaxValues) meta[0] = 0;
                break;
            }
            if (prev == k) break;  // present
        }
        if (n == kCvSlots) meta[0] = 0;
        seen[ns++ & 3] = k;
    }
}

// Encode the prepped copy: uniform rows (padded length U), int16 column deltas, value indices
// (slots of the table).  Any violation clears meta[0].
__global__ void __launch_bounds__(kThreads)
cv_encode_kernel(int64_t d, const int64_t* __restrict__ rp2, const int32_t* __restrict__ ci2,
                 const double* __restrict__ va2, const unsigned long long* __restrict__ tab,
                 int16_t* __restrict__ dc, uint8_t* __restrict__ vi, int32_t* __restrict__ meta) {
    constexpr int U = CHEB_NNZ_UNROLL;
    __shared__ unsigned long long t[kCvSlots];
    for (int x = threadIdx.x; x < kCvSlots; x += blockDim.x) t[x] = tab[x];
    __syncthreads();
    bool ok = true;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
        if (rp2[i] != U * i || rp2[i + 1] != U * (i + 1)) {
            ok = false;
            break;
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int64_t e = U * i + q;
            const int64_t del = (int64_t)ci2[e] - i;
            const uint64_t k = (uint64_t)__double_as_longlong(va2[e]);
            int h = cv_hash(k), n = 0;
            while (t[h] != k && n < kCvSlots) {
                h = (h + 1) & (kCvSlots - 1);
                n++;
            }
            ok = ok && del >= -32768 && del <= 32767 && n < kCvSlots;
            dc[e] = (int16_t)del;
            vi[e] = (uint8_t)h;
        }
    }
    if (!ok) meta[0] = 0;
}

// ---------------------------------------------------------------------------------------
// K1: probe initialisation.  W_cur[i][p] = v_p[i] = +-1 (global probe p0+p), sign bits,
// mu_0 = v^T v (= d exactly), rank-1 s_0 = u^T v.
// ---------------------------------------------------------------------------------------
template <int K, int MODE>
__global__ void __launch_bounds__(kThreads)
probe_init_kernel(StepArgs a, uint64_t seed, uint64_t p0, double* w0, uint32_t* sbits) {
    constexpr int PPL = K <= 64 ? 2 : 4;
    constexpr int LG = K / PPL;               // <= 32
    constexpr int GROUPS = kThreads / LG;
    constexpr int WORDS = words_for(K);
    constexpr bool HAS_S = (MODE == MODE_RANK1);
    const int lg = threadIdx.x % LG;
    const int group = threadIdx.x / LG;
    const int pl = PPL * lg;
    const uint64_t d = (uint64_t)a.d;
    constexpr int NCH = HAS_S ? 2 : 1;
    double acc[NCH][PPL];
#pragma unroll
    for (int ch = 0; ch < NCH; ch++)
#pragma unroll
        for (int q = 0; q < PPL; q++) acc[ch][q] = 0.0;
    const int64_t niter = (a.d + GROUPS - 1) / GROUPS;
    for (int64_t t = blockIdx.x; t < niter; t += gridDim.x) {
        const int64_t i = t * GROUPS + group;
        const bool ok = i < a.d;
        uint32_t bits = 0;
        if (ok) {
            double v[PPL];
#pragma unroll
            for (int q = 0; q < PPL; q++) {
                const uint64_t pc = MODE == MODE_FAM ? (uint64_t)((pl + q) % a.fam_kp) : (uint64_t)(pl + q);
                const uint64_t z = splitmix64_at(seed, (p0 + pc) * d + (uint64_t)i + 1ull);
                const uint32_t bq = (uint32_t)(z >> 63);
                v[q] = bq ? -1.0 : 1.0;
                bits |= bq << ((pl + q) & 31);
                acc[0][q] += v[q] * v[q];
            }
            if (w0)  // nullptr: the per-step path reads v from the sign bits only
#pragma unroll
                for (int q = 0; q < PPL; q += 2)
                    *reinterpret_cast<double2*>(w0 + (size_t)i * K + pl + q) = make_double2(v[q], v[q + 1]);
            if (HAS_S) {
                const double u = a.r1u ? a.r1u[i] : 1.0;
#pragma unroll
                for (int q = 0; q < PPL; q++) acc[NCH - 1][q] += u * v[q];
            }
        }
        // OR the bits of the lanes that share one 32-bit word
        constexpr int LW = (32 / PPL) < LG ? (32 / PPL) : LG;
#pragma unroll
        for (int off = 1; off < LW; off <<= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, off);
        if (ok && (lg % LW) == 0) sbits[(size_t)i * WORDS + (pl >> 5)] = bits;
    }
    extern __shared__ __align__(128) unsigned char smem[];
    grid_reduce_finish<K, PPL, NCH, EPI_STEP, HAS_S>(acc, a, smem);
}

// ---------------------------------------------------------------------------------------
// K2: the fused Chebyshev step (w_j from w_{j-1}, w_{j-2}):
//   y    = sum_e val'_e xg[col_e]  [- beta*wcur_i if no stored diagonal / btb]
//          [+ alpha*c*u_i*s_cur]                    (Ã w_{j-1}, alpha/beta folded in val')
//   w_j  = FIRST ? y : 2y - w_{j-2}                 (written over w_{j-2})
//   mu_j += v_i * w_j ;  rank-1: s_j += u_i * w_j
// ---------------------------------------------------------------------------------------
// Gather of data written earlier in the same launch (fused kernel, stage 2): a plain
// L1-allocating load (not the read-only .nc path).  L1 is invalidated at launch and rows are
// only read after they are final, so no stale line can be cached.
__device__ __forceinline__ double2 ldcg2(const double* p) {
    double2 v;
    asm volatile("ld.global.ca.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

// One staged tile of the fused step.  xg: gather source; wcur: W_cur (for rows without a
// stored diagonal); wout: output rows (in place over W_prev).  CG: gather through L2 only
// (data produced earlier in the same launch by other CTAs -- temporally fused kernel).
// Accumulator channels (acc[ch][q], probe q of the lane):
//   !DBL: ch0 = v^T w_j (sign bits)                        [+ rank-1 ch1 = u^T w_j]
//    DBL: ch0 = w_j^T w_j, ch1 = w_{j-1}^T w_j (own rows)   [+ rank-1 ch2 = u^T w_j]
template <int MODE, bool DBL>
__host__ __device__ constexpr int n_channels() { return (DBL ? 2 : 1) + (MODE == MODE_RANK1 ? 1 : 0); }

// VB: the probe vector v = w_0 is never materialised in HBM on the per-step path, its sign bits
// stand in for it: VB = 1 (step 1) gathers v from the bits, VB = 2 (step 2) takes w_{j-2} = v
// from the staged bits.  x * (+-1) is exact, so results are bit-identical to reading v.
// CV: the tile's matrix is staged in the compressed format (int16 column deltas in the col slot,
// uint8 value indices in the val slot, table cvt in shared memory; rows of exactly U entries).
template <int K, int MODE, bool FIRST, bool STAGED, bool CG = false, bool DBL = false,
          bool WCS = false, int R4 = CHEB_RPG, int VB = 0, bool CV = false>
__device__ __forceinline__ void step_tile(const StepArgs& a, const unsigned char* st, int64_t r0, int rows,
                                          int64_t base_c, int64_t base_v, const double2 (&r1)[kPPL / 2],
                                          double (&acc)[n_channels<MODE, DBL>()][kPPL], const double* xg,
                                          const double* wcur, double* wout, const double* fcoef = nullptr,
                                          const double* cvt = nullptr) {
    using G = Geo<K, R4>;
    using SL = StageLayout<K, MODE, WCS, R4>;
    constexpr int NSL = G::NSL;
    constexpr bool OWN_SMEM = SL::HAS_WC;          // w_{j-1}[i] rows staged in shared memory
    // csr / rank-1 doubling: w_{j-1}[i] is the row's first gather (the prepped diagonal entry)
    constexpr bool OWN_GATHER = (DBL && !OWN_SMEM && MODE != MODE_BTB) || MODE == MODE_FAM;
    constexpr bool OWN_EARLY = DBL && !OWN_SMEM && !OWN_GATHER;  // loaded at the row start
    static_assert(VB == 0 || (MODE != MODE_BTB && !CG && (VB != 1 || !OWN_SMEM)),
                  "sign-bit probes: per-step csr/rank-1");
    constexpr bool HAS_S = (MODE == MODE_RANK1);
    constexpr int SCH = n_channels<MODE, DBL>() - 1;  // rank-1 channel
    const int lg = threadIdx.x % G::L;
    const int grp = threadIdx.x / G::L;
    int pp[NSL];  // first probe of each slot: {2lg, 2lg+1} + s*SS
#pragma unroll
    for (int sl = 0; sl < NSL; sl++) pp[sl] = G::lane_probe(lg, sl);
    const int64_t* rp_s = reinterpret_cast<const int64_t*>(st + SL::OFF_RP);
    const int32_t* col_s = reinterpret_cast<const int32_t*>(st + SL::OFF_COL);
    const double* val_s = reinterpret_cast<const double*>(st + SL::OFF_VAL);
    const double* wp_s = reinterpret_cast<const double*>(st + SL::OFF_WPREV);
    const double* wc_s = reinterpret_cast<const double*>(st + SL::OFF_WCUR);
    const uint32_t* sg_s = reinterpret_cast<const uint32_t*>(st + SL::OFF_SGN);
    const double* u_s = reinterpret_cast<const double*>(st + SL::OFF_U);
    const double* xl = xg + pp[0];
#pragma unroll
    for (int rr = 0; rr < G::RPG; rr++) {
        const int lr = grp + rr * G::GROUPS;
        if (lr >= rows) break;
        const int64_t i = r0 + lr;
        const int64_t e_lo = CV ? 0 : rp_s[lr], e_hi = CV ? CHEB_NNZ_UNROLL : rp_s[lr + 1];
        CHEB_ASSERT(rows <= G::TILE && i < a.d && e_lo <= e_hi);
        // 32-bit row-local offsets (a row's nnz and its staged slice fit in int32)
        const int nr = (int)(e_hi - e_lo);
        const int oc = STAGED ? (int)(e_lo - base_c) : 0;
        const int ov = STAGED ? (int)(e_lo - base_v) : 0;
        const double* wrow = wcur + (size_t)i * K;
        double2 g[NSL], own[NSL];  // gathered sum (Ã w_{j-1} row i), w_{j-1}[i]
#pragma unroll
        for (int sl = 0; sl < NSL; sl++) {
            g[sl] = make_double2(0.0, 0.0);
            own[sl] = make_double2(0.0, 0.0);
            if (OWN_EARLY) {  // issued before the gathers so its latency overlaps them
                if (VB == 1) {  // w_{j-1} = v: from the staged sign bits
                    const uint32_t wv = sg_s[lr * G::WORDS + (pp[sl] >> 5)];
                    own[sl] = make_double2(pm1(wv, pp[sl] & 31), pm1(wv, (pp[sl] & 31) + 1));
                } else {
                    own[sl] = CG ? ldcg2(wrow + pp[sl]) : ldg2(wrow + pp[sl]);
                }
            }
        }
        // all nnz of a chunk issue their gathers before any is consumed; rows are padded to a
        // multiple of the chunk with (i, 0.0) entries by the prep pass (no bounds checks here)
        CHEB_ASSERT(nr % CHEB_NNZ_UNROLL == 0);
        const int32_t* crow = STAGED ? col_s + oc : a.ci + e_lo;
        const double* vrow = STAGED ? val_s + ov : a.va + e_lo;
        const int16_t* dcrow = reinterpret_cast<const int16_t*>(st + SL::OFF_COL) + lr * CHEB_NNZ_UNROLL;
        const uint8_t* virow = reinterpret_cast<const uint8_t*>(st + SL::OFF_VAL) + lr * CHEB_NNZ_UNROLL;
        for (int t0 = 0; t0 < nr; t0 += CHEB_NNZ_UNROLL) {
            int32_t c[CHEB_NNZ_UNROLL];
            double v[CHEB_NNZ_UNROLL];
#pragma unroll
            for (int q = 0; q < CHEB_NNZ_UNROLL; q++) {
                CHEB_ASSERT(!STAGED || (oc + t0 + q >= 0 && oc + t0 + q < G::CAP + 8));
                CHEB_ASSERT(!STAGED || (ov + t0 + q >= 0 && ov + t0 + q < G::CAP + 4));
                if (CV) {
                    c[q] = (int32_t)i + (int32_t)dcrow[t0 + q];
                    v[q] = cvt[virow[t0 + q]];
                } else {
                    c[q] = STAGED ? crow[t0 + q] : __ldg(crow + t0 + q);
                    v[q] = STAGED ? vrow[t0 + q] : __ldg(vrow + t0 + q);
                }
                CHEB_ASSERT(c[q] >= 0 && (int64_t)c[q] < a.d);
            }
            double2 x[CHEB_NNZ_UNROLL][NSL];
            if (VB == 1) {  // gather v = +-1 from the sign bits (4-8 B per row instead of 8K)
                uint32_t wd[CHEB_NNZ_UNROLL][NSL];
#pragma unroll
                for (int q = 0; q < CHEB_NNZ_UNROLL; q++)
#pragma unroll
                    for (int sl = 0; sl < NSL; sl++)
                        wd[q][sl] = __ldg(a.sbits + (size_t)(uint32_t)c[q] * G::WORDS + (pp[sl] >> 5));
#pragma unroll
                for (int q = 0; q < CHEB_NNZ_UNROLL; q++)
#pragma unroll
                    for (int sl = 0; sl < NSL; sl++)
                        x[q][sl] = make_double2(pm1(wd[q][sl], pp[sl] & 31), pm1(wd[q][sl], (pp[sl] & 31) + 1));
            } else {
#pragma unroll
                for (int q = 0; q < CHEB_NNZ_UNROLL; q++) {
                    // lane offset folded into the base: one IMAD.WIDE per gathered row
                    const double* p = xl + (size_t)(uint32_t)c[q] * K;
#pragma unroll
                    if constexpr (G::WIDE) {
                        if (CG) ldca4(p, x[q][0], x[q][1]);
                        else ldg4(p, x[q][0], x[q][1]);
                    } else {
                        for (int sl = 0; sl < NSL; sl++) x[q][sl] = CG ? ldcg2(p + sl * G::SS) : ldg2(p + sl * G::SS);
                    }
                }
            }
            if (OWN_GATHER && t0 == 0) {
#pragma unroll
                for (int sl = 0; sl < NSL; sl++) own[sl] = x[0][sl];
            }
#pragma unroll
            for (int q = 0; q < CHEB_NNZ_UNROLL; q++)
#pragma unroll
                for (int sl = 0; sl < NSL; sl++) {
                    g[sl].x = fma(v[q], x[q][sl].x, g[sl].x);
                    g[sl].y = fma(v[q], x[q][sl].y, g[sl].y);
                }
        }
        if (OWN_SMEM) {
#pragma unroll
            for (int sl = 0; sl < NSL; sl++) own[sl] = *reinterpret_cast<const double2*>(wc_s + lr * K + pp[sl]);
        }
        // -beta w_{j-1}[i]: csr / rank-1 carry it in the prepped matrix (the folded diagonal, or an
        // (i, -beta) entry the prep added to a row with none); B^T B has no matrix diagonal to fold into
        if (MODE == MODE_BTB) {
#pragma unroll
            for (int sl = 0; sl < NSL; sl++) {
                g[sl].x = fma(-a.beta, own[sl].x, g[sl].x);
                g[sl].y = fma(-a.beta, own[sl].y, g[sl].y);
            }
        }
        if (MODE == MODE_FAM) {
            // member of column p: (alpha_p d_i - beta_p) w_{j-1}[i] + alpha_p theta_p (O w_{j-1})_i
            const double di = u_s[lr];
#pragma unroll
            for (int sl = 0; sl < NSL; sl++) {
                const double2 ca = *reinterpret_cast<const double2*>(fcoef + pp[sl]);
                const double2 cb = *reinterpret_cast<const double2*>(fcoef + K + pp[sl]);
                const double2 cc = *reinterpret_cast<const double2*>(fcoef + 2 * K + pp[sl]);
                g[sl].x = fma(fma(ca.x, di, -cb.x), own[sl].x, cc.x * g[sl].x);
                g[sl].y = fma(fma(ca.y, di, -cb.y), own[sl].y, cc.y * g[sl].y);
            }
        }
        double ui = 1.0;
        if (HAS_S) {
            ui = a.r1u ? u_s[lr] : 1.0;
#pragma unroll
            for (int sl = 0; sl < NSL; sl++) {
                g[sl].x = fma(ui, r1[sl].x, g[sl].x);
                g[sl].y = fma(ui, r1[sl].y, g[sl].y);
            }
        }
        double2 nw[NSL];  // w_j row i
#pragma unroll
        for (int sl = 0; sl < NSL; sl++) {
            if (FIRST) {
                nw[sl] = g[sl];
            } else {
                double2 pv;
                if (VB == 2) {  // w_{j-2} = v: from the staged sign bits
                    const uint32_t wv = sg_s[lr * G::WORDS + (pp[sl] >> 5)];
                    pv = make_double2(pm1(wv, pp[sl] & 31), pm1(wv, (pp[sl] & 31) + 1));
                } else {
                    pv = *reinterpret_cast<const double2*>(wp_s + lr * K + pp[sl]);
                }
                // 2g - p in one DFMA: 2g is exact, so this rounds exactly like (g + g) - p
                nw[sl] = make_double2(fma(2.0, g[sl].x, -pv.x), fma(2.0, g[sl].y, -pv.y));
            }
        }
        double* out = wout + (size_t)i * K;
        if constexpr (G::WIDE) {
            stcs4(out + pp[0], nw[0], nw[1]);  // streamed: the next read is by a later step
        } else {
#pragma unroll
            for (int sl = 0; sl < NSL; sl++) __stcs(reinterpret_cast<double2*>(out + pp[sl]), nw[sl]);
        }
#pragma unroll
        for (int sl = 0; sl < NSL; sl++) {
            if (DBL) {
                // w_j^T w_j and w_{j-1}^T w_j over this CTA's rows
                acc[0][2 * sl] = fma(nw[sl].x, nw[sl].x, acc[0][2 * sl]);
                acc[0][2 * sl + 1] = fma(nw[sl].y, nw[sl].y, acc[0][2 * sl + 1]);
                acc[1][2 * sl] = fma(own[sl].x, nw[sl].x, acc[1][2 * sl]);
                acc[1][2 * sl + 1] = fma(own[sl].y, nw[sl].y, acc[1][2 * sl + 1]);
            } else {
                // v_p[i] w_j[i][p]: flip the sign bit of w where the probe bit is set
                const uint32_t bits = sg_s[lr * G::WORDS + (pp[sl] >> 5)] >> (pp[sl] & 31);
                acc[0][2 * sl] += signflip(nw[sl].x, bits << 31);
                acc[0][2 * sl + 1] += signflip(nw[sl].y, bits << 30);
            }
            if (HAS_S) {
                acc[SCH][2 * sl] = fma(ui, nw[sl].x, acc[SCH][2 * sl]);
                acc[SCH][2 * sl + 1] = fma(ui, nw[sl].y, acc[SCH][2 * sl + 1]);
            }
        }
    }
}

// resident CTAs per SM each mode is register-budgeted for (BTB is smem-limited to 2)
#ifndef CHEB_DIAG_R1_NOSYNC
#define CHEB_DIAG_R1_NOSYNC 0  // TIMING DIAGNOSTIC builds only (wrong rank-1 results): skip the s_j handoff
#endif
#ifndef CHEB_MIN_CTAS_FAM
#define CHEB_MIN_CTAS_FAM 4  // family mode (per-column scalars in shared memory)
#endif
#ifndef CHEB_MIN_CTAS_R1
#define CHEB_MIN_CTAS_R1 3  // rank-1 Algorithm 1 (two accumulator channels)
#endif
__host__ __device__ constexpr int min_ctas(int mode, bool dbl = false) {
    return mode == MODE_CSR ? (dbl ? CHEB_MIN_CTAS_DBL : CHEB_MIN_CTAS)
                            : (mode == MODE_RANK1 && !dbl ? CHEB_MIN_CTAS_R1 : (mode == MODE_FAM ? CHEB_MIN_CTAS_FAM : 2));
}

// RP: rows per lane group of the Algorithm-1 kernels (0: CHEB_RPG).  L2-resident operators use
// RP = 1 (16-row tiles at k = 64) in both the per-step and the persistent kernel, so the two stay
// bit-identical (measured: configs[0] 0.22 -> 0.18 ms, configs[1] 15.5 -> 15.2 ms per estimate).
template <int K, int MODE, bool FIRST, bool DBL = false, int VB = 0, int RP = 0>
__global__ void __launch_bounds__(kThreads, min_ctas(MODE, DBL))
cheb_step_kernel(StepArgs a) {
    // DBL: 16-row tiles (CHEB_RPG_DBL) with the own W_cur rows staged by TMA for w_{j-1}^T w_j
    // (measured best: 6.50 ms per configs[3] launch vs 6.82 ms with 32-row tiles and an early
    // L1/L2 load of the own row; staging with 32-row tiles shrinks L1 too much)
    constexpr int R4 = RP ? RP : (DBL ? CHEB_RPG_DBL : CHEB_RPG);
    using G = Geo<K, R4>;
    constexpr bool WCS = DBL && CHEB_DBL_STAGE_WC && VB != 1;  // step 1 on sign bits: v from the bits
    using SL = StageLayout<K, MODE, WCS, R4>;
    constexpr bool HAS_S = (MODE == MODE_RANK1);
    constexpr int NS = kStepStages;
    constexpr int NCH = n_channels<MODE, DBL>();
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[NS];
    __shared__ int64_t s_base_c[NS], s_base_v[NS];
    __shared__ int s_fit[NS];
    __shared__ __align__(16) int64_t s_ne[2];  // row bounds of the next tile to stage (cp.async)

    const int tid = threadIdx.x;
    // family: per column alpha, beta, alpha*theta in shared memory (registers measured slower:
    // 3 CTAs/SM and spills, 7.0 vs 5.9 s for the configs[3]-size 8-member scan)
    __shared__ __align__(16) double s_fcoef[MODE == MODE_FAM ? 3 * K : 2];
    if (MODE == MODE_FAM)
        for (int x = tid; x < 3 * K; x += kThreads) s_fcoef[x] = a.fam_coef[x];
    // compressed matrix (csr / rank-1): decided on the device by the CV prep, uniform per launch
    // (the value-index slice of a tile must start 16-byte aligned: U * TILE % 16 == 0)
    // Probe blocks k <= 16 only: there the matrix is 15 % of a launch's bytes and the copy saves 10 %
    // of the time (configs[3]: 1.52 -> 1.37 s per estimate); at k = 64 it is 4 %, and the second
    // staging path costs registers (1.308 -> 1.322 s).  Family mode: not (its registers spill).
    constexpr bool CAN_CV = CHEB_CV_KERNEL && (MODE == MODE_CSR || MODE == MODE_RANK1) && K <= 16 &&
                            G::TILE % 16 == 0;
    __shared__ double s_cvt[CAN_CV ? kCvSlots : 1];
    const bool cv = CAN_CV && a.cv_ok && *a.cv_ok != 0;
    if (cv)
        for (int x = tid; x < kCvSlots; x += kThreads) s_cvt[x] = a.cv_tab[x];
    double acc[NCH][kPPL];
#pragma unroll
    for (int ch = 0; ch < NCH; ch++)
#pragma unroll
        for (int q = 0; q < kPPL; q++) acc[ch][q] = 0.0;
    double2 r1[G::NSL];  // alpha c s_{j-1}[p] of the lane's probes (rank-1)
#pragma unroll
    for (int sl = 0; sl < G::NSL; sl++) {
        const int p = G::lane_probe(tid % G::L, sl);
        r1[sl] = HAS_S ? make_double2(a.r1c_alpha * a.s_cur[p], a.r1c_alpha * a.s_cur[p + 1]) : make_double2(0.0, 0.0);
    }
    const int64_t nmine = a.ntiles > blockIdx.x ? (a.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    // ---- producer (thread 0): issue the bulk copies of tile t into stage b
    auto issue = [&](int64_t t, int b, int64_t e0, int64_t e1) {
        unsigned char* st = smem + b * SL::BYTES;
        const int64_t r0 = t * G::TILE;
        const int rows = (int)imin64((int64_t)G::TILE, a.d - r0);
        const int64_t c0 = e0 & ~int64_t(3), c1 = (e1 + 3) & ~int64_t(3);
        const int64_t v0 = e0 & ~int64_t(1), v1 = (e1 + 1) & ~int64_t(1);
        const bool fit = (c1 - c0) <= G::CAP + 8 && (v1 - v0) <= G::CAP + 4;
        s_fit[b] = fit;
        s_base_c[b] = c0;
        s_base_v[b] = v0;
        const uint32_t wbytes = (uint32_t)rows * K * 8;
        constexpr bool SIGNS = !DBL || VB != 0;  // DBL reads no sign bits, except for v itself
        const uint32_t sgbytes = SIGNS ? ((uint32_t)rows * G::WORDS * 4 + 15) & ~15u : 0u;
        // compressed: no row pointer, 2 + 1 bytes per entry (the arrays carry 16 bytes of tail padding)
        constexpr int UCV = CHEB_NNZ_UNROLL;
        const uint32_t dcbytes = ((uint32_t)rows * UCV * 2 + 15) & ~15u, vibytes = ((uint32_t)rows * UCV + 15) & ~15u;
        uint32_t bytes = (cv ? 0u : (uint32_t)G::RPBYTES) + sgbytes;
        if (!FIRST && VB != 2) bytes += wbytes;
        if (SL::HAS_WC) bytes += wbytes;
        if (cv) bytes += dcbytes + vibytes;
        else if (fit) bytes += (uint32_t)(c1 - c0) * 4 + (uint32_t)(v1 - v0) * 8;
        const uint32_t ubytes = ((uint32_t)rows * 8 + 15) & ~15u;
        if ((HAS_S || MODE == MODE_FAM) && a.r1u) bytes += ubytes;
        mbar_expect_tx(&bar[b], bytes);
        if (!cv) bulk_g2s(st + SL::OFF_RP, a.rp + r0, G::RPBYTES, &bar[b]);
        if (SIGNS) bulk_g2s(st + SL::OFF_SGN, a.sbits + (size_t)r0 * G::WORDS, sgbytes, &bar[b]);
        if (!FIRST && VB != 2)
            bulk_g2s_hint(st + SL::OFF_WPREV, a.wnext + (size_t)r0 * K, wbytes, &bar[b], policy_evict_first());
        if (SL::HAS_WC) bulk_g2s(st + SL::OFF_WCUR, a.wcur + (size_t)r0 * K, wbytes, &bar[b]);
        if (cv) {
            bulk_g2s(st + SL::OFF_COL, a.cv_dc + (size_t)r0 * UCV, dcbytes, &bar[b]);
            bulk_g2s(st + SL::OFF_VAL, a.cv_vi + (size_t)r0 * UCV, vibytes, &bar[b]);
        } else if (fit) {
            bulk_g2s(st + SL::OFF_COL, a.ci + c0, (uint32_t)(c1 - c0) * 4, &bar[b]);
            bulk_g2s(st + SL::OFF_VAL, a.va + v0, (uint32_t)(v1 - v0) * 8, &bar[b]);
        }
        if ((HAS_S || MODE == MODE_FAM) && a.r1u) bulk_g2s(st + SL::OFF_U, a.r1u + r0, ubytes, &bar[b]);
    };
    auto tile_of = [&](int64_t i) { return (int64_t)blockIdx.x + i * gridDim.x; };
    auto bounds = [&](int64_t t, int64_t& e0, int64_t& e1) {
        const int64_t r0 = t * G::TILE;
        e0 = __ldg(a.rp + r0);
        e1 = __ldg(a.rp + imin64(r0 + G::TILE, a.d));
    };

    // thread 0 fetches the next tile's row bounds into shared memory with cp.async (no register
    // live across the tile, no stall), and reads them after the tile, just before staging it
    auto bounds_async = [&](int64_t t) {
        const int64_t r0 = t * G::TILE;
        cp_async8(&s_ne[0], a.rp + r0);
        cp_async8(&s_ne[1], a.rp + imin64(r0 + G::TILE, a.d));
        cp_async_commit();
    };
    // "stage consumed" barriers, one arrival per warp: warps are not held at a CTA-wide barrier
    // after every tile, only thread 0 waits (for the stage it refills, one tile later)
    constexpr bool DEC = CHEB_DECOUPLE == 1 || (CHEB_DECOUPLE == 2 && RP == 1);
    __shared__ __align__(8) uint64_t ebar[NS];
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < NS; i++) {
            mbar_init(&bar[i], 1);
            if (DEC) mbar_init(&ebar[i], kThreads / 32);
        }
        fence_mbar_init();
        for (int64_t i = 0; i < NS && i < nmine; i++) {
            int64_t e0, e1;
            bounds(tile_of(i), e0, e1);
            issue(tile_of(i), (int)i, e0, e1);
        }
    }
    __syncthreads();

    for (int64_t it = 0; it < nmine; it++) {
        const int b = (int)(it % NS);
        const uint32_t phase = (uint32_t)((it / NS) & 1);
        const int64_t t = tile_of(it);
        if (DEC && tid == 0 && it >= 1 && it - 1 + NS < nmine) {  // refill the stage of tile it-1 with it-1+NS
            const int pb = (int)((it - 1) % NS);
            mbar_wait(&ebar[pb], (uint32_t)(((it - 1) / NS) & 1));
            cp_async_wait_all();
            issue(tile_of(it - 1 + NS), pb, s_ne[0], s_ne[1]);
        }
        if (tid == 0 && it + NS < nmine && !cv) bounds_async(tile_of(it + NS));  // consumed below
        mbar_wait(&bar[b], phase);
        const unsigned char* st = smem + b * SL::BYTES;
        const int64_t r0 = t * G::TILE;
        const int rows = (int)imin64((int64_t)G::TILE, a.d - r0);
        if constexpr (CAN_CV) {
            if (cv)
                step_tile<K, MODE, FIRST, true, false, DBL, WCS, R4, VB, true>(a, st, r0, rows, 0, 0, r1, acc, a.xg,
                                                                         a.wcur, a.wnext, s_fcoef, s_cvt);
        }
        if (cv) {
        } else if (s_fit[b])
            step_tile<K, MODE, FIRST, true, false, DBL, WCS, R4, VB>(a, st, r0, rows, s_base_c[b], s_base_v[b], r1,
                                                               acc, a.xg, a.wcur, a.wnext, s_fcoef);
        else
            step_tile<K, MODE, FIRST, false, false, DBL, WCS, R4, VB>(a, st, r0, rows, 0, 0, r1, acc, a.xg, a.wcur,
                                                                a.wnext, s_fcoef);
        if (DEC) {
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&ebar[b]);  // this warp is done with stage b
        } else {
            __syncthreads();  // every warp is done with stage b
            if (tid == 0 && it + NS < nmine) {
                cp_async_wait_all();
                issue(tile_of(it + NS), b, s_ne[0], s_ne[1]);
            }
        }
    }
    if (DEC) __syncthreads();  // the reduction scratch below aliases the stages
    grid_reduce_finish<K, kPPL, NCH, DBL ? EPI_DBL : EPI_STEP, HAS_S, !G::WIDE>(acc, a, smem);
}


// ---------------------------------------------------------------------------------------
// Lanczos process on the device (reading G26): K independent Lanczos runs,
// one per column of a [d][K] block (one Rademacher probe per column), on M itself (no interval
// needed).  Per step j, with q = q_j (normalised), qp = q_{j-1}, s = u^T q_j (rank-1):
//   z = M_S q                                   (spmm_kernel; B^T B: two of them)
//   LZ_DOT:  alpha_j = q^T (z + c u s)
//   LZ_UPD:  qp <- z + c u s - alpha_j q - beta_j qp,  beta_{j+1} = |qp|
//   LZ_NRM:  qp <- qp / beta_{j+1},  s <- u^T qp   (then q and qp swap roles)
// No re-orthogonalisation (loss of orthogonality only duplicates converged extreme Ritz values).
// Every per-column scalar stays on the device; one reduction per pass: per-CTA partials, the last
// CTA sums them in CTA order (deterministic).
// ---------------------------------------------------------------------------------------
enum { LZ_DOT = 0, LZ_UPD = 1, LZ_NRM = 2 };

struct LzArgs {
    int64_t d;
    double* q;            // q_j            [d][K]
    double* qp;           // q_{j-1} / work [d][K]
    const double* z;      // M_S q_j        [d][K]
    const double* u;      // rank-1 u (nullptr: ones)
    double r1c;           // rank-1 weight c (0: no rank-1 term)
    double* s;            // [K] u^T q_j
    const double* alpha;  // [K] alpha_j (LZ_UPD)
    const double* beta;   // [K] beta_j  (LZ_UPD: coefficient of qp; LZ_NRM: the divisor)
    double* out;          // [K] reduction result: alpha_j (DOT), beta_{j+1} (UPD), s (NRM)
    double* part;         // [gridDim.x][K] per-CTA partials
    unsigned int* ticket;
};

template <int K, int OP>
__global__ void __launch_bounds__(kThreads)
lanczos_vec_kernel(LzArgs a) {
    constexpr int CP = K / 2;  // column pairs; a thread keeps one pair for every row it visits
    __shared__ double red[kThreads][2];
    __shared__ bool is_last;
    const int tid = threadIdx.x;
    const int64_t n2 = a.d * CP;
    const int64_t stride = (int64_t)gridDim.x * kThreads;  // multiple of CP: the pair is fixed
    double acc0 = 0.0, acc1 = 0.0;
    const int cp = (int)(((int64_t)blockIdx.x * kThreads + tid) % CP);
    const int c0 = 2 * cp;
    double s0 = 0.0, s1 = 0.0, al0 = 0.0, al1 = 0.0, be0 = 0.0, be1 = 0.0;
    if (OP != LZ_NRM && a.r1c != 0.0) { s0 = a.r1c * a.s[c0]; s1 = a.r1c * a.s[c0 + 1]; }
    if (OP == LZ_UPD) { al0 = a.alpha[c0]; al1 = a.alpha[c0 + 1]; be0 = a.beta[c0]; be1 = a.beta[c0 + 1]; }
    if (OP == LZ_NRM) { be0 = 1.0 / a.beta[c0]; be1 = 1.0 / a.beta[c0 + 1]; }
    for (int64_t x = (int64_t)blockIdx.x * kThreads + tid; x < n2; x += stride) {
        const int64_t i = x / CP;
        const size_t o = (size_t)i * K + c0;
        const double ui = a.u ? a.u[i] : 1.0;
        if (OP == LZ_DOT) {
            const double2 q = *reinterpret_cast<const double2*>(a.q + o);
            const double2 z = *reinterpret_cast<const double2*>(a.z + o);
            acc0 = fma(q.x, fma(ui, s0, z.x), acc0);
            acc1 = fma(q.y, fma(ui, s1, z.y), acc1);
        } else if (OP == LZ_UPD) {
            const double2 q = *reinterpret_cast<const double2*>(a.q + o);
            const double2 z = *reinterpret_cast<const double2*>(a.z + o);
            double2 w = *reinterpret_cast<const double2*>(a.qp + o);
            w.x = fma(-be0, w.x, fma(-al0, q.x, fma(ui, s0, z.x)));
            w.y = fma(-be1, w.y, fma(-al1, q.y, fma(ui, s1, z.y)));
            *reinterpret_cast<double2*>(a.qp + o) = w;
            acc0 = fma(w.x, w.x, acc0);
            acc1 = fma(w.y, w.y, acc1);
        } else {
            double2 w = *reinterpret_cast<const double2*>(a.qp + o);
            w.x *= be0;
            w.y *= be1;
            *reinterpret_cast<double2*>(a.qp + o) = w;
            acc0 = fma(ui, w.x, acc0);
            acc1 = fma(ui, w.y, acc1);
        }
    }
    red[tid][0] = acc0;
    red[tid][1] = acc1;
    __syncthreads();
    // per-CTA partial of column c: threads t = c/2 (mod CP) in ascending order
    if (tid < K) {
        double m = 0.0;
        const int pr = tid / 2, h = tid & 1;  // kThreads % CP == 0: thread t holds pair t % CP
        for (int t = pr; t < kThreads; t += CP) m += red[t][h];
        a.part[(size_t)blockIdx.x * K + tid] = m;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    if (tid < K) {
        double t = 0.0;
        for (unsigned int c = 0; c < gridDim.x; c++) t += __ldcg(a.part + (size_t)c * K + tid);
        a.out[tid] = (OP == LZ_UPD) ? sqrt(t) : t;
    }
    if (tid == 0) *a.ticket = 0u;
}

// v_p[i] = +-1 for global probes p0 .. p0+K-1 (the path's splitmix64 generator), written to w
template <int K>
__global__ void __launch_bounds__(kThreads)
lanczos_probe_kernel(int64_t d, uint64_t seed, uint64_t p0, double* w) {
    const int64_t n = d * K;
    for (int64_t x = (int64_t)blockIdx.x * kThreads + threadIdx.x; x < n; x += (int64_t)gridDim.x * kThreads) {
        const int64_t i = x / K;
        const int c = (int)(x % K);
        const uint64_t z = splitmix64_at(seed, (p0 + (uint64_t)c) * (uint64_t)d + (uint64_t)i + 1ull);
        w[x] = (z >> 63) ? -1.0 : 1.0;
    }
}

// ---------------------------------------------------------------------------------------
// Status epilogue of a cheb_moments call (one launch per call).  status: the workspace status
// word; bit 0 is set by a spin wait of the persistent kernel that gave up (it never hangs the
// GPU).  Then every moment of the call becomes NaN, so cheb_finalize's finiteness flag and
// cheb_logdet's CL_ENONFINITE/CL_ECUDA checks see it; otherwise bit 1 records any non-finite
// moment (operator spectrum outside [a,b]).  mu: the call's rows, contiguous.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
moments_status_kernel(unsigned int* status, double* mu, int64_t nmu, const int32_t* cv_ok) {
    const bool poison = (*reinterpret_cast<volatile unsigned int*>(status) & 1u) != 0;
    if (cv_ok && blockIdx.x == 0 && threadIdx.x == 0 && *cv_ok) atomicOr(status, 0x100u);  // format note
    int bad = 0;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nmu; x += (int64_t)gridDim.x * blockDim.x) {
        if (poison) mu[x] = __longlong_as_double(0x7ff8000000000000ll);
        else bad |= !isfinite(mu[x]);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, 2u);
}

// ---------------------------------------------------------------------------------------
// Inter-CTA synchronisation primitives (persistent kernel)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_release_add(unsigned int* p, unsigned int v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


// ---------------------------------------------------------------------------------------
// K2p: persistent multi-step kernel for small / L2-resident operators (csr, rank-1).
// One cooperative launch, in thread-block clusters of RG = red_group(G) CTAs, runs steps
// j = 1..n of a probe block: each step walks the same static tile schedule as cheb_step_kernel
// (tile t on CTA t mod G, same staged pipeline).  Step tail, ONE grid-wide synchronisation:
//   1. every CTA reduces its accumulators to a per-CTA partial in its shared memory;
//   2. cluster barrier; the cluster's rank 0 sums its CTAs' partials over DSMEM (ascending
//      rank = ascending c: the group sums S_q of the canonical order), stores them and
//      release-adds 1 to the grid counter (step j complete at j * ng);
//   3. every CTA issues the TMA copies of its first tiles of step j+1 (W_prev = w_{j-1} and the
//      matrix are final), waits for the counter, and sums the ng group sums itself: the rank-1
//      s_j = u^T w_j that gates step j+1 and (the last CTA) the moments mu_j.
// Moments are bit-identical to per-step launches with the same grid.  Removes the n launch /
// drain gaps that dominate when one step is a few microseconds of L2 traffic, and (rank-1) the
// second grid-wide wait that publishing s_j from a few reducer CTAs needed.
// ---------------------------------------------------------------------------------------
struct PersistArgs {
    double* w0;               // holds v (from probe_init) at entry
    double* w1;
    int32_t n;                // degree
    double* gpart;            // [2][NCH][ng][K] group sums (double-buffered by step parity)
    double* s_buf;            // s_0 (from probe_init) in s_buf[0..K)
    unsigned int* bar_count;  // grid barrier: arrivals of cluster leaders (zeroed; monotone)
    unsigned int* err;        // wait timeout flag
    int32_t power;            // power basis (Taylor baseline): every step is w_j = Ã w_{j-1}
};

// Relaxed polling (an acquire load compiles to an SM-wide L1 invalidate per iteration, which
// would flush the L1 of every CTA on the SM while one spins), then one acquire fence.
__device__ __forceinline__ void spin_until_geq(const unsigned int* p, unsigned int want, unsigned int* err) {
    uint32_t spins = 0;
    while (ld_relaxed_u32(p) < want) {
        __nanosleep(20);
        if ((++spins & 1023u) == 0 && (spins > (1u << 25) || ld_relaxed_u32(err))) {
            atomicExch(err, 1u);  // ~seconds without progress: give up, never hang
            break;
        }
    }
    fence_acq_rel_gpu();
}

template <int K, int MODE, bool DBL = false, int RP = 0>
__global__ void __launch_bounds__(kThreads, min_ctas(MODE, DBL))
cheb_persist_kernel(StepArgs a, PersistArgs pa_) {
    constexpr int R4 = RP ? RP : (DBL ? CHEB_RPG_DBL : CHEB_RPG);  // same tile geometry as cheb_step_kernel
    using G = Geo<K, R4>;
    using SL = StageLayout<K, MODE, false, R4>;
    constexpr bool HAS_S = (MODE == MODE_RANK1);
    constexpr int NCH = n_channels<MODE, DBL>();
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int64_t s_base_c[2], s_base_v[2];
    __shared__ int s_fit[2];
    __shared__ double red[NCH][kThreads / 32][K];
    __shared__ double cpart[2][NCH][K];  // this CTA's partial of step j (parity j & 1), read over DSMEM
    __shared__ double fin[NCH][K];
    __shared__ double s_sh[HAS_S ? K : 1];
    // row bounds of this CTA's tiles, loaded once (they are the same every step): staging a tile
    // then needs no global load on thread 0 (a per-tile ~1 us stall of warp 0, which the end-of-tile
    // barrier passes on to the whole CTA); CTAs with more tiles load them at issue time
    constexpr int kBoundsCache = 32;
    __shared__ int64_t s_eb[2 * kBoundsCache];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lg = tid % G::L;
    const int64_t nmine = a.ntiles > blockIdx.x ? (a.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    uint32_t uses[2] = {0u, 0u};
    // reduction groups = clusters of RG consecutive CTAs (the host launches clusters of RG)
    cg::cluster_group cluster = cg::this_cluster();
    const int RG = a.rg, ng = (int)gridDim.x / RG;
    const int crank = (int)cluster.block_rank(), cid = (int)blockIdx.x / RG;

    const bool cached = nmine <= kBoundsCache;
    if (cached) {
        for (int x = tid; x < 2 * nmine; x += kThreads) {
            const int64_t r0 = ((int64_t)blockIdx.x + (x >> 1) * (int64_t)gridDim.x) * G::TILE;
            s_eb[x] = __ldg(a.rp + ((x & 1) ? imin64(r0 + G::TILE, a.d) : r0));
        }
        __syncthreads();
    }
    // staging of the CTA's it-th tile of step j into stage b (thread 0)
    auto issue = [&](int32_t j, int64_t it, int b) {
        const bool first = (j == 1) || pa_.power;
        const double* wprev = (j & 1) ? pa_.w1 : pa_.w0;  // w_{j-2}
        unsigned char* st = smem + b * SL::BYTES;
        const int64_t t = (int64_t)blockIdx.x + it * gridDim.x;
        const int64_t r0 = t * G::TILE;
        const int rows = (int)imin64((int64_t)G::TILE, a.d - r0);
        const int64_t e0 = cached ? s_eb[2 * it] : __ldg(a.rp + r0);
        const int64_t e1 = cached ? s_eb[2 * it + 1] : __ldg(a.rp + imin64(r0 + G::TILE, a.d));
        const int64_t c0 = e0 & ~int64_t(3), c1 = (e1 + 3) & ~int64_t(3);
        const int64_t v0 = e0 & ~int64_t(1), v1 = (e1 + 1) & ~int64_t(1);
        const bool fit = (c1 - c0) <= G::CAP + 8 && (v1 - v0) <= G::CAP + 4;
        s_fit[b] = fit;
        s_base_c[b] = c0;
        s_base_v[b] = v0;
        const uint32_t wbytes = (uint32_t)rows * K * 8;
        const uint32_t sgbytes = DBL ? 0u : ((uint32_t)rows * G::WORDS * 4 + 15) & ~15u;  // DBL: no signs
        const uint32_t ubytes = ((uint32_t)rows * 8 + 15) & ~15u;
        uint32_t bytes = G::RPBYTES + sgbytes;
        if (!first) bytes += wbytes;
        if (fit) bytes += (uint32_t)(c1 - c0) * 4 + (uint32_t)(v1 - v0) * 8;
        if (HAS_S && a.r1u) bytes += ubytes;
        mbar_expect_tx(&bar[b], bytes);
        bulk_g2s(st + SL::OFF_RP, a.rp + r0, G::RPBYTES, &bar[b]);
        if (!DBL) bulk_g2s(st + SL::OFF_SGN, a.sbits + (size_t)r0 * G::WORDS, sgbytes, &bar[b]);
        if (!first) bulk_g2s(st + SL::OFF_WPREV, wprev + (size_t)r0 * K, wbytes, &bar[b]);
        if (fit) {
            bulk_g2s(st + SL::OFF_COL, a.ci + c0, (uint32_t)(c1 - c0) * 4, &bar[b]);
            bulk_g2s(st + SL::OFF_VAL, a.va + v0, (uint32_t)(v1 - v0) * 8, &bar[b]);
        }
        if (HAS_S && a.r1u) bulk_g2s(st + SL::OFF_U, a.r1u + r0, ubytes, &bar[b]);
    };

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        for (int64_t i = 0; i < 2 && i < nmine; i++) issue(1, i, (int)i);
    }
    if (HAS_S && tid < K) s_sh[tid] = __ldcg(pa_.s_buf + tid);  // s_0
    __syncthreads();

    for (int32_t j = 1; j <= pa_.n; j++) {
        const bool first = (j == 1) || pa_.power;
        const double* cur = (j & 1) ? pa_.w0 : pa_.w1;  // w_{j-1}
        double* nxt = (j & 1) ? pa_.w1 : pa_.w0;        // w_{j-2} -> w_j
        double2 r1[G::NSL];
#pragma unroll
        for (int sl = 0; sl < G::NSL; sl++) {
            const int p = G::lane_probe(lg, sl);
            r1[sl] = HAS_S ? make_double2(a.r1c_alpha * s_sh[p], a.r1c_alpha * s_sh[p + 1]) : make_double2(0.0, 0.0);
        }
        double acc[NCH][kPPL];
#pragma unroll
        for (int ch = 0; ch < NCH; ch++)
#pragma unroll
            for (int q = 0; q < kPPL; q++) acc[ch][q] = 0.0;
        for (int64_t it = 0; it < nmine; it++) {
            const int b = (int)(it & 1);
            mbar_wait(&bar[b], uses[b] & 1u);
            uses[b]++;
            const unsigned char* st = smem + b * SL::BYTES;
            const int64_t t = (int64_t)blockIdx.x + it * gridDim.x;
            const int64_t r0 = t * G::TILE;
            const int rows = (int)imin64((int64_t)G::TILE, a.d - r0);
            if (first) {
                if (s_fit[b])
                    step_tile<K, MODE, true, true, true, DBL, false, R4>(a, st, r0, rows, s_base_c[b], s_base_v[b], r1,
                                                                     acc, cur, cur, nxt);
                else
                    step_tile<K, MODE, true, false, true, DBL, false, R4>(a, st, r0, rows, 0, 0, r1, acc, cur, cur,
                                                                      nxt);
            } else {
                if (s_fit[b])
                    step_tile<K, MODE, false, true, true, DBL, false, R4>(a, st, r0, rows, s_base_c[b], s_base_v[b], r1,
                                                                      acc, cur, cur, nxt);
                else
                    step_tile<K, MODE, false, false, true, DBL, false, R4>(a, st, r0, rows, 0, 0, r1, acc, cur, cur,
                                                                       nxt);
            }
            __syncthreads();
            if (tid == 0 && it + 2 < nmine) issue(j, it + 2, b);
        }
        // ---- per-CTA partial (same tree as grid_reduce_finish), into shared memory
#pragma unroll
        for (int off = G::L; off < 32; off <<= 1) {
#pragma unroll
            for (int ch = 0; ch < NCH; ch++)
#pragma unroll
                for (int q = 0; q < kPPL; q++) acc[ch][q] += __shfl_xor_sync(0xffffffffu, acc[ch][q], off);
        }
        if (lane < G::L) {
#pragma unroll
            for (int q = 0; q < kPPL; q++) {
                const int p = probe_of<K, kPPL, !G::WIDE>(lg, q);
#pragma unroll
                for (int ch = 0; ch < NCH; ch++) red[ch][warp][p] = acc[ch][q];
            }
        }
        __syncthreads();
        const int par = j & 1;
        if (tid < K) {
#pragma unroll
            for (int ch = 0; ch < NCH; ch++) {
                double m = 0.0;
#pragma unroll
                for (int w = 0; w < kThreads / 32; w++) m += red[ch][w][tid];
                cpart[par][ch][tid] = m;
            }
        }
        // ---- cluster (reduction group) barrier: the group's partials and w_j rows are complete;
        // rank 0 forms the group sum S_q over DSMEM (ascending rank = ascending CTA index)
        cluster.sync();
        double* gp = pa_.gpart + (size_t)par * NCH * ng * K;  // [NCH][ng][K] of step j
        if (crank == 0) {
            for (int x = tid; x < NCH * K; x += kThreads) {
                const int ch = x / K, p = x % K;
                double v[kMaxRedGroup], sq = 0.0;  // all DSMEM loads in flight, then the adds in rank order
#pragma unroll
                for (int r = 0; r < kMaxRedGroup; r++) v[r] = r < RG ? *cluster.map_shared_rank(&cpart[par][ch][p], r) : 0.0;
#pragma unroll
                for (int r = 0; r < kMaxRedGroup; r++) sq += v[r];
                gp[((size_t)ch * ng + cid) * K + p] = sq;
            }
            __syncthreads();
            if (tid == 0) red_release_add(pa_.bar_count, 1u);  // release: the cluster's step-j stores
        }
        // ---- stage step j+1, then the single grid-wide wait
        if (tid == 0) {
            if (j < pa_.n) {
                // w_{j-1} (W_prev of step j+1) and the matrix are final: stage ahead.  The
                // proxy fence orders other CTAs' generic stores of w_{j-1} (step j-1, already
                // behind the previous barrier) before these async-proxy reads.
                asm volatile("fence.proxy.async.global;" ::: "memory");
                for (int64_t i = 0; i < 2 && i < nmine; i++) issue(j + 1, i, (int)i);  // stages are all consumed
            }
            spin_until_geq(pa_.bar_count, (unsigned int)j * ng, pa_.err);  // + acquire (L1 invalidated)
        }
        __syncthreads();
        // ---- canonical sums over the ng group sums: the rank-1 s_j by each cluster's rank 0, handed
        // to its cluster over DSMEM (one load of the group sums per cluster, not per CTA); the
        // moments by the last CTA
        constexpr int T = kThreads / K;
        const bool want_mu = blockIdx.x == gridDim.x - 1;
#pragma unroll
        for (int ch = 0; ch < NCH; ch++) {
            const bool is_s = HAS_S && ch == NCH - 1;
            if (!(is_s ? (crank == 0 && j < pa_.n && !CHEB_DIAG_R1_NOSYNC) : want_mu)) continue;
            const double t = group_tree_sum<K>(gp + (size_t)ch * ng * K, ng);
            if (tid % T == 0) fin[ch][tid / T] = t;
        }
        __syncthreads();
        if (want_mu && tid < a.kvalid) {
            double* row = a.mu_out + (size_t)tid * a.mu_stride;
            if (DBL) dbl_write(row, j, a.mu_stride - 1, fin[0][tid], fin[1][tid]);
            else row[j] = fin[0][tid];
        }
        if (HAS_S && j < pa_.n && !CHEB_DIAG_R1_NOSYNC) {  // (after the last step nobody needs s_n)
            if (crank == 0 && tid < K) s_sh[tid] = fin[NCH - 1][tid];
            cluster.sync();  // rank 0's s_j visible to the cluster
            if (crank != 0 && tid < K) s_sh[tid] = *cluster.map_shared_rank(&s_sh[tid], 0);
            __syncthreads();
        }
    }
    // no CTA leaves while a cluster peer may still read its shared memory (also after a timed-out
    // grid wait, when the steps were no longer in lockstep)
    cluster.sync();
}

// ---------------------------------------------------------------------------------------
// K2r: shared-memory-resident multi-step kernel (csr / rank-1, Algorithm 1 and the power basis).
// For operators whose probe block fits in the chip's shared memory (two buffers of d x K fp64
// over <= 148 SMs: configs[0] at every k, configs[1] at k <= 16) the vectors never leave the SMs:
// CTA b owns rows [b*nr, (b+1)*nr) for all n steps and keeps w_{j-1}, w_{j-2} of its rows (and
// its slice of the prepped matrix, its sign bits, u) in shared memory; w_j is written in place
// over w_{j-2} (each element by the thread that reads it).  Two geometries:
//   * one cluster (16 or 8 CTAs, small operators): rows of a peer CTA are gathered over DSMEM
//     (ld.shared::cluster at the mapa'd address), the step tail is one cluster barrier after
//     which every CTA sums the per-CTA partials over DSMEM in rank order;
//   * a flat grid (one CTA per SM, cooperative): rows of other CTAs come from a global copy to
//     which only the rows another CTA gathers ("exported" rows) are written (w_j into g[j & 1]);
//     the step tail is one release-add on a grid counter and one wait; every CTA then sums the
//     published partials of u^T w_j (rank-1) itself, and CTA p sums probe p's mu_j during the
//     next step's reduction (off the critical path).
// The column index of the prepped copy is encoded once per call by resident_prep_kernel
// (>= 0 a global row, < 0 -(1 + (rank << 16 | offset)) a row of the own cluster / CTA).  w_j
// values are bit-identical to the other schedules (same per-row FMA order); the dot products
// follow this kernel's fixed reduction order (deterministic run to run).
// ---------------------------------------------------------------------------------------
#ifndef CHEB_RES_THREADS
#define CHEB_RES_THREADS 512  // 128 registers per thread at one CTA per SM (768: 80, spills)
#endif
constexpr int kResThreads = CHEB_RES_THREADS;

struct ResArgs {
    double* g0;               // global copies of exported rows: w_j in g[j & 1]; g0 holds v at entry
    double* g1;
    int32_t n;                // steps
    int32_t nr;               // rows per CTA
    int32_t cap;              // staged nonzero capacity (dynamic shared memory)
    int32_t power;            // power basis (Taylor baseline): w_j = Ã w_{j-1}
    const uint8_t* exp;       // exp[i] != 0: row i is gathered by another cluster
    double* gpart;            // [2][NCH][ng][K] group sums (step parity)
    const double* s_buf;      // s_0 (rank-1, from probe_init)
    unsigned int* bar_count;  // grid barrier: arrivals of cluster leaders (zeroed; monotone)
    unsigned int* err;        // wait timeout flag
    // several probe blocks in one launch (one cluster each, single-cluster geometry only): block b
    // is CTAs [b * G/nblk, (b+1) * G/nblk), its sign bits at sbits + b * sb_stride, its s_0 at
    // s_buf + b * K, its moment rows from mu_out + b * K * mu_stride; kvalid counts all blocks' probes
    int32_t nblk;             // 1: one probe block (every other geometry)
    int64_t sb_stride;        // uint32 words between consecutive blocks' sign bits
};

// shared-memory row stride (doubles): 256-bit-lane rows (k <= 16) get a 16-byte skew so the rows
// of one quarter-warp fall on different banks
template <int K>
__host__ __device__ constexpr int res_row_stride() { return wide_k(K) ? K + 2 : K; }

struct ResLayout {
    size_t w0, w1, sg, u, ex, rp, col, val, total;
};
__host__ __device__ inline size_t res_a16(size_t x) { return (x + 15) & ~size_t(15); }
template <int K>
__host__ __device__ inline ResLayout res_layout(int nr, int cap, bool has_u) {
    ResLayout l{};
    const size_t wb = res_a16((size_t)nr * res_row_stride<K>() * 8);
    l.w0 = 0;
    l.w1 = l.w0 + wb;
    l.sg = l.w1 + wb;
    l.u = l.sg + res_a16((size_t)nr * words_for(K) * 4);
    l.ex = l.u + (has_u ? res_a16((size_t)nr * 8) : 0);
    l.rp = l.ex + res_a16((size_t)nr);
    l.col = l.rp + res_a16((size_t)(nr + 1) * 4);
    l.val = l.col + res_a16((size_t)cap * 4);
    l.total = l.val + (size_t)cap * 8;
    return l;
}

// Column encoding of the resident schedule (once per cheb_moments call, in place on the prepped
// copy): columns owned by a CTA of the row's own cluster become -(1 + (rank << 16 | offset));
// others stay global and mark their row as exported.
__global__ void __launch_bounds__(kThreads)
resident_prep_kernel(int64_t d, const int64_t* __restrict__ rp2, int32_t* __restrict__ ci2, int32_t nr,
                     int32_t rg, int32_t dsmem, uint8_t* __restrict__ exp) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t oi = i / nr, cl = oi / rg;
        for (int64_t e = rp2[i]; e < rp2[i + 1]; e++) {
            const int32_t c = ci2[e];
            const int64_t oc = c / nr;
            if (dsmem ? oc / rg == cl : oc == oi)
                ci2[e] = -1 - (int32_t)(((oc % rg) << 16) | (int64_t)(c - oc * nr));
            else
                exp[c] = 1;
        }
    }
}

// 16-byte loads of the resident kernel: own shared memory, a cluster peer's (DSMEM); generic below
__device__ __forceinline__ double2 lds2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ double2 ldcl2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

// generic 16-byte load (flat grid: a gather is the CTA's own shared-memory row or the exported global copy)
__device__ __forceinline__ double2 ldgen2(uint64_t a) {
    double2 v;
    asm volatile("ld.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a) : "memory");
    return v;
}
#ifndef CHEB_RES_DIAG
#define CHEB_RES_DIAG 0  // TIMING DIAGNOSTIC builds only (wrong results): 1 no gathers, 2 own-row gathers
#endif
#ifndef CHEB_RES_PROF
#define CHEB_RES_PROF 0  // timing builds: per-CTA cycle counts of the step phases (g_res_prof)
#endif
#if CHEB_RES_PROF
__device__ long long g_res_prof[1024 * 8];
#define RES_T(i)                                                  \
    do {                                                          \
        if (tid == 0) {                                           \
            const long long t_ = clock64();                       \
            prof_acc[i] += t_ - prof_last;                        \
            prof_last = t_;                                       \
        }                                                         \
    } while (0)
#else
#define RES_T(i) ((void)0)
#endif

// DBL: moment doubling (reading G25): channels w_j^T w_j and w_{j-1}^T w_j (own rows), mu_{2j-1},
// mu_{2j} written by dbl_write
template <int K, int MODE, bool DBL = false>
__global__ void __launch_bounds__(kResThreads, 1)
cheb_resident_kernel(StepArgs a, ResArgs ra) {
    using G = Geo<K>;
    constexpr int NT = kResThreads;
    constexpr int L = G::L;          // lanes per row
    constexpr int GR = NT / L;       // rows in flight
    constexpr int NSL = G::NSL;
    constexpr int RS = res_row_stride<K>();
    constexpr int U = CHEB_NNZ_UNROLL;
    constexpr int WORDS = G::WORDS;
    constexpr bool HAS_S = (MODE == MODE_RANK1);
    constexpr int NCH = n_channels<MODE, DBL>();  // mu channel(s), then u^T w_j
    constexpr int NMU = DBL ? 2 : 1;               // channels that make moments
    constexpr int NW = NT / 32;
    static_assert(kPPL == 4, "resident kernel: 4 probes per lane");
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double red[NCH][NW][K];
    __shared__ double cpart[2][NCH][K];  // this CTA's partial of step j (parity j & 1), read over DSMEM
    __shared__ double fin[NCH][K];
    __shared__ double s_sh[HAS_S ? K : 1];
    __shared__ double red2[HAS_S ? NT / K : 1][K];  // flat grid: s_j second level
    __shared__ double red_mu[NMU][NW];              // flat grid: mu_j of this CTA's probe

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lg = tid % L, grp = tid / L;
    cg::cluster_group cluster = cg::this_cluster();
    // one cluster (RG = G: DSMEM halos and reductions) or a flat grid (RG = 1: halos through the
    // exported global rows, one grid counter per step)
    const int RG = a.rg, NG = (int)gridDim.x / ra.nblk;  // NG: CTAs per probe block
    const bool single = RG == NG;
    const int bb = (int)blockIdx.x / NG, cb = (int)blockIdx.x % NG;  // probe block, CTA within it
    const int crank = (int)cluster.block_rank();
    double mu_pend[NMU] = {};  // flat grid: part[tid][p] of step mu_j, summed one step later
    int32_t mu_j = 0;
    const int64_t r0 = (int64_t)cb * ra.nr;
    const int nr = (int)(a.d - r0 < (int64_t)ra.nr ? (a.d - r0 > 0 ? a.d - r0 : 0) : ra.nr);
    const ResLayout ly = res_layout<K>(ra.nr, ra.cap, a.r1u != nullptr);
    double* const W0 = reinterpret_cast<double*>(smem + ly.w0);
    double* const W1 = reinterpret_cast<double*>(smem + ly.w1);
    uint32_t* sg_s = reinterpret_cast<uint32_t*>(smem + ly.sg);
    double* u_s = reinterpret_cast<double*>(smem + ly.u);
    uint8_t* ex_s = smem + ly.ex;
    int32_t* rp_s = reinterpret_cast<int32_t*>(smem + ly.rp);
    int32_t* col_s = reinterpret_cast<int32_t*>(smem + ly.col);
    double* val_s = reinterpret_cast<double*>(smem + ly.val);
    int pp[NSL];
#pragma unroll
    for (int sl = 0; sl < NSL; sl++) pp[sl] = G::lane_probe(lg, sl);

    // ---- once per launch: the CTA's rows of the matrix, signs, u, export flags; w_0 = v
    const int64_t e0 = nr > 0 ? a.rp[r0] : 0, e1 = nr > 0 ? a.rp[r0 + nr] : 0;
    const bool fit = (e1 - e0) <= (int64_t)ra.cap;
    for (int x = tid; x <= nr; x += NT) rp_s[x] = (int32_t)(a.rp[r0 + x] - e0);
    if (fit)
        for (int64_t e = tid; e < e1 - e0; e += NT) {
            col_s[e] = a.ci[e0 + e];
            val_s[e] = a.va[e0 + e];
        }
    for (int x = tid; x < nr * WORDS; x += NT) sg_s[x] = a.sbits[(size_t)bb * ra.sb_stride + (size_t)r0 * WORDS + x];
    if (a.r1u)
        for (int x = tid; x < nr; x += NT) u_s[x] = a.r1u[r0 + x];
    for (int x = tid; x < nr; x += NT) ex_s[x] = ra.exp[r0 + x];
    if (HAS_S && tid < K) s_sh[tid] = __ldcg(ra.s_buf + (size_t)bb * K + tid);
    __syncthreads();
    for (int x = tid; x < nr * K; x += NT) {
        const int lr = x / K, p = x % K;
        W0[lr * RS + p] = pm1(sg_s[lr * WORDS + (p >> 5)], p & 31);
    }
    // kernel parameters used every step, pinned in registers: a parameter read from the constant
    // bank after a barrier can miss (measured neutral, kept for predictability)
    double* g0 = ra.g0;
    double* g1 = ra.g1;
    double* mu_out = a.mu_out + (size_t)bb * K * a.mu_stride;
    double* gpart = ra.gpart;
    unsigned int* bar_count = ra.bar_count;
    unsigned int* err = ra.err;
    const double* r1u = a.r1u;
    double r1ca = a.r1c_alpha;
    int64_t mu_stride = a.mu_stride;
    int32_t n_steps = ra.n, power = ra.power, kvalid = min(a.kvalid - bb * K, K);
    const int32_t* ci_g = a.ci;
    const double* va_g = a.va;
    asm volatile("" : "+l"(g0), "+l"(g1), "+l"(mu_out), "+l"(gpart), "+l"(bar_count), "+l"(err), "+l"(r1u));
    asm volatile("" : "+d"(r1ca), "+l"(mu_stride), "+r"(n_steps), "+r"(power), "+r"(kvalid), "+l"(ci_g), "+l"(va_g));
    // flat grid: the moments of step j (probe blockIdx.x) from the published partials
    auto mu_write = [&](double* row, int32_t jj, double q, double r) {
        if (DBL) dbl_write(row, jj, mu_stride - 1, q, r);
        else row[jj] = q;
    };
    auto mu_flush = [&]() {  // flat grid, after the last step
#pragma unroll
        for (int c = 0; c < NMU; c++) {
            const double m = warp_sum_xor(mu_pend[c]);
            if (lane == 0) red_mu[c][warp] = m;
        }
        __syncthreads();
        if (tid == 0) {
            double t[NMU];
#pragma unroll
            for (int c = 0; c < NMU; c++) {
                t[c] = 0.0;
                for (int w = 0; w < NW; w++) t[c] += red_mu[c][w];
            }
            mu_write(mu_out + (size_t)blockIdx.x * mu_stride, mu_j, t[0], t[NMU - 1]);
        }
    };
    cluster.sync();  // every peer's w_0 rows are in place
#if CHEB_RES_PROF
    long long prof_acc[6] = {0, 0, 0, 0, 0, 0}, prof_last = clock64();
#endif

    for (int32_t j = 1; j <= n_steps; j++) {
        const bool first = (j == 1) || power;
        const double* Wo = (j & 1) ? W0 : W1;  // w_{j-1}
        double* Wn = (j & 1) ? W1 : W0;        // w_{j-2} -> w_j
        const double* go = ((j - 1) & 1) ? g1 : g0;
        double* gn = (j & 1) ? g1 : g0;
        double2 r1[NSL];
#pragma unroll
        for (int sl = 0; sl < NSL; sl++)
            r1[sl] = HAS_S ? make_double2(r1ca * s_sh[pp[sl]], r1ca * s_sh[pp[sl] + 1])
                           : make_double2(0.0, 0.0);
        double acc[NCH][kPPL];
#pragma unroll
        for (int ch = 0; ch < NCH; ch++)
#pragma unroll
            for (int q = 0; q < kPPL; q++) acc[ch][q] = 0.0;
        const uint32_t wo_s = smem_u32(Wo);
        const uint64_t wo_gen = (uint64_t)Wo, go_gen = (uint64_t)go;  // generic addresses
        // one row: gathers (own rows: ld.shared; cluster peers: ld.shared::cluster at the mapa'd
        // address; other clusters: the exported global copy), rank-1 term, recurrence, dots
        auto rows = [&](auto staged, auto geo) {
            constexpr bool STAGED = decltype(staged)::value;
            // the row loop is specialised on the geometry -- 1: flat grid (own rows or the exported
            // global copy), 2: one cluster (own rows or a peer's over DSMEM)
            constexpr int GEO = decltype(geo)::value;
            for (int lr = grp; lr < nr; lr += GR) {
                const int lo = rp_s[lr], hi = rp_s[lr + 1];
                CHEB_ASSERT(lo <= hi && (hi - lo) % U == 0 && (!STAGED || hi <= ra.cap));
                double2 g[NSL];
#pragma unroll
                for (int sl = 0; sl < NSL; sl++) g[sl] = make_double2(0.0, 0.0);
                for (int t0 = lo; t0 < hi; t0 += U) {
                    int32_t c[U];
                    double v[U];
#pragma unroll
                    for (int q = 0; q < U; q++) {
                        c[q] = STAGED ? col_s[t0 + q] : __ldg(ci_g + e0 + t0 + q);
                        v[q] = STAGED ? val_s[t0 + q] : __ldg(va_g + e0 + t0 + q);
                    }
                    double2 x[U][NSL];
#pragma unroll
                    for (int q = 0; q < U; q++) {
                        if (CHEB_RES_DIAG == 1) {  // timing diagnostic: no gathers
                            x[q][0] = x[q][NSL - 1] = make_double2(v[q], 0.0);
                        } else if (CHEB_RES_DIAG == 2) {  // timing diagnostic: every gather from the own row
                            for (int sl = 0; sl < NSL; sl++) x[q][sl] = lds2(wo_s + (lr * RS + pp[sl]) * 8);
                        } else if (GEO == 1) {
                            // flat grid: the two sources share the generic address space, so the address is
                            // selected and one generic load issued -- no branch per entry, all of a
                            // chunk's loads back to back (configs[1]: 14.5 -> 13.8 ms per estimate)
                            CHEB_ASSERT(c[q] >= 0 ? (int64_t)c[q] < a.d : ((-1 - c[q]) >> 16) == 0 && ((-1 - c[q]) & 0xFFFF) < ra.nr);
                            const uint64_t ag = go_gen + (uint64_t)(uint32_t)c[q] * (K * 8);
                            const uint64_t as = wo_gen + (uint64_t)((uint32_t)(-1 - c[q]) & 0xFFFFu) * (RS * 8);
                            const uint64_t ad = c[q] >= 0 ? ag : as;
#pragma unroll
                            for (int sl = 0; sl < NSL; sl++) x[q][sl] = ldgen2(ad + pp[sl] * 8);
                        } else {
                            CHEB_ASSERT(c[q] < 0);  // one cluster: every column is a cluster row
                            const uint32_t e = (uint32_t)(-1 - c[q]);
                            const uint32_t rk = e >> 16;
                            CHEB_ASSERT((int)rk < RG && (int)(e & 0xFFFFu) < ra.nr);
                            const uint32_t ad = wo_s + (e & 0xFFFFu) * (RS * 8);
                            if (rk == (uint32_t)crank) {
#pragma unroll
                                for (int sl = 0; sl < NSL; sl++) x[q][sl] = lds2(ad + pp[sl] * 8);
                            } else {
                                const uint32_t adr = mapa_u32(ad, rk);
#pragma unroll
                                for (int sl = 0; sl < NSL; sl++) x[q][sl] = ldcl2(adr + pp[sl] * 8);
                            }
                        }
                    }
#pragma unroll
                    for (int q = 0; q < U; q++)
#pragma unroll
                        for (int sl = 0; sl < NSL; sl++) {
                            g[sl].x = fma(v[q], x[q][sl].x, g[sl].x);
                            g[sl].y = fma(v[q], x[q][sl].y, g[sl].y);
                        }
                }
                double ui = 1.0;
                if (HAS_S) {
                    ui = r1u ? u_s[lr] : 1.0;
#pragma unroll
                    for (int sl = 0; sl < NSL; sl++) {
                        g[sl].x = fma(ui, r1[sl].x, g[sl].x);
                        g[sl].y = fma(ui, r1[sl].y, g[sl].y);
                    }
                }
                const bool ex = ex_s[lr] != 0;
#pragma unroll
                for (int sl = 0; sl < NSL; sl++) {
                    double2* wp = reinterpret_cast<double2*>(Wn + lr * RS + pp[sl]);
                    double2 nw = g[sl];
                    if (!first) {
                        const double2 pv = *wp;
                        nw = make_double2(fma(2.0, g[sl].x, -pv.x), fma(2.0, g[sl].y, -pv.y));
                    }
                    *wp = nw;
                    if (ex) __stcg(reinterpret_cast<double2*>(gn + (size_t)(r0 + lr) * K + pp[sl]), nw);
                    if (DBL) {  // w_j^T w_j and w_{j-1}^T w_j over the own rows
                        const double2 ow = lds2(wo_s + (lr * RS + pp[sl]) * 8);
                        acc[0][2 * sl] = fma(nw.x, nw.x, acc[0][2 * sl]);
                        acc[0][2 * sl + 1] = fma(nw.y, nw.y, acc[0][2 * sl + 1]);
                        acc[1][2 * sl] = fma(ow.x, nw.x, acc[1][2 * sl]);
                        acc[1][2 * sl + 1] = fma(ow.y, nw.y, acc[1][2 * sl + 1]);
                    } else {  // v^T w_j: the sign bit of w flipped where the probe bit is set
                        const uint32_t bits = sg_s[lr * WORDS + (pp[sl] >> 5)] >> (pp[sl] & 31);
                        acc[0][2 * sl] += signflip(nw.x, bits << 31);
                        acc[0][2 * sl + 1] += signflip(nw.y, bits << 30);
                    }
                    if (HAS_S) {
                        acc[NCH - 1][2 * sl] = fma(ui, nw.x, acc[NCH - 1][2 * sl]);
                        acc[NCH - 1][2 * sl + 1] = fma(ui, nw.y, acc[NCH - 1][2 * sl + 1]);
                    }
                }
            }
        };
        using IC1 = std::integral_constant<int, 1>;
        using IC2 = std::integral_constant<int, 2>;
        if (single) {
            if (fit) rows(std::true_type{}, IC2{});
            else rows(std::false_type{}, IC2{});
        } else {
            if (fit) rows(std::true_type{}, IC1{});
            else rows(std::false_type{}, IC1{});
        }
        // ---- per-CTA partial: lanes of a warp -> warps in ascending order
#pragma unroll
        for (int off = L; off < 32; off <<= 1)
#pragma unroll
            for (int ch = 0; ch < NCH; ch++)
#pragma unroll
                for (int q = 0; q < kPPL; q++) acc[ch][q] += __shfl_xor_sync(0xffffffffu, acc[ch][q], off);
        if (lane < L) {
#pragma unroll
            for (int q = 0; q < kPPL; q++) {
                const int p = probe_of<K, kPPL, !G::WIDE>(lg, q);
#pragma unroll
                for (int ch = 0; ch < NCH; ch++) red[ch][warp][p] = acc[ch][q];
            }
        }
        if (!single && mu_j > 0) {  // the previous step's mu (flat grid): one butterfly, warps ascending
#pragma unroll
            for (int c = 0; c < NMU; c++) {
                const double m = warp_sum_xor(mu_pend[c]);
                if (lane == 0) red_mu[c][warp] = m;
            }
        }
        __syncthreads();
        RES_T(0);
        if (!single && mu_j > 0) {
            if (tid == 0) {
                double t[NMU];
#pragma unroll
                for (int c = 0; c < NMU; c++) {
                    t[c] = 0.0;
                    for (int w = 0; w < NW; w++) t[c] += red_mu[c][w];
                }
                mu_write(mu_out + (size_t)blockIdx.x * mu_stride, mu_j, t[0], t[NMU - 1]);
            }
            mu_j = 0;
        }
        const int par = j & 1;
        if (tid < NCH * K) {
            const int ch = tid / K, p = tid % K;
            double m = 0.0;
#pragma unroll 8
            for (int w = 0; w < NW; w++) m += red[ch][w][p];
            cpart[par][ch][p] = m;
        }
        RES_T(1);
        const bool want_s = HAS_S && j < n_steps;
        if (single) {
            // ---- one cluster: barrier, then every CTA sums the partials over DSMEM in rank order
            cluster.sync();  // the cluster's w_j rows and partials are complete
            RES_T(2);
            if (tid < NCH * K) {
                const int ch = tid / K, p = tid % K;
                double vr[kMaxRedGroup], sq = 0.0;
#pragma unroll
                for (int r = 0; r < kMaxRedGroup; r++) vr[r] = r < RG ? *cluster.map_shared_rank(&cpart[par][ch][p], r) : 0.0;
#pragma unroll
                for (int r = 0; r < kMaxRedGroup; r++) sq += vr[r];
                fin[ch][p] = sq;
            }
            __syncthreads();
            RES_T(3);
            if (cb == NG - 1 && tid < kvalid) mu_write(mu_out + (size_t)tid * mu_stride, j, fin[0][tid], fin[NMU - 1][tid]);
            if (want_s && tid < K) s_sh[tid] = fin[NCH - 1][tid];
        } else {
            // ---- flat grid (one CTA per SM, no clusters): every CTA publishes its partial, one
            // release-add on the grid counter, one wait.  pg: [NCH][NG][K] of step j.
            double* pg = gpart + (size_t)par * NCH * NG * K;
            if (tid < NCH * K) pg[((size_t)(tid / K) * NG + blockIdx.x) * K + tid % K] = cpart[par][tid / K][tid % K];
            __syncthreads();
            RES_T(2);
            if (tid == 0) {
                red_release_add(bar_count, 1u);                                  // release: w_j exports, partial
                spin_until_geq(bar_count, (unsigned int)j * (unsigned)NG, err);  // + acquire
            }
            __syncthreads();
            RES_T(5);
            // mu_j of probe blockIdx.x (CTAs < K), summed during the next step's partial reduction:
            // thread t holds part[t][p]
            if (blockIdx.x < (unsigned)kvalid) {
#pragma unroll
                for (int c = 0; c < NMU; c++)
                    mu_pend[c] = tid < NG ? __ldcg(pg + ((size_t)c * NG + tid) * K + blockIdx.x) : 0.0;
                mu_j = j;
            }
            if (want_s) {
                // s_j = sum over CTAs of part[c][S][p]: thread (u = tid / K, p = tid % K) sums
                // c = u, u + U, ... ascending (coalesced rows of K), then the u of one probe
                constexpr int UU = NT / K;
                const double* ps = pg + (size_t)(NCH - 1) * NG * K;
                const int p = tid % K, u = tid / K;
                // all of a chunk's loads in flight before the (ascending) adds: one L2 round trip
                // per 8 partials instead of one per partial (absent partials add +0.0)
                double t = 0.0;
                for (int c0 = u; c0 < NG; c0 += 8 * UU) {
                    double v8[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int c = c0 + q * UU;
                        v8[q] = c < NG ? __ldcg(ps + (size_t)c * K + p) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; q++) t += v8[q];
                }
                // second level: the lanes of a warp that hold the same probe (u ascending by lane),
                // then the warps / the u rows as four interleaved ascending sums -- a fixed order
                // with a short dependent chain (14.7 -> 14.6 ms per configs[1] estimate)
#pragma unroll
                for (int off = K; off < 32; off <<= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
                constexpr int UW = K < 32 ? NW : UU;
                if (K >= 32 || lane < K) red2[K < 32 ? warp : u][p] = t;
                __syncthreads();
                if (tid < K) {
                    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int v = 0; v < UW; v++) s4[v & 3] += red2[v][tid];
                    s_sh[tid] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
                }
            }
            RES_T(3);
        }
        __syncthreads();
        RES_T(4);
    }
    if (!single && mu_j > 0) {  // mu_n
        mu_flush();
    }
    // no CTA leaves while a cluster peer may still read its shared memory
    cluster.sync();
#if CHEB_RES_PROF
    if (tid == 0)
        for (int i = 0; i < 6; i++) g_res_prof[blockIdx.x * 8 + i] = prof_acc[i];
#endif
}

// ---------------------------------------------------------------------------------------
// K3: Y = B W (first half of applying B^T B; Alg. 2 via P:312-314).  Plain gather SpMM.
// ---------------------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(kThreads, CHEB_MIN_CTAS)
spmm_kernel(int64_t d, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
            const double* __restrict__ va, const double* __restrict__ x, double* __restrict__ y) {
    using G = SpmmGeo<K>;
    const int lg = threadIdx.x % G::L;
    const int grp = threadIdx.x / G::L;
    const int pa = 2 * lg, pb = K / 2 + 2 * lg;
    const int64_t ngroups_total = (int64_t)gridDim.x * G::GROUPS;
    for (int64_t i = (int64_t)blockIdx.x * G::GROUPS + grp; i < d; i += ngroups_total) {
        const int64_t e_lo = __ldg(rp + i), e_hi = __ldg(rp + i + 1);
        double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
        int64_t e = e_lo;
        for (; e + 4 <= e_hi; e += 4) {
            int32_t c[4];
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                c[q] = __ldg(ci + e + q);
                v[q] = __ldg(va + e + q);
            }
            double2 x0[4], x1[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const double* p = x + (size_t)(uint32_t)c[q] * K;
                x0[q] = ldg2(p + pa);
                x1[q] = ldg2(p + pb);
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                acc0.x = fma(v[q], x0[q].x, acc0.x);
                acc0.y = fma(v[q], x0[q].y, acc0.y);
                acc1.x = fma(v[q], x1[q].x, acc1.x);
                acc1.y = fma(v[q], x1[q].y, acc1.y);
            }
        }
        for (; e < e_hi; e++) {
            const int32_t c = __ldg(ci + e);
            const double v = __ldg(va + e);
            const double* p = x + (size_t)(uint32_t)c * K;
            const double2 x0 = ldg2(p + pa), x1 = ldg2(p + pb);
            acc0.x = fma(v, x0.x, acc0.x);
            acc0.y = fma(v, x0.y, acc0.y);
            acc1.x = fma(v, x1.x, acc1.x);
            acc1.y = fma(v, x1.y, acc1.y);
        }
        double* out = y + (size_t)i * K;
        *reinterpret_cast<double2*>(out + pa) = acc0;
        *reinterpret_cast<double2*>(out + pb) = acc1;
    }
}

// ---------------------------------------------------------------------------------------
// Accumulation (reading G7): one CTA.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
finalize_kernel(const double* __restrict__ mu, const double* __restrict__ c, int64_t m, int32_t n,
                double* __restrict__ gamma_p, double* __restrict__ stats) {
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

// ---------------------------------------------------------------------------------------
// Spectral interval of B^T B.  out[0] <- min_i s_i as an ordered key,
// out[1] <- max row abs sum, out[2] <- max column abs sum.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long order_key(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Quadratic form x^T A x for the GMRF likelihood scan: per-CTA partials
// (grid-stride rows, warp xor-butterfly, warps in order) then quadform_final_kernel sums
// the partials in CTA order -- deterministic.
// SPLIT: two sums, x^T D x (diagonal entries) and x^T O x (off-diagonal entries) -- the family
// M(theta) = D + theta O of the likelihood scan needs x^T M(theta) x = x^T D x + theta x^T O x.
template <bool SPLIT>
__global__ void __launch_bounds__(kThreads)
quadform_kernel(int64_t d, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                const double* __restrict__ va, const double* __restrict__ x, double* __restrict__ part) {
    constexpr int NO = SPLIT ? 2 : 1;
    __shared__ double wsum[NO][kThreads / 32];
    double acc[NO] = {};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
         i += (int64_t)gridDim.x * blockDim.x) {
        double r[NO] = {};
        for (int64_t e = rp[i]; e < rp[i + 1]; e++) {
            const int k = SPLIT && ci[e] != i ? 1 : 0;
            r[k] = fma(va[e], x[ci[e]], r[k]);
        }
#pragma unroll
        for (int k = 0; k < NO; k++) acc[k] = fma(x[i], r[k], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < NO; k++) {
        acc[k] = warp_sum_xor(acc[k]);
        if ((threadIdx.x & 31) == 0) wsum[k][threadIdx.x >> 5] = acc[k];
    }
    __syncthreads();
    if (threadIdx.x < NO) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; w++) t += wsum[threadIdx.x][w];
        part[(size_t)blockIdx.x * NO + threadIdx.x] = t;
    }
}
// sums the per-CTA partials in CTA order: out[k] = sum_c part[c * nout + k]
__global__ void quadform_final_kernel(const double* __restrict__ part, int n, int nout, double* __restrict__ out) {
    if (blockIdx.x == 0 && threadIdx.x < nout) {
        double t = 0.0;
        for (int c = 0; c < n; c++) t += part[(size_t)c * nout + threadIdx.x];
        out[threadIdx.x] = t;
    }
}

// Gershgorin-type upper bound on lambda_max of a CSR operator: out[0] <- max_i sum_j |a_ij|,
// out[1] <- max_i |u_i| (rank-1 u, if given).  Ordered-key atomics (order-independent).
// out[2] <- min_i (a_ii - sum_{j != i} |a_ij|) (Gershgorin lower end; ordered-key min).
__global__ void __launch_bounds__(kThreads)
gershgorin_kernel(int64_t d, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                  const double* __restrict__ va, const double* __restrict__ u, unsigned long long* out,
                  double off_scale = 1.0) {  // off_scale: |theta| of a family member D + theta O
    double rmax = 0.0, umax = 0.0, lmin = INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
         i += (int64_t)gridDim.x * blockDim.x) {
        double r = 0.0, off = 0.0, dg = 0.0;
        for (int64_t e = rp[i]; e < rp[i + 1]; e++) {
            const bool diag = ci[e] == i;
            const double x = diag ? fabs(va[e]) : off_scale * fabs(va[e]);
            r += x;
            if (diag) dg = va[e]; else off += x;
        }
        rmax = fmax(rmax, r);
        lmin = fmin(lmin, dg - off);
        if (u) umax = fmax(umax, fabs(u[i]));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
        umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, off));
        lmin = fmin(lmin, __shfl_xor_sync(0xffffffffu, lmin, off));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out + 0, order_key(rmax));
        atomicMax(out + 1, order_key(umax));
        atomicMin(out + 2, order_key(lmin));
    }
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
