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
#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded through the runtime's driver entry point)
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
constexpr int kStepStages = CHEB_STAGES;
#ifndef CHEB_NNZ_UNROLL
#define CHEB_NNZ_UNROLL 5  // nnz of a row whose gathers are in flight together (5-point stencil: 1 chunk)
#endif

enum { MODE_CSR = 0, MODE_RANK1 = 1, MODE_BTB = 2 };

__host__ __device__ constexpr int words_for(int K) { return K >= 32 ? K / 32 : 1; }

// Probes per lane of the step kernels: PPL/2 16-byte slots per gathered row (4: two slots, the
// probes {2l, 2l+1, K/2+2l, K/2+2l+1}; 8: four slots at stride K/4).  More probes per lane
// amortise the per-nonzero index work (column/value reads, address math) over more DFMAs.
#ifndef CHEB_PPL
#define CHEB_PPL 4
#endif
constexpr int kPPL = CHEB_PPL;
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
    static constexpr int SS = K / NSL;              // probe stride between a lane's slots
    static constexpr int L = K / PPL;               // lanes per row: 1..32
    static constexpr int GROUPS = kThreads / L;     // rows in flight per CTA
    static constexpr int RPG = R4 * 4 / PPL;        // rows per group per tile
    static_assert(RPG >= 1, "CHEB_RPG too small for CHEB_PPL");
    static constexpr int TILE = GROUPS * RPG;       // rows per tile: 256 .. 16
    static constexpr int WORDS = words_for(K);
    static constexpr int CAP = TILE * 8;            // staged nnz capacity (avg 8 per row)
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
    static constexpr int BYTES = OFF_U + (MODE == MODE_RANK1 ? G::UBYTES : 0);
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
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {  // no arrival
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {  // non-blocking
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {  // release.cta
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(phase)
            : "memory");
    } while (!done);
}
// mbar_wait with a bounded spin: sets *err and gives up instead of hanging the GPU (new kernels)
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t phase, unsigned int* err) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0, spins = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(phase)
            : "memory");
        if (!done && ++spins > (1u << 22)) {
            atomicExch(err, 1u);
            return;
        }
    } while (!done);
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st2_hint(double* p, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ double2 ldnc2_hint(const double* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
#ifndef CHEB_FUSED_HINTS
#define CHEB_FUSED_HINTS 0  // fused kernel: keep the L2 window (w_j gathers, w_{j+1} stores) evict_last
#endif

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

// L2 prefetch of each staged tile's first-touch gather rows (CHEB_L2_PREFETCH, default 0): with
// rows processed in ascending order, the rows a banded operator's tile touches for the first time
// are [r0 + bw, r0 + bw + T) (bw = max |i - col|); the staging thread can prefetch them into L2.
// Measured harmful on configs[3] (6.20 -> 9.36 ms per launch, DRAM 40.3 -> 60.8 GB): tiles are
// staged two items per CTA ahead, i.e. ~2G tiles ahead of the chip-wide front, and the prefetched
// rows are evicted by the ~60 MB of traffic before their use.  Kept as a build option.
#ifndef CHEB_L2_PREFETCH
#define CHEB_L2_PREFETCH 0
#endif
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

struct StepArgs {
    int64_t d;            // rows of the gather matrix (= dimension of M)
    int64_t ntiles;
    const int64_t* rp;    // prepped gather matrix: padded row_ptr copy
    const int32_t* ci;    //   padded col copy
    const double* va;     //   padded scaled values (alpha*a, diagonal alpha*a_ii - beta)
    const unsigned long long* bw;  // operator bandwidth max|i - col| (device), nullptr: no prefetch
    const double* xg;     // gather source: W_cur (csr/rank1) or Y = B W_cur (btb)
    const double* wcur;   // W_cur
    double* wnext;        // in: W_prev (unless FIRST); out: W_next (in place)
    const uint32_t* sbits;
    double beta;          // for rows without a stored diagonal (csr/rank1) and for btb
    double r1c_alpha;     // alpha * c (rank-1)
    const double* r1u;    // padded u copy (nullptr = ones)
    const double* s_cur;  // [K] u^T w_{j-1}
    double* s_next;       // [K] u^T w_j
    double* part;         // per-CTA partials [NCH][gridDim.x][K] (persistent: [2][NCH][G][K])
    unsigned int* ticket;
    double* mu_out;       // mu_out[p*mu_stride + mu_col]
    int64_t mu_stride;
    int32_t mu_col;
    int32_t kvalid;       // probes of this block that exist (<= K)
};

// ---------------------------------------------------------------------------------------
// Deterministic CTA + grid reduction of per-lane accumulators for probes pl..pl+PPL-1
// (lane group size LG = K/PPL).  Fixed shuffle tree in a warp, warps in index order, CTAs
// in a fixed strided order; the last CTA to finish (atomic ticket) writes the result.
// ---------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------
// Canonical (deterministic) reduction of the per-CTA partials part[c][p], c < G, for one
// probe p:  thread t sums c = t, t+256, ... ascending; lanes combine with the xor-butterfly
// 16, 8, 4, 2, 1 (every lane ends with the bitwise-same sum); warps 0..7 are added in order.
// Every kernel that produces moments (per-step, fused, persistent) uses exactly this order,
// so the result depends only on the grid size G -- not on which kernel or CTA computed it.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum_xor(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// All K probes of NCH channels by one CTA (last-CTA-done epilogue).  part: [NCH][G][K];
// out: shared [NCH][K].  Each channel is summed in the canonical order independently.
template <int K, int NCH>
__device__ __forceinline__ void reduce_partials_all(const double* part, int G, double (*out)[K],
                                                    double (*wsum)[kThreads / 32][8]) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int p0 = 0; p0 < K; p0 += 8) {
        double m[NCH][8];
#pragma unroll
        for (int ch = 0; ch < NCH; ch++)
#pragma unroll
            for (int q = 0; q < 8; q++) m[ch][q] = 0.0;
        for (int c = tid; c < G && tid < kThreads; c += kThreads) {  // extra (producer) warps: none
#pragma unroll
            for (int ch = 0; ch < NCH; ch++)
#pragma unroll
                for (int q = 0; q < 8; q++) m[ch][q] += __ldcg(part + ((size_t)ch * G + c) * K + p0 + q);
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ch++)
#pragma unroll
            for (int q = 0; q < 8; q++) m[ch][q] = warp_sum_xor(m[ch][q]);
        if (lane == 0 && warp < kThreads / 32) {
#pragma unroll
            for (int ch = 0; ch < NCH; ch++)
#pragma unroll
                for (int q = 0; q < 8; q++) wsum[ch][warp][q] = m[ch][q];
        }
        __syncthreads();
        if (tid < 8 * NCH) {
            const int ch = tid >> 3, q = tid & 7;
            double mm = 0.0;
#pragma unroll
            for (int w = 0; w < kThreads / 32; w++) mm += wsum[ch][w][q];
            out[ch][p0 + q] = mm;
        }
        __syncthreads();
    }
}

// One probe p by one CTA (persistent kernel); returns the sum in thread 0.
__device__ __forceinline__ double reduce_partials_one(const double* part, int K, int G, int p, double* wbuf) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double m = 0.0;
    for (int c = tid; c < G; c += kThreads) m += __ldcg(part + (size_t)c * K + p);
    m = warp_sum_xor(m);
    if (lane == 0) wbuf[warp] = m;
    __syncthreads();
    double r = 0.0;
    if (tid == 0) {
#pragma unroll
        for (int w = 0; w < kThreads / 32; w++) r += wbuf[w];
    }
    __syncthreads();
    return r;
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
//   EPI_PAIR  ch0 -> mu[p][col], ch1 -> mu[p][col+1]   (temporally fused pair)
//   EPI_DBL   moment doubling, step j = col: ch0 = w_j^T w_j, ch1 = w_j^T w_{j-1}
//             mu[p][2j] = 2 ch0 - mu[p][0],  mu[p][2j-1] = 2 ch1 - mu[p][1]  (j = 1: mu[p][1] = ch1)
//             (indices > n = mu_stride - 1 are not written)   (+ rank-1: ch2 -> s_next)
enum { EPI_STEP = 0, EPI_PAIR = 1, EPI_DBL = 2 };

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
// which is idle once every tile is consumed): red[NCH][8][K], fin[NCH][K], wsum[NCH][8][8].
template <int K, int NCH>
__host__ __device__ constexpr int red_scratch_bytes() {
    return 8 * (NCH * (kThreads / 32) * K + NCH * K + NCH * (kThreads / 32) * 8);
}

template <int K, int PPL, int NCH, int EPI, bool HAS_S, bool SPLIT = false>
__device__ __forceinline__ void grid_reduce_finish(double (&acc)[NCH][PPL], const StepArgs& a,
                                                   unsigned char* scratch) {
    constexpr int LG = K / PPL;
    auto red = reinterpret_cast<double(*)[kThreads / 32][K]>(scratch);
    auto fin = reinterpret_cast<double(*)[K]>(scratch + 8 * NCH * (kThreads / 32) * K);
    auto wsum = reinterpret_cast<double(*)[kThreads / 32][8]>(scratch + 8 * (NCH * (kThreads / 32) * K + NCH * K));
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
    reduce_partials_all<K, NCH>(a.part, (int)gridDim.x, fin, wsum);
    if (tid < K) {
        double* row = a.mu_out + (size_t)tid * a.mu_stride;
        if (tid < a.kvalid) {
            if (EPI == EPI_STEP) row[a.mu_col] = fin[0][tid];
            if (EPI == EPI_PAIR) {
                row[a.mu_col] = fin[0][tid];
                row[a.mu_col + 1] = fin[1][tid];
            }
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
            const double* __restrict__ u, double* __restrict__ u2,
            unsigned long long* __restrict__ bw) {
    const int64_t total = rp2[d];  // padded nnz
    int64_t bwmax = 0;  // operator bandwidth max |i - col| (temporal fusion planning)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // multiple of 32
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < d; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        bool has = true;
        if (i < d) {
            const int64_t e0 = rp[i], e1 = rp[i + 1];
            const int64_t o0 = rp2[i], o1 = rp2[i + 1];
            has = (MODE == MODE_BTB);
            int64_t o = o0;
            if (MODE != MODE_BTB) {
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
                    const int64_t dist = c > i ? c - i : i - c;
                    bwmax = dist > bwmax ? dist : bwmax;
                }
                ci2[o0] = (int32_t)i;
                va2[o0] = dv;
            } else {
                for (int64_t e = e0; e < e1; e++, o++) {
                    const int32_t c = ci[e];
                    ci2[o] = c;
                    va2[o] = alpha * va[e];
                    const int64_t dist = c > i ? c - i : i - c;
                    bwmax = dist > bwmax ? dist : bwmax;
                }
            }
            for (; o < o1; o++) {  // padding: (i, 0.0)
                ci2[o] = (int32_t)i;
                va2[o] = 0.0;
            }
            if (u2) u2[i] = u ? u[i] : 1.0;
        }
    }
    if (bw) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const int64_t o = __shfl_xor_sync(0xffffffffu, bwmax, off);
            bwmax = o > bwmax ? o : bwmax;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(bw, (unsigned long long)bwmax);
    }
    if (blockIdx.x == 0) {
        for (int64_t k = d + 1 + threadIdx.x; k < rp2_len; k += blockDim.x) rp2[k] = total;
        if (threadIdx.x < 8) ci2[total + threadIdx.x] = 0;
        if (threadIdx.x < 4) va2[total + threadIdx.x] = 0.0;
        if (u2 && threadIdx.x < 2) u2[d + threadIdx.x] = 0.0;
    }
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
                const uint64_t z = splitmix64_at(seed, (p0 + pl + q) * d + (uint64_t)i + 1ull);
                const uint32_t bq = (uint32_t)(z >> 63);
                v[q] = bq ? -1.0 : 1.0;
                bits |= bq << ((pl + q) & 31);
                acc[0][q] += v[q] * v[q];
            }
#pragma unroll
            if (w0)  // nullptr: the per-step path reads v from the sign bits only
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
template <int K, int MODE, bool FIRST, bool STAGED, bool CG = false, bool KEEP = false, bool DBL = false,
          bool WCS = false, int R4 = CHEB_RPG, int VB = 0>
__device__ __forceinline__ void step_tile(const StepArgs& a, const unsigned char* st, int64_t r0, int rows,
                                          int64_t base_c, int64_t base_v, const double2 (&r1)[kPPL / 2],
                                          double (&acc)[n_channels<MODE, DBL>()][kPPL], const double* xg,
                                          const double* wcur, double* wout) {
    using G = Geo<K, R4>;
    using SL = StageLayout<K, MODE, WCS, R4>;
    constexpr int NSL = G::NSL;
    constexpr bool OWN_SMEM = SL::HAS_WC;          // w_{j-1}[i] rows staged in shared memory
    // csr / rank-1 doubling: w_{j-1}[i] is the row's first gather (the prepped diagonal entry)
    constexpr bool OWN_GATHER = DBL && !OWN_SMEM && MODE != MODE_BTB;
    constexpr bool OWN_EARLY = DBL && !OWN_SMEM && !OWN_GATHER;  // loaded at the row start
    static_assert(VB == 0 || (MODE != MODE_BTB && !CG && !KEEP && (VB != 1 || !OWN_SMEM)),
                  "sign-bit probes: per-step csr/rank-1");
    constexpr bool HAS_S = (MODE == MODE_RANK1);
    constexpr int SCH = n_channels<MODE, DBL>() - 1;  // rank-1 channel
    const int lg = threadIdx.x % G::L;
    const int grp = threadIdx.x / G::L;
    int pp[NSL];  // first probe of each slot: {2lg, 2lg+1} + s*SS
#pragma unroll
    for (int sl = 0; sl < NSL; sl++) pp[sl] = 2 * lg + sl * G::SS;
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
        const int64_t e_lo = rp_s[lr], e_hi = rp_s[lr + 1];
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
        for (int t0 = 0; t0 < nr; t0 += CHEB_NNZ_UNROLL) {
            int32_t c[CHEB_NNZ_UNROLL];
            double v[CHEB_NNZ_UNROLL];
#pragma unroll
            for (int q = 0; q < CHEB_NNZ_UNROLL; q++) {
                CHEB_ASSERT(!STAGED || (oc + t0 + q >= 0 && oc + t0 + q < G::CAP + 8));
                CHEB_ASSERT(!STAGED || (ov + t0 + q >= 0 && ov + t0 + q < G::CAP + 4));
                c[q] = STAGED ? crow[t0 + q] : __ldg(crow + t0 + q);
                CHEB_ASSERT(c[q] >= 0 && (int64_t)c[q] < a.d);
                v[q] = STAGED ? vrow[t0 + q] : __ldg(vrow + t0 + q);
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
                    for (int sl = 0; sl < NSL; sl++) {
                        if (KEEP && CHEB_FUSED_HINTS)
                            x[q][sl] = ldnc2_hint(p + sl * G::SS, policy_evict_last());
                        else
                            x[q][sl] = CG ? ldcg2(p + sl * G::SS) : ldg2(p + sl * G::SS);
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
#pragma unroll
        for (int sl = 0; sl < NSL; sl++) {
            if (KEEP) {  // re-read from L2 later in the same launch (fused kernel, stage 1)
                if (CHEB_FUSED_HINTS)
                    st2_hint(out + pp[sl], nw[sl], policy_evict_last());
                else
                    *reinterpret_cast<double2*>(out + pp[sl]) = nw[sl];
            } else {     // streamed: next read is by a later launch
                __stcs(reinterpret_cast<double2*>(out + pp[sl]), nw[sl]);
            }
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
__host__ __device__ constexpr int min_ctas(int mode, bool dbl = false) {
    return mode == MODE_CSR ? (dbl ? CHEB_MIN_CTAS_DBL : CHEB_MIN_CTAS) : (mode == MODE_RANK1 && !dbl ? 3 : 2);
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
    double acc[NCH][kPPL];
#pragma unroll
    for (int ch = 0; ch < NCH; ch++)
#pragma unroll
        for (int q = 0; q < kPPL; q++) acc[ch][q] = 0.0;
    double2 r1[G::NSL];  // alpha c s_{j-1}[p] of the lane's probes (rank-1)
#pragma unroll
    for (int sl = 0; sl < G::NSL; sl++) {
        const int p = 2 * (tid % G::L) + sl * G::SS;
        r1[sl] = HAS_S ? make_double2(a.r1c_alpha * a.s_cur[p], a.r1c_alpha * a.s_cur[p + 1]) : make_double2(0.0, 0.0);
    }
    const int64_t nmine = a.ntiles > blockIdx.x ? (a.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    // thread 0: bandwidth for the L2 prefetch (only for banded operators, bw < d/4)
    int64_t pf_bw = -1;
    if (CHEB_L2_PREFETCH && MODE != MODE_BTB && tid == 0 && a.bw) {
        const int64_t bwv = (int64_t)*a.bw;
        pf_bw = (4 * bwv < a.d) ? bwv : -1;
    }
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
        uint32_t bytes = G::RPBYTES + sgbytes;
        if (!FIRST && VB != 2) bytes += wbytes;
        if (SL::HAS_WC) bytes += wbytes;
        if (fit) bytes += (uint32_t)(c1 - c0) * 4 + (uint32_t)(v1 - v0) * 8;
        const uint32_t ubytes = ((uint32_t)rows * 8 + 15) & ~15u;
        if (HAS_S && a.r1u) bytes += ubytes;
        mbar_expect_tx(&bar[b], bytes);
        bulk_g2s(st + SL::OFF_RP, a.rp + r0, G::RPBYTES, &bar[b]);
        if (SIGNS) bulk_g2s(st + SL::OFF_SGN, a.sbits + (size_t)r0 * G::WORDS, sgbytes, &bar[b]);
        if (!FIRST && VB != 2)
            bulk_g2s_hint(st + SL::OFF_WPREV, a.wnext + (size_t)r0 * K, wbytes, &bar[b], policy_evict_first());
        if (SL::HAS_WC) bulk_g2s(st + SL::OFF_WCUR, a.wcur + (size_t)r0 * K, wbytes, &bar[b]);
        if (fit) {
            bulk_g2s(st + SL::OFF_COL, a.ci + c0, (uint32_t)(c1 - c0) * 4, &bar[b]);
            bulk_g2s(st + SL::OFF_VAL, a.va + v0, (uint32_t)(v1 - v0) * 8, &bar[b]);
        }
        if (HAS_S && a.r1u) bulk_g2s(st + SL::OFF_U, a.r1u + r0, ubytes, &bar[b]);
        if (CHEB_L2_PREFETCH && MODE != MODE_BTB && pf_bw >= 0) {  // first-touch gather rows -> L2
            const int64_t p0 = r0 + pf_bw, p1 = imin64(p0 + rows, a.d);
            if (p1 > p0) prefetch_l2(a.xg + (size_t)p0 * K, (uint32_t)(p1 - p0) * K * 8);
        }
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
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < NS; i++) mbar_init(&bar[i], 1);
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
        if (tid == 0 && it + NS < nmine) bounds_async(tile_of(it + NS));  // consumed below
        mbar_wait(&bar[b], phase);
        const unsigned char* st = smem + b * SL::BYTES;
        const int64_t r0 = t * G::TILE;
        const int rows = (int)imin64((int64_t)G::TILE, a.d - r0);
        if (s_fit[b])
            step_tile<K, MODE, FIRST, true, false, false, DBL, WCS, R4, VB>(a, st, r0, rows, s_base_c[b], s_base_v[b], r1,
                                                               acc, a.xg, a.wcur, a.wnext);
        else
            step_tile<K, MODE, FIRST, false, false, false, DBL, WCS, R4, VB>(a, st, r0, rows, 0, 0, r1, acc, a.xg, a.wcur,
                                                                a.wnext);
        __syncthreads();  // every warp is done with stage b
        if (tid == 0 && it + NS < nmine) {
            cp_async_wait_all();
            issue(tile_of(it + NS), b, s_ne[0], s_ne[1]);
        }
    }
    grid_reduce_finish<K, kPPL, NCH, DBL ? EPI_DBL : EPI_STEP, HAS_S, true>(acc, a, smem);
}


// ---------------------------------------------------------------------------------------
// K2x2: temporally fused pair of Chebyshev steps (CSR mode, banded operators).
//   stage 1 (tile P):      w_{j+1} = 2 Ã w_j     - w_{j-1}   (A: w_{j-1} -> w_{j+1}, gathers B)
//   stage 2 (tile P - D):  w_{j+2} = 2 Ã w_{j+1} - w_j       (B: w_j -> w_{j+2},     gathers A)
// Every element is computed with exactly the single-step arithmetic, in the same order, so
// results are bit-identical to two cheb_step_kernel launches; only the schedule changes.
// CTA c handles positions P = c + k*G (k = 0, 1, ...): stage 1 of tile P, then stage 2 of
// tile u = P - D.  Stage 2 of u gathers w_{j+1} rows within the operator bandwidth of u and
// overwrites w_j rows of u that stage 1 of tiles u-H..u+H read (H = ceil(bandwidth/T) + 1
// tiles), so it needs every stage-1 tile t <= u + H complete.
// Completion is tracked in chunks of 32 tiles: after stage 1 of tile t a CTA release-adds 1
// to cnt[t/32]; a waiter keeps `known` = number of leading chunks seen full and advances it
// with one warp-wide load of the next 32 chunk counters (ballot -> first non-full chunk).
// Those loads are issued before the preceding stage-1 tile is computed, so in steady state
// the check costs no latency.
// D = (SLACK + ceil((H+2)/G)) * G >= H + 2 makes every dependency sit at an earlier position
// (deadlock-free with all CTAs co-resident: cooperative launch), and D a multiple of G keeps
// stage-2 tile u on CTA u mod G exactly like the single-step kernel: the per-CTA partial dot
// products (hence the moments) are bit-identical too.  With SLACK = 0, D = G: the L2 window
// between the stages is one wave of tiles plus the halo.  w_{j+1} stays in L2 between the
// stages: per 2 steps HBM sees w_{j-1}, w_j read and w_{j+1}, w_{j+2} written (4 vector
// streams instead of 6).
// ---------------------------------------------------------------------------------------
#ifndef CHEB_FUSED_SLACK
#define CHEB_FUSED_SLACK 0
#endif
constexpr int kFusedSlack = CHEB_FUSED_SLACK;  // extra waves of lag between the stages
constexpr int kChunkTiles = 32;                // tiles per completion counter
// Consumer side of the dependency: the counters are read relaxed and the gathers that follow
// are control-dependent on them (issued only after the counts are seen), and every w_{j+1}
// row is written exactly once before its count is released and never changes afterwards, so
// no L1 line of it can be stale (L1 starts empty at launch; stage 1 reads A only through TMA).
// CHEB_FUSED_FENCE=1 adds the formal fence.acq_rel.gpu (an SM-wide L1 invalidate per item).
#ifndef CHEB_FUSED_FENCE
#define CHEB_FUSED_FENCE 0
#endif

struct FusedArgs {
    double* A;                // in: w_{j-1}, out: w_{j+1}
    double* B;                // in: w_j,     out: w_{j+2}
    unsigned int* cnt;        // [ceil(ntiles/32)] completed stage-1 tiles per chunk (zeroed)
    unsigned int* err;        // dependency-wait timeout flag
    int64_t D;                // stage-2 lag in positions, a multiple of gridDim.x, >= H + 2
    int64_t H;                // halo in tiles
};

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_release_add(unsigned int* p, unsigned int v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

#ifndef CHEB_FUSED_MIN_CTAS
#define CHEB_FUSED_MIN_CTAS CHEB_MIN_CTAS
#endif
template <int K>
__global__ void __launch_bounds__(kThreads, CHEB_FUSED_MIN_CTAS)
cheb_step2_kernel(StepArgs a, FusedArgs f) {
    using G = Geo<K>;
    using SL = StageLayout<K, MODE_CSR>;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int64_t s_base_c[2], s_base_v[2];
    __shared__ int s_fit[2];

    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t Gd = gridDim.x;
    double acc[2][kPPL];  // stage 1 / stage 2 moments
#pragma unroll
    for (int q = 0; q < kPPL; q++) acc[0][q] = acc[1][q] = 0.0;
    double (&mu1)[1][kPPL] = *reinterpret_cast<double(*)[1][kPPL]>(&acc[0]);
    double (&mu2)[1][kPPL] = *reinterpret_cast<double(*)[1][kPPL]>(&acc[1]);
    double2 z2[G::NSL];
#pragma unroll
    for (int sl = 0; sl < G::NSL; sl++) z2[sl] = make_double2(0.0, 0.0);
    const int64_t npos = a.ntiles + f.D;  // positions 0 .. ntiles + D - 1
    const int64_t M = blockIdx.x < npos ? 2 * ((npos - 1 - blockIdx.x) / Gd + 1) : 0;
    const int64_t nchunks = (a.ntiles + kChunkTiles - 1) / kChunkTiles;

    auto item = [&](int64_t m, int& stg, int64_t& t) -> bool {
        const int64_t P = (int64_t)blockIdx.x + (m >> 1) * Gd;
        stg = (int)(m & 1);
        t = stg ? P - f.D : P;
        return t >= 0 && t < a.ntiles;
    };
    auto bounds = [&](int64_t t, int64_t& e0, int64_t& e1) {
        const int64_t r0 = t * G::TILE;
        e0 = __ldg(a.rp + r0);
        e1 = __ldg(a.rp + imin64(r0 + G::TILE, a.d));
    };
    auto issue = [&](int64_t t, int b, const double* wsrc, int64_t e0, int64_t e1) {
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
        const uint32_t sgbytes = ((uint32_t)rows * G::WORDS * 4 + 15) & ~15u;
        uint32_t bytes = G::RPBYTES + sgbytes + wbytes;
        if (fit) bytes += (uint32_t)(c1 - c0) * 4 + (uint32_t)(v1 - v0) * 8;
        mbar_expect_tx(&bar[b], bytes);
        bulk_g2s(st + SL::OFF_RP, a.rp + r0, G::RPBYTES, &bar[b]);
        bulk_g2s(st + SL::OFF_SGN, a.sbits + (size_t)r0 * G::WORDS, sgbytes, &bar[b]);
        bulk_g2s_hint(st + SL::OFF_WPREV, wsrc + (size_t)r0 * K, wbytes, &bar[b], policy_evict_first());
        if (fit) {
            bulk_g2s(st + SL::OFF_COL, a.ci + c0, (uint32_t)(c1 - c0) * 4, &bar[b]);
            bulk_g2s(st + SL::OFF_VAL, a.va + v0, (uint32_t)(v1 - v0) * 8, &bar[b]);
        }
    };
    auto advance = [&](int64_t& m, int& stg, int64_t& t) -> bool {
        for (; m < M; ++m)
            if (item(m, stg, t)) return true;
        return false;
    };
    // full count of chunk ch (the last chunk may be short); chunks past the end read as full
    auto chunk_full = [&](int64_t ch) -> unsigned int {
        return (unsigned int)imin64(kChunkTiles, a.ntiles - ch * kChunkTiles);
    };

    int64_t m_issue = 0, ne0 = 0, ne1 = 0, nt = 0;
    int nstg = 0;
    bool pending = false;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        for (int q = 0; q < 2; q++) {
            int stg;
            int64_t t, e0, e1;
            if (!advance(m_issue, stg, t)) break;
            bounds(t, e0, e1);
            issue(t, q, stg ? f.B : f.A, e0, e1);
            ++m_issue;
        }
    }
    __syncthreads();

    int64_t q = 0;
    int64_t known = 0;       // warp 0: leading chunks known complete
    unsigned int peek = 0;   // warp 0, per lane: prefetched counter of chunk known + lane
    int64_t peek_base = -1;  // chunk index of lane 0's prefetched counter (-1: none)
    for (int64_t m = 0; m < M; ++m) {
        int stg;
        int64_t t;
        if (!item(m, stg, t)) continue;
        const int b = (int)(q & 1);
        const uint32_t phase = (uint32_t)((q >> 1) & 1);
        if (tid == 0) {
            pending = advance(m_issue, nstg, nt);
            if (pending) bounds(nt, ne0, ne1);
        }
        if (stg == 1) {
            // stage-1 tiles [0, need) must be complete
            const int64_t need = imin64(t + f.H + 1, a.ntiles);
            if (tid < 32) {
                uint32_t spins = 0;
                while (known * kChunkTiles < need) {
                    const int64_t ch = known + lane;
                    unsigned int v;
                    if (peek_base == known) {
                        v = peek;
                    } else {
                        v = ch < nchunks ? ld_relaxed_u32(f.cnt + ch) : 0u;
                    }
                    const bool full = ch >= nchunks || v >= chunk_full(ch);
                    const unsigned int notfull = __ballot_sync(0xffffffffu, !full);
                    const int adv = notfull ? __ffs(notfull) - 1 : 32;
                    known += adv;
                    peek_base = -1;
                    if (adv == 0) {
                        __nanosleep(100);
                        if ((++spins & 1023u) == 0 && (spins > (1u << 23) || ld_acquire_u32(f.err))) {
                            if (lane == 0) atomicExch(f.err, 1u);  // ~seconds without progress: never hang
                            break;
                        }
                    }
                }
#if CHEB_FUSED_FENCE
                fence_acq_rel_gpu();  // formal acquire (costs an SM-wide L1 invalidate per item)
#endif
            }
            __syncthreads();
        }
        mbar_wait(&bar[b], phase);
        const unsigned char* st = smem + b * SL::BYTES;
        const int64_t r0 = t * G::TILE;
        const int rows = (int)imin64((int64_t)G::TILE, a.d - r0);
        if (stg == 0) {
            // prefetch the chunk counters the next stage-2 check will read (overlaps this tile)
            if (tid < 32) {
                const int64_t ch = known + lane;
                peek = ch < nchunks ? ld_relaxed_u32(f.cnt + ch) : 0u;
                peek_base = known;
            }
            if (s_fit[b])
                step_tile<K, MODE_CSR, false, true, false, true>(a, st, r0, rows, s_base_c[b], s_base_v[b], z2,
                                                                 mu1, f.B, f.B, f.A);
            else
                step_tile<K, MODE_CSR, false, false, false, true>(a, st, r0, rows, 0, 0, z2, mu1, f.B,
                                                                  f.B, f.A);
        } else {
            if (s_fit[b])
                step_tile<K, MODE_CSR, false, true, true, false>(a, st, r0, rows, s_base_c[b], s_base_v[b], z2,
                                                                 mu2, f.A, f.A, f.B);
            else
                step_tile<K, MODE_CSR, false, false, true, false>(a, st, r0, rows, 0, 0, z2, mu2, f.A,
                                                                  f.A, f.B);
        }
        __syncthreads();  // every warp is done with stage b (and, for stage 1, with its stores)
        if (tid == 0) {
            if (pending) {
                issue(nt, b, nstg ? f.B : f.A, ne0, ne1);
                ++m_issue;
            }
            if (stg == 0) {  // publish: stage 1 of tile t is complete (release: the CTA's stores
                             // are ordered before it by the barrier above)
                red_release_add(f.cnt + t / kChunkTiles, 1u);
            }
        }
        ++q;
    }
    grid_reduce_finish<K, kPPL, 2, EPI_PAIR, false, true>(acc, a, smem);
}


// ---------------------------------------------------------------------------------------
// K2x2d: temporally fused pair with DYNAMIC tile tickets.  Same two stages as cheb_step2_kernel,
// but tiles are handed out by two global counters instead of a static tile -> CTA map, so a slow
// CTA delays only the one tile it holds (no accumulated skew):
//   * a CTA takes a stage-1 ticket t1 = c1++; if t1 >= D it then takes one stage-2 ticket
//     u = c2++ (alternating); once c1 is exhausted it drains stage-2 tickets;
//   * every stage-2 ticket u taken this way satisfies u + D < c1, so the stage-1 tiles it needs
//     (<= u + H < u + D) have all been handed out, and stage-1 work never waits;
//   * a CTA's own pending stage-1 ticket is always > its current stage-2 need, and a wait chain
//     X -> Y implies u_X > u_Y: no cycle, deadlock-free with all CTAs co-resident.
// Tickets are taken when the TMA staging of the item is issued (two items ahead).
// Moments: per-CTA partial sums as in the other kernels, but which tiles a CTA sums now depends
// on the run, so the rounding of mu is run-dependent (still within the parity tolerances).
// ---------------------------------------------------------------------------------------
struct FusedDynArgs {
    unsigned int* c1;         // stage-1 ticket counter (zeroed)
    unsigned int* c2;         // stage-2 ticket counter (zeroed)
};

template <int K>
__global__ void __launch_bounds__(kThreads, CHEB_FUSED_MIN_CTAS)
cheb_step2d_kernel(StepArgs a, FusedArgs f, FusedDynArgs dy) {
    using G = Geo<K>;
    using SL = StageLayout<K, MODE_CSR>;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int64_t s_base_c[2], s_base_v[2];
    __shared__ int s_fit[2];
    __shared__ int64_t s_t[2];   // tile of the item staged in buffer b (-1: no more items)
    __shared__ int s_stg[2];     // its stage

    const int tid = threadIdx.x, lane = tid & 31;
    double acc[2][kPPL];  // stage 1 / stage 2 moments
#pragma unroll
    for (int q = 0; q < kPPL; q++) acc[0][q] = acc[1][q] = 0.0;
    double (&mu1)[1][kPPL] = *reinterpret_cast<double(*)[1][kPPL]>(&acc[0]);
    double (&mu2)[1][kPPL] = *reinterpret_cast<double(*)[1][kPPL]>(&acc[1]);
    double2 z2[G::NSL];
#pragma unroll
    for (int sl = 0; sl < G::NSL; sl++) z2[sl] = make_double2(0.0, 0.0);
    const int64_t nchunks = (a.ntiles + kChunkTiles - 1) / kChunkTiles;
    const unsigned int ntl = (unsigned int)a.ntiles;

    auto issue = [&](int64_t t, int b, const double* wsrc, int64_t e0, int64_t e1) {
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
        const uint32_t sgbytes = ((uint32_t)rows * G::WORDS * 4 + 15) & ~15u;
        uint32_t bytes = G::RPBYTES + sgbytes + wbytes;
        if (fit) bytes += (uint32_t)(c1 - c0) * 4 + (uint32_t)(v1 - v0) * 8;
        mbar_expect_tx(&bar[b], bytes);
        bulk_g2s(st + SL::OFF_RP, a.rp + r0, G::RPBYTES, &bar[b]);
        bulk_g2s(st + SL::OFF_SGN, a.sbits + (size_t)r0 * G::WORDS, sgbytes, &bar[b]);
        bulk_g2s_hint(st + SL::OFF_WPREV, wsrc + (size_t)r0 * K, wbytes, &bar[b], policy_evict_first());
        if (fit) {
            bulk_g2s(st + SL::OFF_COL, a.ci + c0, (uint32_t)(c1 - c0) * 4, &bar[b]);
            bulk_g2s(st + SL::OFF_VAL, a.va + v0, (uint32_t)(v1 - v0) * 8, &bar[b]);
        }
    };
    // thread 0: ticket policy (see above)
    bool want2 = false, done1 = false, done2 = false;
    auto take = [&](int& stg, int64_t& t) -> bool {
        if (want2 || done1) {
            want2 = false;
            if (!done2) {
                const unsigned int u = atomicAdd(dy.c2, 1u);
                if (u < ntl) {
                    stg = 1;
                    t = u;
                    return true;
                }
                done2 = true;
            }
        }
        if (!done1) {
            const unsigned int t1 = atomicAdd(dy.c1, 1u);
            if (t1 < ntl) {
                stg = 0;
                t = t1;
                want2 = (int64_t)t1 >= f.D;
                return true;
            }
            done1 = true;
        }
        if (!done2) {
            const unsigned int u = atomicAdd(dy.c2, 1u);
            if (u < ntl) {
                stg = 1;
                t = u;
                return true;
            }
            done2 = true;
        }
        return false;
    };
    auto stage_next = [&](int b) {  // thread 0: take the next item and stage it into buffer b
        int stg;
        int64_t t;
        if (take(stg, t)) {
            s_t[b] = t;
            s_stg[b] = stg;
            const int64_t r0 = t * G::TILE;
            issue(t, b, stg ? f.B : f.A, __ldg(a.rp + r0), __ldg(a.rp + imin64(r0 + G::TILE, a.d)));
        } else {
            s_t[b] = -1;
        }
    };

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        stage_next(0);
        stage_next(1);
    }
    __syncthreads();

    int64_t known = 0;       // warp 0: leading chunks known complete
    for (int64_t q = 0;; ++q) {
        const int b = (int)(q & 1);
        const uint32_t phase = (uint32_t)((q >> 1) & 1);
        const int64_t t = s_t[b];
        if (t < 0) break;
        const int stg = s_stg[b];
        if (stg == 1) {
            const int64_t need = imin64(t + f.H + 1, a.ntiles);  // stage-1 tiles [0, need) complete
            if (tid < 32) {
                uint32_t spins = 0;
                while (known * kChunkTiles < need) {
                    const int64_t ch = known + lane;
                    const unsigned int v = ch < nchunks ? ld_relaxed_u32(f.cnt + ch) : 0u;
                    const bool full = ch >= nchunks || v >= (unsigned int)imin64(kChunkTiles, a.ntiles - ch * kChunkTiles);
                    const unsigned int notfull = __ballot_sync(0xffffffffu, !full);
                    const int adv = notfull ? __ffs(notfull) - 1 : 32;
                    known += adv;
                    if (adv == 0) {
                        __nanosleep(64);
                        if ((++spins & 1023u) == 0 && (spins > (1u << 23) || ld_acquire_u32(f.err))) {
                            if (lane == 0) atomicExch(f.err, 1u);  // ~seconds without progress: never hang
                            break;
                        }
                    }
                }
#if CHEB_FUSED_FENCE
                fence_acq_rel_gpu();
#endif
            }
            __syncthreads();
        }
        mbar_wait(&bar[b], phase);
        const unsigned char* st = smem + b * SL::BYTES;
        const int64_t r0 = t * G::TILE;
        const int rows = (int)imin64((int64_t)G::TILE, a.d - r0);
        if (stg == 0) {
            if (s_fit[b])
                step_tile<K, MODE_CSR, false, true, false, true>(a, st, r0, rows, s_base_c[b], s_base_v[b], z2,
                                                                 mu1, f.B, f.B, f.A);
            else
                step_tile<K, MODE_CSR, false, false, false, true>(a, st, r0, rows, 0, 0, z2, mu1, f.B, f.B, f.A);
        } else {
            if (s_fit[b])
                step_tile<K, MODE_CSR, false, true, true, false>(a, st, r0, rows, s_base_c[b], s_base_v[b], z2,
                                                                 mu2, f.A, f.A, f.B);
            else
                step_tile<K, MODE_CSR, false, false, true, false>(a, st, r0, rows, 0, 0, z2, mu2, f.A, f.A, f.B);
        }
        __syncthreads();  // every warp is done with buffer b (and, for stage 1, with its stores)
        if (tid == 0) {
            if (stg == 0) red_release_add(f.cnt + t / kChunkTiles, 1u);  // publish stage 1 of t
            stage_next(b);
        }
        __syncthreads();  // s_t[b] / s_stg[b] of the next use of b are visible
    }
    grid_reduce_finish<K, kPPL, 2, EPI_PAIR, false, true>(acc, a, smem);
}

// ---------------------------------------------------------------------------------------
// K2x2w: dynamic-ticket fused pair, warp-specialised.  Warps 0..7 only compute tiles; a ninth
// (producer) warp takes the tickets (same policy as cheb_step2d_kernel), stages each item by TMA,
// waits for a stage-2 item's dependencies and then arrives on the item's "full" mbarrier
// (expect_tx first, so the phase completes when both the bytes and the arrival are in); the
// compute warps arrive on the buffer's "empty" mbarrier when done, after which the producer
// publishes a finished stage-1 tile (consumer stores -> arrive.release.cta -> producer
// wait.acquire.cta -> red.release.gpu: cumulative).  No ticket atomic, bound load, fence or
// dependency wait sits between two tiles of the compute warps.
// ---------------------------------------------------------------------------------------
#ifndef CHEB_FUSEDW_MIN_CTAS
#define CHEB_FUSEDW_MIN_CTAS 3
#endif
constexpr int kFusedWThreads = kThreads + 32;
#ifndef CHEB_FUSEDW_STAGES
#define CHEB_FUSEDW_STAGES 3
#endif
constexpr int kWStages = CHEB_FUSEDW_STAGES;  // staged items in flight per CTA

template <int K>
__global__ void __launch_bounds__(kFusedWThreads, CHEB_FUSEDW_MIN_CTAS)
cheb_step2w_kernel(StepArgs a, FusedArgs f, FusedDynArgs dy) {
    using G = Geo<K>;
    using SL = StageLayout<K, MODE_CSR>;
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NS = kWStages;
    __shared__ __align__(8) uint64_t full[NS], empty[NS];
    __shared__ int64_t s_base_c[NS], s_base_v[NS], s_t[NS];
    __shared__ int s_fit[NS], s_stg[NS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double acc[2][kPPL];  // stage 1 / stage 2 moments (compute warps)
#pragma unroll
    for (int q = 0; q < kPPL; q++) acc[0][q] = acc[1][q] = 0.0;
    if (tid == 0) {
        for (int x = 0; x < NS; x++) {
            mbar_init(&full[x], 1);
            mbar_init(&empty[x], kThreads / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kThreads / 32) {
        // ------------------------------------------------------------------ producer warp
        const int64_t nchunks = (a.ntiles + kChunkTiles - 1) / kChunkTiles;
        const unsigned int ntl = (unsigned int)a.ntiles;
        // Ticket policy of cheb_step2d_kernel, split so the atomic for item q+1 is issued one item
        // ahead and only examined in the next iteration (it overlaps this item's bound loads, TMA
        // issue and dependency wait).  lane 0 state:
        bool want2 = false, done1 = false, done2 = false;
        auto choose = [&]() -> int {  // counter of the next ticket: 1, 2, or 0 (none left)
            if ((want2 || done1) && !done2) {
                want2 = false;
                return 2;
            }
            if (!done1) return 1;
            return done2 ? 0 : 2;
        };
        auto draw = [&](int ctr) -> unsigned int { return ctr == 1 ? atomicAdd(dy.c1, 1u) : ctr == 2 ? atomicAdd(dy.c2, 1u) : 0u; };
        // classify a drawn ticket (falling back to the other counter when one is exhausted)
        auto resolve = [&](int ctr, unsigned int raw, int& stg, int64_t& t) -> bool {
            for (;;) {
                if (ctr == 0) return false;
                if (raw < ntl) {
                    stg = ctr == 2 ? 1 : 0;
                    t = raw;
                    if (ctr == 1) want2 = (int64_t)raw >= f.D;
                    return true;
                }
                if (ctr == 1) done1 = true;
                else done2 = true;
                ctr = choose();
                raw = draw(ctr);
            }
        };
        int64_t pf_bw = -1;  // lane 0: bandwidth for the L2 prefetch (banded operators only)
        if (CHEB_L2_PREFETCH && lane == 0 && a.bw) {
            const int64_t bwv = (int64_t)*a.bw;
            pf_bw = (4 * bwv < a.d) ? bwv : -1;
        }
        int64_t known = 0;
        int64_t prev_t[NS], pend[NS];  // pend: item in buffer x whose completion is not yet observed
        int prev_stg[NS];
        for (int x = 0; x < NS; x++) {
            prev_t[x] = -1;
            pend[x] = -1;
            prev_stg[x] = 1;
        }
        // Publish finished stage-1 tiles as soon as the compute warps release them -- also while
        // this warp spins on a dependency, so a wait never holds back this CTA's own finished
        // tiles (else two CTAs could wait on each other's unpublished tiles).
        auto retire = [&](int x, bool block) {
            if (pend[x] < 0) return;
            const uint32_t ph = (uint32_t)((pend[x] / NS) & 1);
            if (block) mbar_wait(&empty[x], ph);
            else if (!mbar_test(&empty[x], ph)) return;
            if (lane == 0 && prev_stg[x] == 0) red_release_add(f.cnt + prev_t[x] / kChunkTiles, 1u);
            pend[x] = -1;
        };
        int ctr_n = 0;          // lane 0: counter and raw value of the ticket drawn for the next item
        unsigned int raw_n = 0;
        if (lane == 0) {
            ctr_n = choose();
            raw_n = draw(ctr_n);
        }
        int64_t q = 0;
        for (;; ++q) {
            const int b = (int)(q % NS);
            int stg = 0;
            int64_t t = -1, e0 = 0, e1 = 0;
            bool ok = false;
            if (lane == 0) {
                ok = resolve(ctr_n, raw_n, stg, t);
                if (ok) {  // bound loads of this item, then the next ticket: both in flight below
                    const int64_t r0 = t * G::TILE;
                    e0 = __ldg(a.rp + r0);
                    e1 = __ldg(a.rp + imin64(r0 + G::TILE, a.d));
                    ctr_n = choose();
                    raw_n = draw(ctr_n);
                }
            }
            for (int x = 0; x < NS; x++)
                if (x != b) retire(x, false);
            retire(b, true);  // buffer b is free once the compute warps are done with item q-NS
            ok = __shfl_sync(0xffffffffu, ok, 0);
            if (!ok) {
                if (lane == 0) {
                    s_t[b] = -1;
                    mbar_arrive(&full[b]);
                }
                break;
            }
            stg = __shfl_sync(0xffffffffu, stg, 0);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (lane == 0) {
                unsigned char* st = smem + b * SL::BYTES;
                const int64_t r0 = t * G::TILE;
                const int rows = (int)imin64((int64_t)G::TILE, a.d - r0);
                const int64_t c0 = e0 & ~int64_t(3), c1 = (e1 + 3) & ~int64_t(3);
                const int64_t v0 = e0 & ~int64_t(1), v1 = (e1 + 1) & ~int64_t(1);
                const bool fit = (c1 - c0) <= G::CAP + 8 && (v1 - v0) <= G::CAP + 4;
                s_fit[b] = fit;
                s_base_c[b] = c0;
                s_base_v[b] = v0;
                s_t[b] = t;
                s_stg[b] = stg;
                const double* wsrc = stg ? f.B : f.A;
                const uint32_t wbytes = (uint32_t)rows * K * 8;
                const uint32_t sgbytes = ((uint32_t)rows * G::WORDS * 4 + 15) & ~15u;
                uint32_t bytes = G::RPBYTES + sgbytes + wbytes;
                if (fit) bytes += (uint32_t)(c1 - c0) * 4 + (uint32_t)(v1 - v0) * 8;
                mbar_expect_tx_only(&full[b], bytes);
                bulk_g2s(st + SL::OFF_RP, a.rp + r0, G::RPBYTES, &full[b]);
                bulk_g2s(st + SL::OFF_SGN, a.sbits + (size_t)r0 * G::WORDS, sgbytes, &full[b]);
                bulk_g2s_hint(st + SL::OFF_WPREV, wsrc + (size_t)r0 * K, wbytes, &full[b], policy_evict_first());
                if (fit) {
                    bulk_g2s(st + SL::OFF_COL, a.ci + c0, (uint32_t)(c1 - c0) * 4, &full[b]);
                    bulk_g2s(st + SL::OFF_VAL, a.va + v0, (uint32_t)(v1 - v0) * 8, &full[b]);
                }
                if (CHEB_L2_PREFETCH && stg == 0 && pf_bw >= 0) {  // stage-1 first-touch rows of w_j
                    const int64_t p0 = r0 + pf_bw, p1 = imin64(p0 + rows, a.d);
                    if (p1 > p0) prefetch_l2(f.B + (size_t)p0 * K, (uint32_t)(p1 - p0) * K * 8);
                }
            }
            if (stg == 1) {  // stage-1 tiles [0, need) must be complete before the gathers
                const int64_t need = imin64(t + f.H + 1, a.ntiles);
                uint32_t spins = 0;
                while (known * kChunkTiles < need) {
                    const int64_t ch = known + lane;
                    const unsigned int v = ch < nchunks ? ld_relaxed_u32(f.cnt + ch) : 0u;
                    const bool fullc = ch >= nchunks || v >= (unsigned int)imin64(kChunkTiles, a.ntiles - ch * kChunkTiles);
                    const unsigned int notfull = __ballot_sync(0xffffffffu, !fullc);
                    const int adv = notfull ? __ffs(notfull) - 1 : 32;
                    known += adv;
                    if (adv == 0) {
                        for (int x = 0; x < NS; x++)
                            if (x != b) retire(x, false);  // keep publishing while waiting
                        __nanosleep(64);
                        if ((++spins & 1023u) == 0 && (spins > (1u << 23) || ld_acquire_u32(f.err))) {
                            if (lane == 0) atomicExch(f.err, 1u);  // ~seconds without progress: never hang
                            break;
                        }
                    }
                }
#if CHEB_FUSED_FENCE
                fence_acq_rel_gpu();
#endif
            }
            __syncwarp();
            prev_t[b] = t;
            prev_stg[b] = stg;
            pend[b] = q;
            if (lane == 0) mbar_arrive(&full[b]);  // release.cta: the smem metadata above
        }
        for (int x = 0; x < NS; x++) retire(x, true);  // the last items may still be computing
    } else {
        // ------------------------------------------------------------------ compute warps
        double2 z2[G::NSL];
#pragma unroll
        for (int sl = 0; sl < G::NSL; sl++) z2[sl] = make_double2(0.0, 0.0);
        double (&mu1)[1][kPPL] = *reinterpret_cast<double(*)[1][kPPL]>(&acc[0]);
        double (&mu2)[1][kPPL] = *reinterpret_cast<double(*)[1][kPPL]>(&acc[1]);
        for (int64_t q = 0;; ++q) {
            const int b = (int)(q % NS);
            mbar_wait(&full[b], (uint32_t)((q / NS) & 1));
            const int64_t t = s_t[b];
            if (t < 0) break;
            const int stg = s_stg[b];
            const unsigned char* st = smem + b * SL::BYTES;
            const int64_t r0 = t * G::TILE;
            const int rows = (int)imin64((int64_t)G::TILE, a.d - r0);
            if (stg == 0) {
                if (s_fit[b])
                    step_tile<K, MODE_CSR, false, true, false, true>(a, st, r0, rows, s_base_c[b], s_base_v[b], z2,
                                                                     mu1, f.B, f.B, f.A);
                else
                    step_tile<K, MODE_CSR, false, false, false, true>(a, st, r0, rows, 0, 0, z2, mu1, f.B, f.B,
                                                                      f.A);
            } else {
                if (s_fit[b])
                    step_tile<K, MODE_CSR, false, true, true, false>(a, st, r0, rows, s_base_c[b], s_base_v[b], z2,
                                                                     mu2, f.A, f.A, f.B);
                else
                    step_tile<K, MODE_CSR, false, false, true, false>(a, st, r0, rows, 0, 0, z2, mu2, f.A, f.A,
                                                                      f.B);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[b]);  // release.cta: this warp's stores and smem reads
        }
    }
    __syncthreads();  // all warps out of the loops; the stage buffers become the reduction scratch
    grid_reduce_finish<K, kPPL, 2, EPI_PAIR, false, true>(acc, a, smem);
}

// ---------------------------------------------------------------------------------------
// K2p: persistent multi-step kernel for small / L2-resident operators (csr, rank-1).
// One cooperative launch runs steps j = 1..n of a probe block: each step walks the same
// static tile schedule as cheb_step_kernel (tile t on CTA t mod G, same staged pipeline) and
// writes per-CTA partial dot products; CTAs then arrive at a grid barrier (monotone
// counter: step j is complete when it reaches j*G).  Before waiting, each CTA already issues
// the TMA copies of its first tiles of step j+1 (W_prev = w_{j-1} and the matrix are final),
// so the barrier latency overlaps the next step's staging.  After the barrier every CTA
// reduces the rank-1 partials itself (s_j = u^T w_j, same fixed order everywhere) and CTA 0
// reduces mu_j, in the order grid_reduce_finish uses: moments are bit-identical to per-step
// launches with the same grid.  Removes the n launch/drain gaps that dominate when one step
// is a few microseconds of L2 traffic.
// ---------------------------------------------------------------------------------------
struct PersistArgs {
    double* w0;               // holds v (from probe_init) at entry
    double* w1;
    int32_t n;                // degree
    double* part;             // [2][NCH][gridDim.x][K] partials (double-buffered by step parity)
    double* s_buf;            // [2][K] s_j by step parity (s_0 from probe_init in s_buf[0])
    unsigned int* bar_count;  // grid barrier arrivals (zeroed; monotone)
    unsigned int* s_count;    // rank-1: probes whose s_j is published (zeroed; monotone)
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
    __shared__ double wbuf[kThreads / 32];
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
            const int p = 2 * lg + sl * G::SS;
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
                    step_tile<K, MODE, true, true, true, false, DBL, false, R4>(a, st, r0, rows, s_base_c[b], s_base_v[b], r1,
                                                                     acc, cur, cur, nxt);
                else
                    step_tile<K, MODE, true, false, true, false, DBL, false, R4>(a, st, r0, rows, 0, 0, r1, acc, cur, cur,
                                                                      nxt);
            } else {
                if (s_fit[b])
                    step_tile<K, MODE, false, true, true, false, DBL, false, R4>(a, st, r0, rows, s_base_c[b], s_base_v[b], r1,
                                                                      acc, cur, cur, nxt);
                else
                    step_tile<K, MODE, false, false, true, false, DBL, false, R4>(a, st, r0, rows, 0, 0, r1, acc, cur, cur,
                                                                       nxt);
            }
            __syncthreads();
            if (tid == 0 && it + 2 < nmine) issue(j, it + 2, b);
        }
        // ---- per-CTA partials (same tree as grid_reduce_finish)
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
                const int p = probe_of<K, kPPL, true>(lg, q);
#pragma unroll
                for (int ch = 0; ch < NCH; ch++) red[ch][warp][p] = acc[ch][q];
            }
        }
        __syncthreads();
        double* part = pa_.part + (size_t)(j & 1) * NCH * gridDim.x * K;  // [NCH][G][K] of step j
        if (tid < K) {
#pragma unroll
            for (int ch = 0; ch < NCH; ch++) {
                double m = 0.0;
#pragma unroll
                for (int w = 0; w < kThreads / 32; w++) m += red[ch][w][tid];
                part[((size_t)ch * gridDim.x + blockIdx.x) * K + tid] = m;
            }
        }
        // ---- grid barrier, split: arrive, stage step j+1, wait
        __syncthreads();
        if (tid == 0) {
            red_release_add(pa_.bar_count, 1u);  // release: the CTA's stores of step j (barrier above)
            if (j < pa_.n) {
                // w_{j-1} (W_prev of step j+1) and the matrix are final: stage ahead.  The
                // proxy fence orders other CTAs' generic stores of w_{j-1} (step j-1, already
                // behind the previous barrier) before these async-proxy reads.
                asm volatile("fence.proxy.async.global;" ::: "memory");
                for (int64_t i = 0; i < 2 && i < nmine; i++) issue(j + 1, i, (int)i);  // stages are all consumed
            }
            spin_until_geq(pa_.bar_count, (unsigned int)j * gridDim.x, pa_.err);  // + acquire (L1 invalidated)
        }
        __syncthreads();
        // ---- canonical reductions of step j's partials: CTA c owns probes c, c+G, ...
        // rank-1: s_j = u^T w_j gates the next step, so it is reduced and published first; the
        // moments follow off the critical path (the parity-double-buffered partials of step j are
        // next overwritten in step j+2, which starts after this CTA publishes s_{j+1})
        if (HAS_S) {
            for (int p = blockIdx.x; p < K; p += gridDim.x) {
                const double sv = reduce_partials_one(part + (size_t)(NCH - 1) * gridDim.x * K, K, (int)gridDim.x, p, wbuf);
                if (tid == 0) pa_.s_buf[(j & 1) * K + p] = sv;
            }
            if (tid == 0) {
                const unsigned int mine = blockIdx.x < K ? (K - 1 - blockIdx.x) / gridDim.x + 1 : 0;
                if (mine) red_release_add(pa_.s_count, mine);
            }
        }
        for (int p = blockIdx.x; p < K; p += gridDim.x) {
            double v[NCH];
#pragma unroll
            for (int ch = 0; ch < (HAS_S ? NCH - 1 : NCH); ch++)
                v[ch] = reduce_partials_one(part + (size_t)ch * gridDim.x * K, K, (int)gridDim.x, p, wbuf);
            if (tid == 0 && p < a.kvalid) {
                double* row = a.mu_out + (size_t)p * a.mu_stride;
                if (DBL) dbl_write(row, j, a.mu_stride - 1, v[0], v[1]);
                else row[j] = v[0];
            }
        }
        if (HAS_S) {
            if (tid == 0) spin_until_geq(pa_.s_count, (unsigned int)j * K, pa_.err);  // every s_j published
            __syncthreads();
            if (tid < K) s_sh[tid] = __ldcg(pa_.s_buf + (j & 1) * K + tid);
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------------------
// Gather-staged step (opt-in, CSR): per tile of T = 1024/K rows, the sorted unique rows of W_cur the
// tile's nonzeros reference ("gather list", at most S = 4096/K rows) are fetched into shared memory
// by TMA tile::gather4 (4 rows per instruction); every nonzero carries a 16-bit slot into that
// list instead of its column, so the compute warps read their neighbours from shared memory.
// ---------------------------------------------------------------------------------------
#ifndef CHEB_GS_LIST
#define CHEB_GS_LIST 3328  // gather-list capacity x k: 52 rows at k = 64 (5-point stencil tiles need 50)
#endif
__host__ __device__ constexpr int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

template <int K>
struct GsGeo {
    static_assert(K >= 16, "gather-staged kernels: K >= 16");
    static constexpr int T = 1024 / K;        // rows per tile (one row per lane group of 256 threads)
    static constexpr int S = (CHEB_GS_LIST / K) & ~3;  // gather-list capacity (rows, multiple of 4)
    static constexpr int CAPV = T * 8;        // staged nonzeros per tile (padded CSR)
    static constexpr int WORDS = words_for(K);
    static constexpr int OFF_GATH = 0;
    static constexpr int OFF_WPREV = OFF_GATH + S * K * 8;
    static constexpr int OFF_VAL = OFF_WPREV + T * K * 8;
    static constexpr int OFF_SL = OFF_VAL + (CAPV + 4) * 8;
    static constexpr int OFF_RP = OFF_SL + ((CAPV + 16) * 2 + 15) / 16 * 16;
    static constexpr int OFF_SGN = OFF_RP + (T + 2) * 8;
    static constexpr int BYTES = (OFF_SGN + ((T * WORDS * 4 + 15) / 16) * 16 + 1023) / 1024 * 1024;  // TMA dst alignment
};

// One warp per tile: sort the tile's (padded) columns in shared memory (bitonic), compact the
// unique ones into gl[t*S ..], pad the list to a multiple of 4 with its last row, and write each
// nonzero's slot (lower_bound in the list).  Tiles with more than CAPV nonzeros or S unique rows
// set *ovf (the host then keeps the regular kernels for this operator).
template <int K>
__global__ void __launch_bounds__(kThreads)
gather_list_kernel(int64_t d, int64_t ntiles, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                   int32_t* __restrict__ gl, int32_t* __restrict__ gl_len, uint16_t* __restrict__ sl,
                   unsigned int* __restrict__ ovf) {
    using GG = GsGeo<K>;
    constexpr int C2 = next_pow2(GG::CAPV);
    __shared__ int32_t buf[kThreads / 32][C2];
    __shared__ int32_t uq[kThreads / 32][GG::S + 4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t t = (int64_t)blockIdx.x * (kThreads / 32) + warp; t < ntiles; t += (int64_t)gridDim.x * (kThreads / 32)) {
        const int64_t r0 = t * GG::T;
        const int64_t r1 = imin64(r0 + GG::T, d);
        const int64_t e0 = rp[r0], e1 = rp[r1];
        const int n = (int)(e1 - e0);
        if (n > GG::CAPV) {
            if (lane == 0) {
                gl_len[t] = -1;
                atomicOr(ovf, 1u);
            }
            continue;
        }
        int32_t* b = buf[warp];
        for (int x = lane; x < C2; x += 32) b[x] = x < n ? ci[e0 + x] : 0x7fffffff;
        __syncwarp();
        int np = 1;
        while (np < n) np <<= 1;
        for (int k2 = 2; k2 <= np; k2 <<= 1)
            for (int j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
                for (int x = lane; x < np; x += 32) {
                    const int y = x ^ j2;
                    if (y > x) {
                        const bool up = (x & k2) == 0;
                        const int32_t bx = b[x], by = b[y];
                        if ((bx > by) == up) {
                            b[x] = by;
                            b[y] = bx;
                        }
                    }
                }
                __syncwarp();
            }
        // compact the unique values (warp ballot prefix per 32-chunk)
        int u = 0;
        for (int base = 0; base < np; base += 32) {
            const int x = base + lane;
            const bool keep = x < n && (x == 0 || b[x] != b[x - 1]);
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            const int pos = u + __popc(m & ((1u << lane) - 1u));
            if (keep && pos < GG::S) uq[warp][pos] = b[x];
            u += __popc(m);
        }
        __syncwarp();
        if (u > GG::S) {
            if (lane == 0) {
                gl_len[t] = -1;
                atomicOr(ovf, 1u);
            }
            continue;
        }
        const int u4 = n == 0 ? 0 : (u + 3) & ~3;
        for (int x = lane; x < u4; x += 32) gl[t * GG::S + x] = uq[warp][x < u ? x : u - 1];
        if (lane == 0) gl_len[t] = u4;
        for (int x = lane; x < n; x += 32) {  // slot of each nonzero: lower_bound in uq
            const int32_t c = ci[e0 + x];
            int lo = 0, hi = u;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (uq[warp][mid] < c) lo = mid + 1;
                else hi = mid;
            }
            sl[e0 + x] = (uint16_t)lo;
        }
        __syncwarp();
    }
}

struct GsArgs {
    const int32_t* gl;      // [ntiles][S] gather rows of each tile (multiple of 4 used)
    const int32_t* gl_len;  // [ntiles] used entries of gl (multiple of 4)
    const uint16_t* sl;     // [padded nnz] slot of each nonzero in its tile's gather list
    int64_t ntiles;         // tiles of GsGeo<K>::T rows
    unsigned int* err;      // wait-timeout flag (never hang)
};

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tmap, int32_t col, int4 rows,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(col), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w),
        "r"(smem_u32(bar))
        : "memory");
}

// Gather-staged fused Chebyshev step (CSR, Algorithm 1).  Warps 0..7 compute (one row per lane
// group, T rows per tile), warp 8 stages tiles: gather list + row bounds (one warp-wide load),
// expect_tx, then every lane issues its own gather4 of 4 list rows, lane 0 the bulk copies of
// W_prev, the tile's values / slots, row pointers and sign words; NS-deep pipeline with
// full/empty mbarriers.  Static tile -> CTA map (t = c + i*G) and per-CTA partial sums: moments are
// deterministic.  The gather source W_cur is described by a 2D tensor map [d][K] fp64, box {K, 1}.
#ifndef CHEB_GS_STAGES
#define CHEB_GS_STAGES 3
#endif
template <int K, bool FIRST>
__global__ void __launch_bounds__(kThreads + 32, 2)
cheb_step_gs_kernel(StepArgs a, GsArgs g, const __grid_constant__ CUtensorMap tmap) {
    using GG = GsGeo<K>;
    using G = Geo<K>;
    constexpr int NS = CHEB_GS_STAGES;
    static_assert(G::GROUPS == GG::T, "one row per lane group");
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[NS], empty[NS];
    __shared__ int64_t s_v0[NS], s_s0[NS], s_e0[NS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nmine = g.ntiles > blockIdx.x ? (g.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    double acc[1][kPPL];
#pragma unroll
    for (int q = 0; q < kPPL; q++) acc[0][q] = 0.0;
    if (tid == 0) {
        for (int x = 0; x < NS; x++) {
            mbar_init(&full[x], 1);
            mbar_init(&empty[x], kThreads / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kThreads / 32) {
        // ------------------------------------------------------------------ producer warp
        // metadata of a tile (list length, the list, row bounds): all loads issued together and
        // one tile ahead, so their latency overlaps the current tile's staging
        constexpr int LPL = (GG::S / 4 + 31) / 32;  // int4 list chunks per lane
        struct Meta {
            int len;
            int4 gr[LPL];
            int64_t e0, e1;
        };
        auto load_meta = [&](int64_t t, Meta& m) {
            const int64_t r0 = t * GG::T;
            const int rows = (int)imin64((int64_t)GG::T, a.d - r0);
            m.len = __ldg(g.gl_len + t);
#pragma unroll
            for (int c = 0; c < LPL; c++) {
                const int x = lane + 32 * c;
                m.gr[c] = x < GG::S / 4 ? __ldg(reinterpret_cast<const int4*>(g.gl + t * GG::S) + x) : make_int4(0, 0, 0, 0);
            }
            m.e0 = __ldg(a.rp + r0);
            m.e1 = __ldg(a.rp + r0 + rows);
        };
        Meta cur, nxt;
        if (nmine > 0) load_meta(blockIdx.x, nxt);
        for (int64_t it = 0; it < nmine; it++) {
            const int b = (int)(it % NS);
            cur = nxt;
            if (it + 1 < nmine) load_meta((int64_t)blockIdx.x + (it + 1) * gridDim.x, nxt);
            if (it >= NS) mbar_wait_bounded(&empty[b], (uint32_t)(((it / NS) - 1) & 1), g.err);
            const int64_t t = (int64_t)blockIdx.x + it * gridDim.x;
            const int64_t r0 = t * GG::T;
            const int rows = (int)imin64((int64_t)GG::T, a.d - r0);
            const int len = cur.len;  // multiple of 4, <= S
            unsigned char* st = smem + b * GG::BYTES;
            if (lane == 0) {
                const int64_t e0 = cur.e0, e1 = cur.e1;
                const int64_t v0 = e0 & ~int64_t(1), v1 = (e1 + 1) & ~int64_t(1);
                const int64_t s0 = e0 & ~int64_t(7), s1 = (e1 + 7) & ~int64_t(7);
                s_v0[b] = v0;
                s_s0[b] = s0;
                s_e0[b] = e0;
                const uint32_t wbytes = (uint32_t)rows * K * 8;
                const uint32_t sgbytes = ((uint32_t)rows * GG::WORDS * 4 + 15) & ~15u;
                uint32_t bytes = (uint32_t)len * K * 8 + (uint32_t)(GG::T + 2) * 8 + sgbytes +
                                 (uint32_t)(v1 - v0) * 8 + (uint32_t)(s1 - s0) * 2;
                if (!FIRST) bytes += wbytes;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[b])),
                             "r"(bytes)
                             : "memory");
                bulk_g2s(st + GG::OFF_RP, a.rp + r0, (GG::T + 2) * 8, &full[b]);
                bulk_g2s(st + GG::OFF_SGN, a.sbits + (size_t)r0 * GG::WORDS, sgbytes, &full[b]);
                if (!FIRST)
                    bulk_g2s_hint(st + GG::OFF_WPREV, a.wnext + (size_t)r0 * K, wbytes, &full[b], policy_evict_first());
                bulk_g2s(st + GG::OFF_VAL, a.va + v0, (uint32_t)(v1 - v0) * 8, &full[b]);
                bulk_g2s(st + GG::OFF_SL, g.sl + s0, (uint32_t)(s1 - s0) * 2, &full[b]);
            }
            __syncwarp();
#pragma unroll
            for (int c = 0; c < LPL; c++) {  // every 4-row chunk of the list: one gather4
                const int x = lane + 32 * c;
                if (4 * x < len) tma_gather4(st + GG::OFF_GATH + (size_t)x * 4 * K * 8, &tmap, 0, cur.gr[c], &full[b]);
            }
        }
    } else {
        // ------------------------------------------------------------------ compute warps
        const int lg = tid % G::L, grp = tid / G::L;
        int pp[G::NSL];
#pragma unroll
        for (int sl = 0; sl < G::NSL; sl++) pp[sl] = 2 * lg + sl * G::SS;
        for (int64_t it = 0; it < nmine; it++) {
            const int b = (int)(it % NS);
            mbar_wait_bounded(&full[b], (uint32_t)((it / NS) & 1), g.err);
            const unsigned char* st = smem + b * GG::BYTES;
            const int64_t t = (int64_t)blockIdx.x + it * gridDim.x;
            const int64_t r0 = t * GG::T;
            const int rows = (int)imin64((int64_t)GG::T, a.d - r0);
            const int lr = grp;
            if (lr < rows) {
                const int64_t i = r0 + lr;
                const int64_t* rp_s = reinterpret_cast<const int64_t*>(st + GG::OFF_RP);
                const double* val_s = reinterpret_cast<const double*>(st + GG::OFF_VAL);
                const uint16_t* sl_s = reinterpret_cast<const uint16_t*>(st + GG::OFF_SL);
                const double* gath = reinterpret_cast<const double*>(st + GG::OFF_GATH);
                const double* wp_s = reinterpret_cast<const double*>(st + GG::OFF_WPREV);
                const uint32_t* sg_s = reinterpret_cast<const uint32_t*>(st + GG::OFF_SGN);
                const int ov = (int)(rp_s[lr] - s_v0[b]), os = (int)(rp_s[lr] - s_s0[b]);
                const int nr = (int)(rp_s[lr + 1] - rp_s[lr]);
                double2 g2[G::NSL];
#pragma unroll
                for (int sl = 0; sl < G::NSL; sl++) g2[sl] = make_double2(0.0, 0.0);
                for (int t0 = 0; t0 < nr; t0 += CHEB_NNZ_UNROLL) {
#pragma unroll
                    for (int q = 0; q < CHEB_NNZ_UNROLL; q++) {
                        const double v = val_s[ov + t0 + q];
                        const double* xr = gath + (int)sl_s[os + t0 + q] * K;
#pragma unroll
                        for (int sl = 0; sl < G::NSL; sl++) {
                            const double2 x = *reinterpret_cast<const double2*>(xr + pp[sl]);
                            g2[sl].x = fma(v, x.x, g2[sl].x);
                            g2[sl].y = fma(v, x.y, g2[sl].y);
                        }
                    }
                }
                double* out = a.wnext + (size_t)i * K;
#pragma unroll
                for (int sl = 0; sl < G::NSL; sl++) {
                    double2 nw = g2[sl];
                    if (!FIRST) {
                        const double2 pv = *reinterpret_cast<const double2*>(wp_s + lr * K + pp[sl]);
                        nw = make_double2(fma(2.0, g2[sl].x, -pv.x), fma(2.0, g2[sl].y, -pv.y));
                    }
                    __stcs(reinterpret_cast<double2*>(out + pp[sl]), nw);
                    const uint32_t bits = sg_s[lr * GG::WORDS + (pp[sl] >> 5)] >> (pp[sl] & 31);
                    acc[0][2 * sl] += signflip(nw.x, bits << 31);
                    acc[0][2 * sl + 1] += signflip(nw.y, bits << 30);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[b]);
        }
    }
    __syncthreads();  // stage buffers become the reduction scratch
    grid_reduce_finish<K, kPPL, 1, EPI_STEP, false, true>(acc, a, smem);
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
__global__ void __launch_bounds__(kThreads)
quadform_kernel(int64_t d, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                const double* __restrict__ va, const double* __restrict__ x, double* __restrict__ part) {
    __shared__ double wsum[kThreads / 32];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
         i += (int64_t)gridDim.x * blockDim.x) {
        double r = 0.0;
        for (int64_t e = rp[i]; e < rp[i + 1]; e++) r = fma(va[e], x[ci[e]], r);
        acc = fma(x[i], r, acc);
    }
    acc = warp_sum_xor(acc);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; w++) t += wsum[w];
        part[blockIdx.x] = t;
    }
}

__global__ void quadform_final_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int c = 0; c < n; c++) t += part[c];
        *out = t;
    }
}

// Gershgorin-type upper bound on lambda_max of a CSR operator: out[0] <- max_i sum_j |a_ij|,
// out[1] <- max_i |u_i| (rank-1 u, if given).  Ordered-key atomics (order-independent).
// out[2] <- min_i (a_ii - sum_{j != i} |a_ij|) (Gershgorin lower end; ordered-key min).
__global__ void __launch_bounds__(kThreads)
gershgorin_kernel(int64_t d, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                  const double* __restrict__ va, const double* __restrict__ u, unsigned long long* out) {
    double rmax = 0.0, umax = 0.0, lmin = INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
         i += (int64_t)gridDim.x * blockDim.x) {
        double r = 0.0, off = 0.0, dg = 0.0;
        for (int64_t e = rp[i]; e < rp[i + 1]; e++) {
            const double x = fabs(va[e]);
            r += x;
            if (ci[e] == i) dg = va[e]; else off += x;
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
