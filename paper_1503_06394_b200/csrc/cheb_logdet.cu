// cheb_logdet.cu -- host side of the C ABI (include/cheb_logdet.h): validation,
// fp64 coefficient routine, workspace planning, stream-ordered launch sequence,
// kernel accounting.  Device kernels live in cheb_kernels.cuh.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "cheb_logdet.h"
#include "cheb_kernels.cuh"

using namespace chebld;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CL_CUDA(call)                                                                 \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(CL_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                        __FILE__, __LINE__);                                          \
    } while (0)

// ---- step-kernel profiling (CUDA events on the launching stream) ------------
struct Profiler {
    std::mutex mu;
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[3];  // [0] single step, [1] fused pair,
                                                               // [2] persistent (all n steps)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
    double ms[3] = {0.0, 0.0, 0.0};
    int64_t n[3] = {0, 0, 0};
} g_prof;

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}
// schedule controls (process-wide; CHEB_FUSION / CHEB_PERSISTENT env vars set the initial value)
std::atomic<int> g_fusion{env_int("CHEB_FUSION", 1)};  // 1 off (default), 2 auto, 3 forced, 4 forced static
std::atomic<int> g_persistent{env_int("CHEB_PERSISTENT", 1)};  // 0 off, 1 auto (default), 2 forced
std::atomic<int> g_small_tiles{env_int("CHEB_SMALL_TILES", 1)};  // 1 auto (default), 0 standard geometry
std::atomic<int> g_doubling{env_int("CHEB_DOUBLING", 0)};      // 0 off (default), 1 moment doubling
std::atomic<int> g_gather{env_int("CHEB_GATHER", 0)};          // 0 off (default), 1 gather-staged steps

struct ProfScope {
    cudaStream_t s;
    int kind;
    std::pair<cudaEvent_t, cudaEvent_t> pr{nullptr, nullptr};
    explicit ProfScope(cudaStream_t st, int k = 0) : s(st), kind(k) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        if (!g_prof.on) return;
        if (!g_prof.pool.empty()) {
            pr = g_prof.pool.back();
            g_prof.pool.pop_back();
        } else {
            cudaEventCreate(&pr.first);
            cudaEventCreate(&pr.second);
        }
        cudaEventRecord(pr.first, s);
    }
    ~ProfScope() {
        if (!pr.first) return;
        cudaEventRecord(pr.second, s);
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.ev[kind].push_back(pr);
    }
};

int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

constexpr int kMaxCtasPerSm = 8;  // partial buffers are sized for this

struct DevBuf {  // owning device allocation (freed on scope exit)
    void* p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
};

// Grow-only device arenas reused across the synchronous entry points (cheb_logdet,
// cheb_logdet_host) of a host thread: repeated estimates do not pay cudaMalloc/cudaFree of a
// multi-GB workspace every call.  [0]: workspace + result buffers, [1]: the host operator's
// device copy.  cheb_release_cache() frees them.
struct Arena {
    int dev = -1;
    void* p = nullptr;
    size_t cap = 0;
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        dev = -1;
    }
    ~Arena() { release(); }
};
thread_local Arena g_arena[2];

int arena_get(int slot, size_t bytes, void** out) {
    Arena& A = g_arena[slot];
    int dev = 0;
    cudaGetDevice(&dev);
    if (A.p && (A.cap < bytes || A.dev != dev)) A.release();
    if (!A.p) {
        cudaError_t e = cudaMalloc(&A.p, bytes);
        if (e != cudaSuccess) {
            A.p = nullptr;
            return fail(CL_ENOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
        }
        A.cap = bytes;
        A.dev = dev;
    }
    *out = A.p;
    return CL_OK;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

bool valid_k(int k) { return k == 8 || k == 16 || k == 32 || k == 64 || k == 128; }

// rows per tile: Geo<K, R4>::TILE; the workspace is planned for the larger of the two geometries
int tile_rows(int k, int r4 = CHEB_RPG) { return r4 * kThreads * 4 / k; }
int tile_rows_max(int k) { return tile_rows(k, std::max(CHEB_RPG, CHEB_RPG_DBL)); }

struct Layout {
    size_t w0, w1, y, sbits, part, sbuf, ticket;
    size_t rp2, ci2, va2, u2, cnt, misc, cnt64, scan, gl, gl_len, sl, total;
    int64_t gs_ntiles;
    size_t scan_bytes;
    int64_t rp2_len;
};

// Workspace of cheb_moments for dimension d, gather-matrix nnz, probe block k.
Layout plan(int64_t d, int64_t nnz, int k, int kind, int sms) {
    Layout L{};
    size_t off = 0;
    const size_t wbytes = align256((size_t)d * k * sizeof(double));
    const int words = k >= 32 ? k / 32 : 1;
    const size_t maxgrid = (size_t)sms * kMaxCtasPerSm;
    const int64_t ntiles = (d + tile_rows_max(k) - 1) / tile_rows_max(k);
    L.w0 = off; off += wbytes;
    L.w1 = off; off += wbytes;
    L.y = off; if (kind == CL_OP_BTB) off += wbytes;
    L.sbits = off; off += align256((size_t)d * words * sizeof(uint32_t) + 16);
    // per-CTA partials: up to 3 channels (doubling + rank-1) x 2 step parities (persistent kernel)
    L.part = off; off += align256(6 * maxgrid * k * sizeof(double));
    L.sbuf = off; off += align256(2 * (size_t)k * sizeof(double));
    L.ticket = off; off += 256;
    L.rp2_len = ntiles * tile_rows_max(k) + 2;
    L.rp2 = off; off += align256((size_t)L.rp2_len * sizeof(int64_t));
    // rows padded to a multiple of the gather chunk: at most (U - 1) extra entries per row
    // (a row with no stored diagonal gets one extra (i, -beta) entry: at most U more per row)
    const size_t pnnz = (size_t)nnz + (size_t)CHEB_NNZ_UNROLL * (size_t)d;
    L.ci2 = off; off += align256((pnnz + 8) * sizeof(int32_t));
    L.va2 = off; off += align256((pnnz + 4) * sizeof(double));
    L.cnt64 = off; off += align256(((size_t)d + 1) * sizeof(int64_t));  // padded row lengths
    L.scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, L.scan_bytes, (const int64_t*)nullptr, (int64_t*)nullptr, (int)(d + 1));
    L.scan = off; off += align256(L.scan_bytes);
    L.u2 = off; if (kind == CL_OP_CSR_RANK1) off += align256(((size_t)d + 2) * sizeof(double));
    L.cnt = off; off += align256(((size_t)ntiles + 64) * sizeof(unsigned int));  // fused wave counters
    // gather-staged kernels (csr, k >= 16): per-tile gather lists and per-nonzero slots
    L.gs_ntiles = 0;
    L.gl = L.gl_len = L.sl = off;
    if (kind == CL_OP_CSR && k >= 16) {
        const int T = 1024 / k, S = (CHEB_GS_LIST / k) & ~3;
        L.gs_ntiles = (d + T - 1) / T;
        L.gl = off; off += align256((size_t)L.gs_ntiles * S * sizeof(int32_t));
        L.gl_len = off; off += align256((size_t)L.gs_ntiles * sizeof(int32_t));
        L.sl = off; off += align256((pnnz + 16) * sizeof(uint16_t));
    }
    L.misc = off; off += 256;  // [0] u64 bandwidth, [8] u32 wait-timeout flag, [16] barrier count,
                               // [20] barrier generation, [24] rank-1 s_ready
    L.total = off;
    return L;
}

int64_t gather_nnz(const cl_operator* op) { return op->kind == CL_OP_BTB ? op->At.nnz : op->A.nnz; }

int check_csr(const cl_csr& A, const char* name) {
    if (A.n_rows < 0 || A.n_cols < 0 || A.nnz < 0)
        return fail(CL_EINVAL, "%s: negative dimension", name);
    if (A.n_rows > 0 && (!A.row_ptr || (A.nnz > 0 && (!A.col_idx || !A.val))))
        return fail(CL_EINVAL, "%s: NULL pointer", name);
    if (A.n_cols >= (int64_t(1) << 31) || A.n_rows >= (int64_t(1) << 31))
        return fail(CL_EDIM, "%s: dimension >= 2^31 (int32 column indices)", name);
    return CL_OK;
}

int check_op(const cl_operator* op) {
    if (!op) return fail(CL_EINVAL, "operator is NULL");
    if (op->kind != CL_OP_CSR && op->kind != CL_OP_CSR_RANK1 && op->kind != CL_OP_BTB)
        return fail(CL_EINVAL, "unknown operator kind %d", op->kind);
    int rc = check_csr(op->A, "A");
    if (rc) return rc;
    if (op->A.n_rows == 0) return fail(CL_EDIM, "empty operator (d = 0)");
    if (op->A.n_rows != op->A.n_cols) return fail(CL_EDIM, "A must be square (%lld x %lld)",
                                                  (long long)op->A.n_rows, (long long)op->A.n_cols);
    if (op->kind == CL_OP_BTB) {
        if ((rc = check_csr(op->At, "At"))) return rc;
        if (op->At.n_rows != op->A.n_cols || op->At.n_cols != op->A.n_rows || op->At.nnz != op->A.nnz)
            return fail(CL_EDIM, "At is not shaped as the transpose of B");
    }
    if (op->kind == CL_OP_CSR_RANK1 && !std::isfinite(op->r1_c))
        return fail(CL_EINVAL, "rank-1 weight is not finite");
    return CL_OK;
}

int check_ab(double a, double b, int32_t degree) {
    if (!std::isfinite(a) || !std::isfinite(b) || !(a > 0.0) || !(b > a))
        return fail(CL_EINVAL, "need finite 0 < a < b (got a=%g b=%g)", a, b);
    if (degree < 0) return fail(CL_EINVAL, "degree < 0");
    return CL_OK;
}

// Tiles per CTA below which a step-kernel grid is shrunk (small operators: fewer CTAs mean a
// deeper per-CTA pipeline and cheaper grid-wide reductions/barriers).  CHEB_MIN_TILES tunes it.
int min_tiles_per_cta() {
    static int v = [] {
        const char* e = getenv("CHEB_MIN_TILES");
        const int x = e ? atoi(e) : 1;
        return x < 1 ? 1 : x;
    }();
    return v;
}

// Cap on resident CTAs per SM for the staged step kernels (CHEB_STEP_OCC; 0 = occupancy limit).
int step_occ_cap() {
    static int v = [] {
        const char* e = getenv("CHEB_STEP_OCC");
        return e ? atoi(e) : 0;
    }();
    return v;
}

template <typename Kern>
int grid_for(Kern kern, int64_t ntiles, int sms, size_t dyn_smem = 0) {
    int occ = 0;
    if (dyn_smem > 0) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, dyn_smem);
    if (dyn_smem > 0 && step_occ_cap() > 0 && occ > step_occ_cap()) occ = step_occ_cap();
    if (occ < 1) occ = 1;
    if (occ > kMaxCtasPerSm) occ = kMaxCtasPerSm;
    int64_t g = (int64_t)sms * occ;
    if (dyn_smem > 0) {  // staged step kernels: keep >= min_tiles_per_cta() tiles per CTA
        const int64_t cap = (ntiles + min_tiles_per_cta() - 1) / min_tiles_per_cta();
        if (g > cap) g = cap;
    }
    if (g > ntiles) g = ntiles;
    return (int)(g < 1 ? 1 : g);
}

// ---- operator prep (once per cheb_moments call): scaled/padded gather matrix ---------
template <int MODE>
void run_prep(const cl_operator* op, double alpha, double beta, char* ws, const Layout& L,
              cudaStream_t st, int sms) {
    const cl_csr& G2 = (MODE == MODE_BTB) ? op->At : op->A;
    const int64_t d = G2.n_rows;
    int grid = (int)std::min<int64_t>((d + kThreads) / kThreads, (int64_t)sms * 8);
    if (grid < 1) grid = 1;
    // padded row pointer: lengths rounded up to the gather chunk, exclusive scan (CUB)
    prep_count_kernel<<<grid, kThreads, 0, st>>>(d, G2.row_ptr, G2.col_idx, MODE != MODE_BTB ? 1 : 0,
                                                 (int64_t*)(ws + L.cnt64));
    size_t sb = L.scan_bytes;
    cub::DeviceScan::ExclusiveSum(ws + L.scan, sb, (const int64_t*)(ws + L.cnt64), (int64_t*)(ws + L.rp2),
                                  (int)(d + 1), st);
    g_launches += 1;  // prep_count_kernel (the CUB scan kernels are library code, not counted)
    prep_kernel<MODE><<<grid, kThreads, 0, st>>>(
        d, G2.row_ptr, G2.col_idx, G2.val, alpha, beta, (int64_t*)(ws + L.rp2), L.rp2_len,
        (int32_t*)(ws + L.ci2), (double*)(ws + L.va2),
        MODE == MODE_RANK1 ? op->r1_u : nullptr, MODE == MODE_RANK1 ? (double*)(ws + L.u2) : nullptr,
        MODE != MODE_BTB ? (unsigned long long*)(ws + L.misc) : nullptr);
    g_launches++;
}

// Fused pairs with dynamic tile tickets (cheb_step2d_kernel) instead of the static map
// (CHEB_FUSED_DYN, default 1).
// fusion modes: 2 auto / 3 forced -> warp-specialised dynamic kernel; 4 static map; 5 dynamic,
// thread-0 producer
bool fused_dynamic() { return g_fusion.load() != 4; }
bool fused_ws() { return g_fusion.load() == 2 || g_fusion.load() == 3; }
// Dynamic lag beyond the halo, in units of the grid size (CHEB_FUSED_LAG; default 1.5 for the
// warp-specialised kernel, whose producer holds up to kWStages + 1 tickets, 1.0 otherwise): the
// stage-1 tiles a stage-2 ticket needs were handed out D - H tiles earlier and may still be in
// flight; measured optimum on configs[3] (profiles/r01_fusion_study.md).
double fused_lag_waves() {
    const char* e = getenv("CHEB_FUSED_LAG");
    return e ? atof(e) : (fused_ws() ? 1.5 : 1.0);
}

// Temporal fusion plan (CSR mode): stage-2 halo H (tiles) and lag D (positions).
struct FusionPlan {
    bool on = false;          // temporally fused pairs
    bool persistent = false;  // all steps in one persistent cooperative launch
    int64_t H = 0, D = 0;
    int G = 0;                // fused grid (= the single-step grid, for bit-identical moments)
    bool power = false;       // power basis (Taylor baseline): w_j = Ã w_{j-1}, every step "FIRST"
    bool doubling = false;    // moment doubling: ceil(n/2) applications of Ã give mu_0..mu_n
    bool vbits = false;       // per-step csr/rank-1: v = w_0 lives only as sign bits (steps 1, 2)
    bool gather = false;      // gather-staged step kernels (csr): TMA gather4 of each tile's rows
    bool small = false;       // L2-resident operator: 16-row tiles for the Algorithm-1 kernels (RP = 1)
    CUtensorMap tmap[2];      // W buffers 0/1 as [d][k] fp64 tensors (gather mode)
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda
// dependency, so the library still loads on machines without a driver).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int encode_rows_map(CUtensorMap* m, void* base, int64_t d, int k) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            return fail(CL_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
        fn = (EncodeTiledFn)p;
    }
    cuuint64_t gdim[2] = {(cuuint64_t)k, (cuuint64_t)d};
    cuuint64_t gstride[1] = {(cuuint64_t)k * 8};
    cuuint32_t box[2] = {(cuuint32_t)k, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CL_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return CL_OK;
}

// launch of a sign-bit step variant (own attribute for its dynamic shared memory)
template <int K, int MODE, bool FIRST, bool DBL, int VB, int RP = 0>
void launch_step(int grid, size_t smem, cudaStream_t st, const StepArgs& a) {
    static bool attr = false;  // benign race: the attribute value is the same for every caller
    if (!attr) {
        cudaFuncSetAttribute(cheb_step_kernel<K, MODE, FIRST, DBL, VB, RP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(200 * 1024));
        attr = true;
    }
    cheb_step_kernel<K, MODE, FIRST, DBL, VB, RP><<<grid, kThreads, smem, st>>>(a);
}

// ---- one probe block: K1, then n x ([K3] K2) --------------------------------
// RP: tile geometry of the Algorithm-1 kernels (0: CHEB_RPG; 1: 16-row tiles for L2-resident
// operators, FusionPlan::small); fused pairs always run with RP = 0
template <int K, int MODE, int RP = 0>
int run_block(const cl_operator* op, double alpha, double beta, int32_t n, uint64_t seed,
              int64_t p0, int kvalid, char* ws, const Layout& L, double* mu_rows,
              int64_t mu_stride, cudaStream_t st, int sms, const FusionPlan& fp) {
    constexpr int R4S = RP ? RP : CHEB_RPG;
    using G = Geo<K, R4S>;  // per-step / fused geometry; the doubling kernels use Geo<K, CHEB_RPG_DBL>
    constexpr int R4D = RP ? RP : CHEB_RPG_DBL;  // doubling kernels: same RP rule
    using GD = Geo<K, R4D>;
    using SL = StageLayout<K, MODE, false, R4S>;
    using SLD = StageLayout<K, MODE, false, R4D>;
    const int64_t d = op->A.n_cols;
    double* w[2] = {(double*)(ws + L.w0), (double*)(ws + L.w1)};
    double* y = (double*)(ws + L.y);
    uint32_t* sbits = (uint32_t*)(ws + L.sbits);
    double* sbuf = (double*)(ws + L.sbuf);

    StepArgs a{};
    a.d = d;
    a.rp = (const int64_t*)(ws + L.rp2);
    a.ci = (const int32_t*)(ws + L.ci2);
    a.va = (const double*)(ws + L.va2);
    a.bw = (MODE != MODE_BTB && op->A.nnz > 0) ? (const unsigned long long*)(ws + L.misc) : nullptr;
    a.sbits = sbits;
    a.beta = beta;
    a.r1c_alpha = alpha * op->r1_c;
    a.r1u = (MODE == MODE_RANK1 && op->r1_u) ? (const double*)(ws + L.u2) : nullptr;
    a.part = (double*)(ws + L.part);
    a.ticket = (unsigned int*)(ws + L.ticket);
    a.mu_out = mu_rows;
    a.mu_stride = mu_stride;
    a.kvalid = kvalid;

    // K1
    {
        constexpr int groups = kThreads / (K <= 64 ? K / 2 : K / 4);
        const int64_t niter = (d + groups - 1) / groups;
        constexpr size_t init_smem = red_scratch_bytes<K, MODE == MODE_RANK1 ? 2 : 1>();
        cudaFuncSetAttribute(probe_init_kernel<K, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)init_smem);
        const int grid = grid_for(probe_init_kernel<K, MODE>, niter, sms);
        a.mu_col = 0;
        a.s_next = sbuf;
        probe_init_kernel<K, MODE><<<grid, kThreads, init_smem, st>>>(a, seed, (uint64_t)p0,
                                                                    fp.vbits ? nullptr : w[0], sbits);
        g_launches++;
    }
    if (n < 1) return CL_OK;

    const int tile = fp.doubling ? GD::TILE : G::TILE;
    a.ntiles = (d + tile - 1) / tile;
    // dynamic shared memory: the staged tiles, reused as the reduction scratch at the end
    const size_t smem = std::max<size_t>(fp.doubling ? SLD::SMEM : SL::SMEM, red_scratch_bytes<K, 2>());  // persistent, fused
    const size_t smem_step = std::max<size_t>(
        (size_t)kStepStages * (fp.doubling ? StageLayout<K, MODE, CHEB_DBL_STAGE_WC, R4D>::BYTES : SL::BYTES),
        red_scratch_bytes<K, 3>());  // cheb_step_kernel
    const int grid_first = fp.doubling ? grid_for(cheb_step_kernel<K, MODE, true, true, 0, RP>, a.ntiles, sms, smem_step)
                                       : grid_for(cheb_step_kernel<K, MODE, true, false, 0, RP>, a.ntiles, sms, smem_step);
    const int grid_step = fp.doubling ? grid_for(cheb_step_kernel<K, MODE, false, true, 0, RP>, a.ntiles, sms, smem_step)
                                      : grid_for(cheb_step_kernel<K, MODE, false, false, 0, RP>, a.ntiles, sms, smem_step);
    int grid_spmm = 1;
    if (MODE == MODE_BTB) {
        const int64_t ng = (op->A.n_rows + SpmmGeo<K>::GROUPS - 1) / SpmmGeo<K>::GROUPS;
        grid_spmm = grid_for(spmm_kernel<K>, ng, sms);
    }
    // moment doubling (reading G25): steps j = 1..ceil(n/2); the epilogue of step j writes
    // mu_{2j-1} and mu_{2j} (indices <= n) from w_j^T w_{j-1} and w_j^T w_j
    const int32_t nsteps = fp.doubling ? (n + 1) / 2 : n;
    if (MODE != MODE_BTB && fp.persistent) {
        auto pkern = fp.doubling ? cheb_persist_kernel<K, MODE, true, RP> : cheb_persist_kernel<K, MODE, false, RP>;
        const int grid_p = grid_for(pkern, a.ntiles, sms, smem);
        PersistArgs pp{};
        pp.w0 = w[0];
        pp.w1 = w[1];
        pp.n = nsteps;
        pp.part = (double*)(ws + L.part);
        pp.s_buf = sbuf;
        pp.bar_count = (unsigned int*)(ws + L.misc + 16);
        pp.s_count = (unsigned int*)(ws + L.misc + 20);
        pp.err = (unsigned int*)(ws + L.misc + 8);
        pp.power = fp.power ? 1 : 0;
        CL_CUDA(cudaMemsetAsync(ws + L.misc + 16, 0, 16, st));
        void* args[] = {&a, &pp};
        ProfScope ps(st, 2);
        CL_CUDA(cudaLaunchCooperativeKernel((const void*)pkern, dim3(grid_p), dim3(kThreads), args, smem, st));
        g_launches++;
        return CL_OK;
    }
    int grid_fused = 0;
    if (MODE == MODE_CSR && fp.on) grid_fused = fp.G;
    for (int32_t j = 1; j <= nsteps; j++) {
        const double* cur = w[(j - 1) & 1];
        double* nxt = w[j & 1];
        if (MODE == MODE_CSR && RP == 0 && fp.on && !fp.doubling && j >= 2 && j + 1 <= n) {
            // steps j and j+1 in one launch: A = w_{j-2} -> w_j, B = w_{j-1} -> w_{j+1}
            FusedArgs f{};
            f.A = nxt;
            f.B = (double*)cur;
            f.cnt = (unsigned int*)(ws + L.cnt);
            f.err = (unsigned int*)(ws + L.misc + 8);
            f.D = fp.D;
            f.H = fp.H;
            a.mu_col = j;
            const int64_t nchunks = (a.ntiles + kChunkTiles - 1) / kChunkTiles;
            CL_CUDA(cudaMemsetAsync(f.cnt, 0, ((size_t)nchunks + 1) * sizeof(unsigned int), st));
            ProfScope ps(st, 1);
            if (fused_dynamic()) {
                FusedDynArgs dy{};
                dy.c1 = (unsigned int*)(ws + L.misc + 32);
                dy.c2 = (unsigned int*)(ws + L.misc + 36);
                CL_CUDA(cudaMemsetAsync(ws + L.misc + 32, 0, 8, st));
                void* args[] = {&a, &f, &dy};
                if (fused_ws()) {
                    const size_t smem_w = std::max<size_t>((size_t)kWStages * SL::BYTES, red_scratch_bytes<K, 2>());
                    cudaFuncSetAttribute(cheb_step2w_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_w);
                    CL_CUDA(cudaLaunchCooperativeKernel((const void*)cheb_step2w_kernel<K>, dim3(grid_fused),
                                                        dim3(kFusedWThreads), args, smem_w, st));
                } else {
                    CL_CUDA(cudaLaunchCooperativeKernel((const void*)cheb_step2d_kernel<K>, dim3(grid_fused),
                                                        dim3(kThreads), args, smem, st));
                }
            } else {
                void* args[] = {&a, &f};
                CL_CUDA(cudaLaunchCooperativeKernel((const void*)cheb_step2_kernel<K>, dim3(grid_fused),
                                                    dim3(kThreads), args, smem, st));
            }
            g_launches++;
            j++;  // consumed two steps
            continue;
        }
        if (MODE == MODE_BTB) {
            spmm_kernel<K><<<grid_spmm, kThreads, 0, st>>>(op->A.n_rows, op->A.row_ptr, op->A.col_idx,
                                                          op->A.val, cur, y);
            g_launches++;
        }
        a.xg = (MODE == MODE_BTB) ? y : cur;
        a.wcur = cur;
        a.wnext = nxt;
        a.s_cur = sbuf + ((j - 1) & 1) * K;
        a.s_next = sbuf + (j & 1) * K;
        a.mu_col = j;
        ProfScope ps(st);
        if (MODE == MODE_CSR && fp.gather) {  // gather-staged steps (Algorithm 1, csr)
            if constexpr (K >= 16) {
                using GG = GsGeo<K>;
                GsArgs gs{};
                gs.gl = (const int32_t*)(ws + L.gl);
                gs.gl_len = (const int32_t*)(ws + L.gl_len);
                gs.sl = (const uint16_t*)(ws + L.sl);
                gs.ntiles = L.gs_ntiles;
                gs.err = (unsigned int*)(ws + L.misc + 8);
                const size_t smem_gs = std::max<size_t>((size_t)CHEB_GS_STAGES * GG::BYTES, red_scratch_bytes<K, 1>());
                const int grid_gs = (int)std::min<int64_t>((int64_t)sms * 2, L.gs_ntiles);
                if (j == 1) {
                    cudaFuncSetAttribute(cheb_step_gs_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_gs);
                    cheb_step_gs_kernel<K, true><<<grid_gs, kThreads + 32, smem_gs, st>>>(a, gs, fp.tmap[(j - 1) & 1]);
                } else {
                    cudaFuncSetAttribute(cheb_step_gs_kernel<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_gs);
                    cheb_step_gs_kernel<K, false><<<grid_gs, kThreads + 32, smem_gs, st>>>(a, gs, fp.tmap[(j - 1) & 1]);
                }
                g_launches++;
                continue;
            }
        }
        // steps 1 and 2 read v = w_0 from the sign bits when it was not materialised (fp.vbits);
        // same grids as the plain kernels, so the moments are bit-identical either way
        constexpr int V1 = MODE != MODE_BTB ? 1 : 0, V2 = MODE != MODE_BTB ? 2 : 0;
        const bool vb1 = fp.vbits && j == 1, vb2 = fp.vbits && j == 2 && !fp.power;
        if (fp.doubling) {
            if (j == 1) {
                if (vb1) launch_step<K, MODE, true, true, V1, RP>(grid_first, smem_step, st, a);
                else launch_step<K, MODE, true, true, 0, RP>(grid_first, smem_step, st, a);
            } else {
                if (vb2) launch_step<K, MODE, false, true, V2, RP>(grid_step, smem_step, st, a);
                else launch_step<K, MODE, false, true, 0, RP>(grid_step, smem_step, st, a);
            }
        } else if (j == 1 || fp.power) {  // power basis: w_j = Ã w_{j-1} (no w_{j-2} term), ping-pong
            if (vb1) launch_step<K, MODE, true, false, V1, RP>(grid_first, smem_step, st, a);
            else launch_step<K, MODE, true, false, 0, RP>(grid_first, smem_step, st, a);
        } else {
            if (vb2) launch_step<K, MODE, false, false, V2, RP>(grid_step, smem_step, st, a);
            else launch_step<K, MODE, false, false, 0, RP>(grid_step, smem_step, st, a);
        }
        g_launches++;
    }
    return CL_OK;
}

template <int K>
int run_block_mode(const cl_operator* op, double alpha, double beta, int32_t n, uint64_t seed,
                   int64_t p0, int kvalid, char* ws, const Layout& L, double* mu_rows,
                   int64_t mu_stride, cudaStream_t st, int sms, const FusionPlan& fp) {
    const bool small = fp.small && !fp.on;
    switch (op->kind) {
        case CL_OP_CSR:
            if (small) return run_block<K, MODE_CSR, 1>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp);
            return run_block<K, MODE_CSR>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp);
        case CL_OP_CSR_RANK1:
            if (small) return run_block<K, MODE_RANK1, 1>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp);
            return run_block<K, MODE_RANK1>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp);
        default:
            return run_block<K, MODE_BTB>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp);
    }
}

void prep_mode(const cl_operator* op, double alpha, double beta, char* ws, const Layout& L,
               cudaStream_t st, int sms) {
    switch (op->kind) {
        case CL_OP_CSR: run_prep<MODE_CSR>(op, alpha, beta, ws, L, st, sms); break;
        case CL_OP_CSR_RANK1: run_prep<MODE_RANK1>(op, alpha, beta, ws, L, st, sms); break;
        default: run_prep<MODE_BTB>(op, alpha, beta, ws, L, st, sms); break;
    }
}

int fused_ws_occupancy(int k) {  // cheb_step2w_kernel: 288 threads per CTA
    auto occ_of = [](auto kern, size_t smem) {
        int occ = 0;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFusedWThreads, smem);
        return occ < 1 ? 1 : (occ > kMaxCtasPerSm ? kMaxCtasPerSm : occ);
    };
    switch (k) {
        case 8: return occ_of(cheb_step2w_kernel<8>, std::max<size_t>((size_t)kWStages * StageLayout<8, MODE_CSR>::BYTES, red_scratch_bytes<8, 2>()));
        case 16: return occ_of(cheb_step2w_kernel<16>, std::max<size_t>((size_t)kWStages * StageLayout<16, MODE_CSR>::BYTES, red_scratch_bytes<16, 2>()));
        case 32: return occ_of(cheb_step2w_kernel<32>, std::max<size_t>((size_t)kWStages * StageLayout<32, MODE_CSR>::BYTES, red_scratch_bytes<32, 2>()));
        case 64: return occ_of(cheb_step2w_kernel<64>, std::max<size_t>((size_t)kWStages * StageLayout<64, MODE_CSR>::BYTES, red_scratch_bytes<64, 2>()));
        default: return occ_of(cheb_step2w_kernel<128>, std::max<size_t>((size_t)kWStages * StageLayout<128, MODE_CSR>::BYTES, red_scratch_bytes<128, 2>()));
    }
}

int fused_occupancy(int k) {
    // both fused kernels (static map / dynamic tickets) run with the same shared memory; a
    // cooperative grid must fit the smaller occupancy
    auto occ_of = [](auto kern, size_t smem) {
        int occ = 0;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
        return occ < 1 ? 1 : (occ > kMaxCtasPerSm ? kMaxCtasPerSm : occ);
    };
    auto both = [&](auto ks, auto kd, size_t smem) { return std::min(occ_of(ks, smem), occ_of(kd, smem)); };
    switch (k) {
        case 8: return both(cheb_step2_kernel<8>, cheb_step2d_kernel<8>, std::max<size_t>(StageLayout<8, MODE_CSR>::SMEM, red_scratch_bytes<8, 2>()));
        case 16: return both(cheb_step2_kernel<16>, cheb_step2d_kernel<16>, std::max<size_t>(StageLayout<16, MODE_CSR>::SMEM, red_scratch_bytes<16, 2>()));
        case 32: return both(cheb_step2_kernel<32>, cheb_step2d_kernel<32>, std::max<size_t>(StageLayout<32, MODE_CSR>::SMEM, red_scratch_bytes<32, 2>()));
        case 64: return both(cheb_step2_kernel<64>, cheb_step2d_kernel<64>, std::max<size_t>(StageLayout<64, MODE_CSR>::SMEM, red_scratch_bytes<64, 2>()));
        default: return both(cheb_step2_kernel<128>, cheb_step2d_kernel<128>, std::max<size_t>(StageLayout<128, MODE_CSR>::SMEM, red_scratch_bytes<128, 2>()));
    }
}

int step_grid_csr(int k, int64_t ntiles, int sms) {
    switch (k) {
        case 8: return grid_for(cheb_step_kernel<8, MODE_CSR, false>, ntiles, sms, std::max<size_t>(kStepStages * StageLayout<8, MODE_CSR>::BYTES, red_scratch_bytes<8, 3>()));
        case 16: return grid_for(cheb_step_kernel<16, MODE_CSR, false>, ntiles, sms, std::max<size_t>(kStepStages * StageLayout<16, MODE_CSR>::BYTES, red_scratch_bytes<16, 3>()));
        case 32: return grid_for(cheb_step_kernel<32, MODE_CSR, false>, ntiles, sms, std::max<size_t>(kStepStages * StageLayout<32, MODE_CSR>::BYTES, red_scratch_bytes<32, 3>()));
        case 64: return grid_for(cheb_step_kernel<64, MODE_CSR, false>, ntiles, sms, std::max<size_t>(kStepStages * StageLayout<64, MODE_CSR>::BYTES, red_scratch_bytes<64, 3>()));
        default: return grid_for(cheb_step_kernel<128, MODE_CSR, false>, ntiles, sms, std::max<size_t>(kStepStages * StageLayout<128, MODE_CSR>::BYTES, red_scratch_bytes<128, 3>()));
    }
}

int pick_k(int64_t m) {
    // One block when m <= 64 (smallest k >= m: the matrix is read once per step);
    // otherwise blocks of 64 (measured faster than 128 on B200 at config 3).
    if (m > 32) return 64;
    if (m > 16) return 32;
    if (m > 8) return 16;
    return 8;
}

}  // namespace

// ============================================================================
extern "C" {

int cheb_version(void) { return 100; }

int cheb_release_cache(void) {
    for (auto& A : g_arena) A.release();
    return CL_OK;
}

const char* cheb_last_error(void) { return g_err.c_str(); }

int64_t cheb_launch_count(void) { return g_launches.load(); }

int cheb_profile_begin(void) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (int k = 0; k < 3; k++) {
        for (auto& p : g_prof.ev[k]) g_prof.pool.push_back(p);
        g_prof.ev[k].clear();
        g_prof.ms[k] = 0.0;
        g_prof.n[k] = 0;
    }
    g_prof.on = true;
    return CL_OK;
}

int cheb_profile_end(double* step_ms, int64_t* step_launches) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = false;
    for (int k = 0; k < 3; k++) {
        double tot = 0.0;
        for (auto& p : g_prof.ev[k]) {
            cudaError_t e = cudaEventSynchronize(p.second);
            if (e != cudaSuccess) return fail(CL_ECUDA, "event sync: %s", cudaGetErrorString(e));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, p.first, p.second);
            tot += ms;
        }
        g_prof.ms[k] = tot;
        g_prof.n[k] = (int64_t)g_prof.ev[k].size();
        for (auto& p : g_prof.ev[k]) g_prof.pool.push_back(p);
        g_prof.ev[k].clear();
    }
    if (step_ms) *step_ms = g_prof.ms[0];
    if (step_launches) *step_launches = g_prof.n[0];
    return CL_OK;
}

int cheb_profile_fused(double* ms, int64_t* launches) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (ms) *ms = g_prof.ms[1];
    if (launches) *launches = g_prof.n[1];
    return CL_OK;
}

int cheb_profile_persistent(double* ms, int64_t* launches) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (ms) *ms = g_prof.ms[2];
    if (launches) *launches = g_prof.n[2];
    return CL_OK;
}

int cheb_set_persistent(int32_t mode) {
    if (mode < 0 || mode > 2) return fail(CL_EINVAL, "persistent mode must be 0, 1 or 2");
    g_persistent = mode;
    return CL_OK;
}

int cheb_set_small_tiles(int32_t mode) {
    if (mode < 0 || mode > 1) return fail(CL_EINVAL, "small-tiles mode must be 0 or 1");
    g_small_tiles = mode;
    return CL_OK;
}

int cheb_get_small_tiles(void) { return g_small_tiles.load(); }

int cheb_set_doubling(int32_t on) {
    if (on < 0 || on > 1) return fail(CL_EINVAL, "doubling mode must be 0 or 1");
    g_doubling = on;
    return CL_OK;
}

int cheb_get_doubling(void) { return g_doubling.load(); }

int cheb_set_gather(int32_t on) {
    if (on < 0 || on > 1) return fail(CL_EINVAL, "gather mode must be 0 or 1");
    g_gather = on;
    return CL_OK;
}

int cheb_get_gather(void) { return g_gather.load(); }

int cheb_set_fusion(int32_t steps) {
    if (steps < 1 || steps > 5) return fail(CL_EINVAL, "fusion mode must be 1..5");
    g_fusion = steps;
    return CL_OK;
}

// Host fp64 coefficient routine: accumulate, node by node, f(x_k)
// times T_j(x_k) for all j with the scalar recurrence, then scale.
int cheb_coeffs_log(double a, double b, int32_t degree, double* c_out) {
    int rc = check_ab(a, b, degree);
    if (rc) return rc;
    if (!c_out) return fail(CL_EINVAL, "c_out is NULL");
    const int n = degree;
    std::vector<double> acc((size_t)n + 1, 0.0);
    const double half_w = 0.5 * (b - a), mid = 0.5 * (b + a);
    for (int k = 0; k <= n; k++) {
        const double x = std::cos(M_PI * (k + 0.5) / (n + 1.0));
        const double f = std::log(half_w * x + mid);
        double tm1 = 1.0, t = x;
        acc[0] += f;
        if (n >= 1) acc[1] += f * x;
        for (int j = 2; j <= n; j++) {
            const double tn = 2.0 * x * t - tm1;
            acc[j] += f * tn;
            tm1 = t;
            t = tn;
        }
    }
    const double s0 = 1.0 / (n + 1.0), s1 = 2.0 / (n + 1.0);
    for (int j = 0; j <= n; j++) {
        const double cj = (j == 0 ? s0 : s1) * acc[j];
        if (!std::isfinite(cj)) return fail(CL_ENONFINITE, "coefficient %d not finite", j);
        c_out[j] = cj;
    }
    return CL_OK;
}

size_t cheb_workspace_bytes(const cl_operator* op, int32_t probe_block) {
    if (check_op(op)) return 0;
    if (!valid_k(probe_block)) {
        fail(CL_EINVAL, "probe_block must be 8, 16, 32, 64 or 128 (got %d)", probe_block);
        return 0;
    }
    return plan(op->A.n_cols, gather_nnz(op), probe_block, op->kind, sm_count()).total;
}

namespace {
int moments_impl(const cl_operator* op, double alpha, double beta, bool power, int32_t degree,
                 int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                 void* workspace, size_t ws_bytes, double* mu_out, void* stream);
}

int cheb_moments(const cl_operator* op, double a, double b, int32_t degree,
                 int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                 void* workspace, size_t ws_bytes, double* mu_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if ((rc = check_ab(a, b, degree))) return rc;
    return moments_impl(op, 2.0 / (b - a), (b + a) / (b - a), false, degree, probe_begin, probe_end, seed,
                        probe_block, workspace, ws_bytes, mu_out, stream);
}

int cheb_power_moments(const cl_operator* op, double s, int32_t degree, int64_t probe_begin,
                       int64_t probe_end, uint64_t seed, int32_t probe_block, void* workspace,
                       size_t ws_bytes, double* mu_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if (!std::isfinite(s) || !(s > 0.0)) return fail(CL_EINVAL, "need finite s > 0");
    if (degree < 0) return fail(CL_EINVAL, "degree < 0");
    // A = I - M/s = alpha*M - beta*I with alpha = -1/s, beta = -1
    return moments_impl(op, -1.0 / s, -1.0, true, degree, probe_begin, probe_end, seed, probe_block,
                        workspace, ws_bytes, mu_out, stream);
}

int cheb_affine_power_moments(const cl_operator* op, double alpha, double beta, int32_t degree,
                              int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                              void* workspace, size_t ws_bytes, double* mu_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if (!std::isfinite(alpha) || !std::isfinite(beta)) return fail(CL_EINVAL, "alpha/beta not finite");
    if (degree < 0) return fail(CL_EINVAL, "degree < 0");
    return moments_impl(op, alpha, beta, true, degree, probe_begin, probe_end, seed, probe_block, workspace,
                        ws_bytes, mu_out, stream);
}

namespace {
double unkey(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double x;
    memcpy(&x, &b, sizeof(x));
    return x;
}
}  // namespace

int cheb_norm_bound(const cl_operator* op, double* s_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if (!s_out) return fail(CL_EINVAL, "s_out is NULL");
    if (op->kind == CL_OP_BTB) {
        double ab[2];
        // ||B||_1 ||B||_inf bounds sigma_max(B)^2; Johnson's bound is not needed here
        cudaStream_t st = (cudaStream_t)stream;
        DevBuf buf;
        CL_CUDA(cudaMalloc(&buf.p, 3 * sizeof(unsigned long long)));
        unsigned long long init[3] = {~0ull, 0ull, 0ull};
        CL_CUDA(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
        const int64_t d = op->A.n_rows;
        int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
        bounds_btb_kernel<<<grid, kThreads, 0, st>>>(d, op->A.row_ptr, op->A.col_idx, op->A.val,
                                                      op->At.row_ptr, op->At.col_idx, op->At.val,
                                                      (unsigned long long*)buf.p);
        g_launches++;
        CL_CUDA(cudaGetLastError());
        unsigned long long h[3];
        CL_CUDA(cudaMemcpyAsync(h, buf.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        CL_CUDA(cudaStreamSynchronize(st));
        ab[1] = unkey(h[1]) * unkey(h[2]);
        *s_out = ab[1];
        return CL_OK;
    }
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf buf;
    CL_CUDA(cudaMalloc(&buf.p, 3 * sizeof(unsigned long long)));
    unsigned long long init[3] = {0ull, 0ull, ~0ull};
    CL_CUDA(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const int64_t d = op->A.n_rows;
    int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    const double* u = op->kind == CL_OP_CSR_RANK1 ? op->r1_u : nullptr;
    gershgorin_kernel<<<grid, kThreads, 0, st>>>(d, op->A.row_ptr, op->A.col_idx, op->A.val, u,
                                                  (unsigned long long*)buf.p);
    g_launches++;
    CL_CUDA(cudaGetLastError());
    unsigned long long h[3];
    CL_CUDA(cudaMemcpyAsync(h, buf.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    double s = unkey(h[0]);
    if (op->kind == CL_OP_CSR_RANK1) {
        const double umax = op->r1_u ? unkey(h[1]) : 1.0;
        s += std::fabs(op->r1_c) * umax * umax * (double)d;  // |c| |u_i| sum_j |u_j| <= |c| umax^2 d
    }
    *s_out = s;
    return CL_OK;
}

int cheb_gershgorin(const cl_csr* A, double* lo_hi, void* stream) {
    int rc;
    if (!A || !lo_hi) return fail(CL_EINVAL, "NULL pointer");
    if ((rc = check_csr(*A, "A"))) return rc;
    if (A->n_rows != A->n_cols || A->n_rows < 1) return fail(CL_EDIM, "A must be square and non-empty");
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf buf;
    CL_CUDA(cudaMalloc(&buf.p, 3 * sizeof(unsigned long long)));
    unsigned long long init[3] = {0ull, 0ull, ~0ull};
    CL_CUDA(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const int64_t d = A->n_rows;
    int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    gershgorin_kernel<<<grid, kThreads, 0, st>>>(d, A->row_ptr, A->col_idx, A->val, nullptr,
                                                  (unsigned long long*)buf.p);
    g_launches++;
    CL_CUDA(cudaGetLastError());
    unsigned long long h[3];
    CL_CUDA(cudaMemcpyAsync(h, buf.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    lo_hi[0] = unkey(h[2]);
    lo_hi[1] = unkey(h[0]);
    return CL_OK;
}

int cheb_quadform(const cl_csr* A, const double* x, double* out, void* stream) {
    int rc;
    if (!A || !x || !out) return fail(CL_EINVAL, "NULL pointer");
    if ((rc = check_csr(*A, "A"))) return rc;
    if (A->n_rows != A->n_cols || A->n_rows < 1) return fail(CL_EDIM, "A must be square and non-empty");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t d = A->n_rows;
    const int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    DevBuf buf;
    CL_CUDA(cudaMalloc(&buf.p, sizeof(double) * (grid + 1)));
    double* part = (double*)buf.p;
    quadform_kernel<<<grid, kThreads, 0, st>>>(d, A->row_ptr, A->col_idx, A->val, x, part);
    quadform_final_kernel<<<1, 32, 0, st>>>(part, grid, part + grid);
    g_launches += 2;
    CL_CUDA(cudaGetLastError());
    CL_CUDA(cudaMemcpyAsync(out, part + grid, sizeof(double), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    return CL_OK;
}

int cheb_taylor_coeffs(double s, int32_t degree, double* c_out) {
    if (!std::isfinite(s) || !(s > 0.0)) return fail(CL_EINVAL, "need finite s > 0");
    if (degree < 0 || !c_out) return fail(CL_EINVAL, "bad degree or NULL c_out");
    c_out[0] = std::log(s);  // log det M = d log s + log det(M/s), log det(M/s) = tr log(I - A)
    for (int32_t k = 1; k <= degree; k++) c_out[k] = -1.0 / (double)k;  // log(1-x) = -sum x^k/k
    return CL_OK;
}

namespace {
int moments_impl(const cl_operator* op, double alpha, double beta, bool power, int32_t degree,
                 int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                 void* workspace, size_t ws_bytes, double* mu_out, void* stream) {
    int rc;
    if (probe_begin < 0 || probe_end <= probe_begin)
        return fail(CL_EINVAL, "need 0 <= probe_begin < probe_end");
    if (!valid_k(probe_block)) return fail(CL_EINVAL, "probe_block must be 8, 16, 32, 64 or 128");
    if (!workspace || !mu_out) return fail(CL_EINVAL, "NULL workspace or mu_out");
    const int sms = sm_count();
    const Layout L = plan(op->A.n_cols, gather_nnz(op), probe_block, op->kind, sms);
    if (ws_bytes < L.total)
        return fail(CL_ENOMEM, "workspace too small: %zu < %zu", ws_bytes, L.total);
    if ((uintptr_t)workspace & 255) return fail(CL_EINVAL, "workspace must be 256-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    char* ws = (char*)workspace;
    const int64_t stride = (int64_t)degree + 1;
    CL_CUDA(cudaGetLastError());
    CL_CUDA(cudaMemsetAsync(ws + L.ticket, 0, 256, st));
    CL_CUDA(cudaMemsetAsync(ws + L.misc, 0, 256, st));
    prep_mode(op, alpha, beta, ws, L, st, sms);
    FusionPlan fp;
    fp.power = power;
    fp.doubling = !power && g_doubling.load() == 1;
    if (op->kind != CL_OP_BTB) {
        // L2-resident working set (two probe-block buffers + matrix): the per-step launch and
        // drain gaps dominate, so run all steps in one launch; small tiles either way (the per-step
        // and persistent schedules keep one geometry, hence bit-identical moments)
        int l2 = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        const double wset = 2.0 * op->A.n_cols * probe_block * 8.0 + 12.0 * op->A.nnz + 8.0 * op->A.n_cols;
        // 16-row-per-group tiles also pay for Algorithm 1 at k <= 16 (configs[3], k = 16: 1565 vs
        // 1608 ms per estimate), where a standard tile has 128+ rows
        fp.small = g_small_tiles.load() != 0 && (wset <= 0.5 * (double)l2 || (probe_block <= 16 && !fp.doubling));
        if (g_persistent.load() > 0 && degree >= 1) fp.persistent = g_persistent.load() == 2 || wset <= 0.5 * (double)l2;
        if (getenv("CHEB_DEBUG")) fprintf(stderr, "[chebld] L2=%d working set=%.0f\n", l2, wset);
    }
    if (!fp.persistent && !power && !fp.doubling && op->kind == CL_OP_CSR && g_fusion.load() >= 2 && degree >= 3) {
        // needs the operator bandwidth computed by the prep kernel: one small D2H per call
        unsigned long long bw = 0;
        CL_CUDA(cudaMemcpyAsync(&bw, ws + L.misc, sizeof(bw), cudaMemcpyDeviceToHost, st));
        CL_CUDA(cudaStreamSynchronize(st));
        const int T = tile_rows(probe_block);
        const int64_t ntiles = (op->A.n_cols + T - 1) / T;
        // same grid as the single-step kernel (bit-identical per-CTA partial sums), limited to
        // what the fused kernel can keep co-resident
        int64_t G = step_grid_csr(probe_block, ntiles, sms);
        const int64_t Gmax = (int64_t)sms * (fused_ws() ? fused_ws_occupancy(probe_block) : fused_occupancy(probe_block));
        if (G > Gmax) G = Gmax;
        fp.G = (int)G;
        fp.H = (int64_t)((bw + T - 1) / T) + 1;
        fp.D = (kFusedSlack + (fp.H + 2 + G - 1) / G) * G;
        if (fused_dynamic()) fp.D = fp.H + 2 + (int64_t)(G * fused_lag_waves());  // tickets: any D > H
        if (getenv("CHEB_FUSED_NOWAIT")) fp.H = -1;  // TIMING DIAGNOSTIC ONLY: wrong results
        const double window = (double)(fp.D + fp.H + 2) * T * probe_block * 8.0 * 2.0;
        int l2 = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        fp.on = g_fusion.load() >= 3 || (ntiles >= 4 * fp.D && window <= 0.4 * (double)l2);
    }
    // gather-staged steps (opt-in): csr, Algorithm 1, per-step schedule, k >= 16; needs every tile's
    // nonzeros / unique rows within capacity (checked by the list-building pass: one sync)
    if (g_gather.load() == 1 && op->kind == CL_OP_CSR && probe_block >= 16 && !fp.persistent && !fp.on && !power &&
        !fp.doubling && L.gs_ntiles > 0) {
        unsigned int* ovf = (unsigned int*)(ws + L.misc + 44);
        const int grid = (int)std::min<int64_t>((L.gs_ntiles + 7) / 8, (int64_t)sms * 16);
        switch (probe_block) {
            case 16: gather_list_kernel<16><<<grid, kThreads, 0, st>>>(op->A.n_rows, L.gs_ntiles, (const int64_t*)(ws + L.rp2), (const int32_t*)(ws + L.ci2), (int32_t*)(ws + L.gl), (int32_t*)(ws + L.gl_len), (uint16_t*)(ws + L.sl), ovf); break;
            case 32: gather_list_kernel<32><<<grid, kThreads, 0, st>>>(op->A.n_rows, L.gs_ntiles, (const int64_t*)(ws + L.rp2), (const int32_t*)(ws + L.ci2), (int32_t*)(ws + L.gl), (int32_t*)(ws + L.gl_len), (uint16_t*)(ws + L.sl), ovf); break;
            case 64: gather_list_kernel<64><<<grid, kThreads, 0, st>>>(op->A.n_rows, L.gs_ntiles, (const int64_t*)(ws + L.rp2), (const int32_t*)(ws + L.ci2), (int32_t*)(ws + L.gl), (int32_t*)(ws + L.gl_len), (uint16_t*)(ws + L.sl), ovf); break;
            default: gather_list_kernel<128><<<grid, kThreads, 0, st>>>(op->A.n_rows, L.gs_ntiles, (const int64_t*)(ws + L.rp2), (const int32_t*)(ws + L.ci2), (int32_t*)(ws + L.gl), (int32_t*)(ws + L.gl_len), (uint16_t*)(ws + L.sl), ovf); break;
        }
        g_launches++;
        unsigned int hovf = 1;
        CL_CUDA(cudaMemcpyAsync(&hovf, ovf, sizeof(hovf), cudaMemcpyDeviceToHost, st));
        CL_CUDA(cudaStreamSynchronize(st));
        fp.gather = (hovf == 0);
        if (fp.gather) {
            if ((rc = encode_rows_map(&fp.tmap[0], ws + L.w0, op->A.n_cols, probe_block))) return rc;
            if ((rc = encode_rows_map(&fp.tmap[1], ws + L.w1, op->A.n_cols, probe_block))) return rc;
        }
    }
    // per-step csr/rank-1 without fused pairs: v = w_0 only as sign bits (CHEB_VBITS=0 disables)
    fp.vbits = !fp.persistent && !fp.on && !fp.gather && op->kind != CL_OP_BTB && env_int("CHEB_VBITS", 1) != 0;
    if (getenv("CHEB_DEBUG"))
        fprintf(stderr, "[chebld] d=%lld nnz=%lld k=%d kind=%d persistent=%d fused=%d doubling=%d gather=%d H=%lld D=%lld\n",
                (long long)op->A.n_cols, (long long)op->A.nnz, probe_block, op->kind, (int)fp.persistent,
                (int)fp.on, (int)fp.doubling, (int)fp.gather, (long long)fp.H, (long long)fp.D);
    for (int64_t p0 = probe_begin; p0 < probe_end; p0 += probe_block) {
        const int kvalid = (int)std::min<int64_t>(probe_block, probe_end - p0);
        double* rows = mu_out + (size_t)(p0 - probe_begin) * stride;
        switch (probe_block) {
            case 8: rc = run_block_mode<8>(op, alpha, beta, degree, seed, p0, kvalid, ws, L, rows, stride, st, sms, fp); break;
            case 16: rc = run_block_mode<16>(op, alpha, beta, degree, seed, p0, kvalid, ws, L, rows, stride, st, sms, fp); break;
            case 32: rc = run_block_mode<32>(op, alpha, beta, degree, seed, p0, kvalid, ws, L, rows, stride, st, sms, fp); break;
            case 64: rc = run_block_mode<64>(op, alpha, beta, degree, seed, p0, kvalid, ws, L, rows, stride, st, sms, fp); break;
            default: rc = run_block_mode<128>(op, alpha, beta, degree, seed, p0, kvalid, ws, L, rows, stride, st, sms, fp); break;
        }
        if (rc) return rc;
    }
    CL_CUDA(cudaGetLastError());
    return CL_OK;
}
}  // namespace

int cheb_finalize(const double* mu, const double* c, int64_t m, int32_t degree,
                  double* gamma_p, double* stats, void* stream) {
    if (!mu || !c || !gamma_p || !stats) return fail(CL_EINVAL, "NULL pointer");
    if (m < 1 || degree < 0) return fail(CL_EINVAL, "need m >= 1, degree >= 0");
    finalize_kernel<<<1, kThreads, 0, (cudaStream_t)stream>>>(mu, c, m, degree, gamma_p, stats);
    g_launches++;
    CL_CUDA(cudaGetLastError());
    return CL_OK;
}

namespace {


int logdet_device(const cl_operator* op, double a, double b, int32_t degree, int32_t num_probes,
                  uint64_t seed, int32_t probe_block, cl_result* out, cudaStream_t st) {
    const int k = probe_block ? probe_block : pick_k(num_probes);
    if (!valid_k(k)) return fail(CL_EINVAL, "probe_block must be 0, 8, 16, 32, 64 or 128");
    const size_t ws_bytes = plan(op->A.n_cols, gather_nnz(op), k, op->kind, sm_count()).total;
    const size_t mu_n = (size_t)num_probes * (degree + 1);
    const size_t aux_bytes = sizeof(double) * (mu_n + (degree + 1) + num_probes + 4);
    struct { void* p; } ws, aux;
    int rc0 = arena_get(0, align256(ws_bytes) + aux_bytes, &ws.p);
    if (rc0) return rc0;
    aux.p = (char*)ws.p + align256(ws_bytes);
    double* mu = (double*)aux.p;
    double* c = mu + mu_n;
    double* gp = c + degree + 1;
    double* stats = gp + num_probes;
    std::vector<double> ch((size_t)degree + 1);
    int rc = cheb_coeffs_log(a, b, degree, ch.data());
    if (rc) return rc;
    CL_CUDA(cudaMemcpyAsync(c, ch.data(), ch.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    rc = cheb_moments(op, a, b, degree, 0, num_probes, seed, k, ws.p, ws_bytes, mu, st);
    if (rc) return rc;
    rc = cheb_finalize(mu, c, num_probes, degree, gp, stats, st);
    if (rc) return rc;
    double hstats[3];
    unsigned int ferr = 0;
    CL_CUDA(cudaMemcpyAsync(hstats, stats, sizeof(hstats), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaMemcpyAsync(&ferr, (char*)ws.p + plan(op->A.n_cols, gather_nnz(op), k, op->kind, sm_count()).misc + 8,
                            sizeof(ferr), cudaMemcpyDeviceToHost, st));
    if (out->per_probe)
        CL_CUDA(cudaMemcpyAsync(out->per_probe, gp, sizeof(double) * num_probes, cudaMemcpyDeviceToHost, st));
    if (out->moments)
        CL_CUDA(cudaMemcpyAsync(out->moments, mu, sizeof(double) * mu_n, cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    out->logdet = hstats[0];
    out->stderr_ = hstats[1];
    out->num_probes = num_probes;
    out->degree = degree;
    out->probe_block = k;
    if (ferr) return fail(CL_ECUDA, "fused-step dependency wait timed out (CTAs not co-resident?)");
    if (hstats[2] != 1.0 || !std::isfinite(hstats[0]))
        return fail(CL_ENONFINITE, "non-finite estimate: [a,b]=[%g,%g] likely does not enclose the spectrum", a, b);
    return CL_OK;
}

}  // namespace

int cheb_logdet(const cl_operator* op, double a, double b, int32_t degree, int32_t num_probes,
                uint64_t seed, int32_t probe_block, cl_result* out) {
    auto t0 = std::chrono::steady_clock::now();
    int rc;
    if ((rc = check_op(op))) return rc;
    if ((rc = check_ab(a, b, degree))) return rc;
    if (num_probes < 1) return fail(CL_EINVAL, "num_probes < 1");
    if (!out) return fail(CL_EINVAL, "out is NULL");
    cudaStream_t st;
    CL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    rc = logdet_device(op, a, b, degree, num_probes, seed, probe_block, out, st);
    cudaStreamDestroy(st);
    out->elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

int cheb_logdet_host(const cl_operator* op, double a, double b, int32_t degree, int32_t num_probes,
                     uint64_t seed, int32_t probe_block, cl_result* out) {
    auto t0 = std::chrono::steady_clock::now();
    int rc;
    if ((rc = check_op(op))) return rc;
    if ((rc = check_ab(a, b, degree))) return rc;
    if (num_probes < 1) return fail(CL_EINVAL, "num_probes < 1");
    if (!out) return fail(CL_EINVAL, "out is NULL");
    cudaStream_t st;
    CL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cl_operator dop = *op;
    // one arena block holds the device copy of every operator array
    auto csr_bytes = [](const cl_csr& A) {
        return align256(sizeof(int64_t) * (A.n_rows + 1)) + align256(sizeof(int32_t) * A.nnz) +
               align256(sizeof(double) * A.nnz);
    };
    size_t need = csr_bytes(op->A);
    if (op->kind == CL_OP_BTB) need += csr_bytes(op->At);
    if (op->kind == CL_OP_CSR_RANK1 && op->r1_u) need += align256(sizeof(double) * op->A.n_cols);
    void* blk = nullptr;
    const double t_alloc = now_s();
    if ((rc = arena_get(1, need, &blk))) {
        cudaStreamDestroy(st);
        return rc;
    }
    size_t used = 0;
    auto up = [&](const void* h, size_t bytes, const void** dptr) -> int {
        if (!h || bytes == 0) return CL_OK;
        char* d = (char*)blk + used;
        used += align256(bytes);
        CL_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
        *dptr = d;
        return CL_OK;
    };
    auto up_csr = [&](cl_csr& A) -> int {
        int r;
        if ((r = up(A.row_ptr, sizeof(int64_t) * (A.n_rows + 1), (const void**)&A.row_ptr))) return r;
        if ((r = up(A.col_idx, sizeof(int32_t) * A.nnz, (const void**)&A.col_idx))) return r;
        return up(A.val, sizeof(double) * A.nnz, (const void**)&A.val);
    };
    rc = up_csr(dop.A);
    if (!rc && dop.kind == CL_OP_BTB) rc = up_csr(dop.At);
    if (!rc && dop.kind == CL_OP_CSR_RANK1 && dop.r1_u)
        rc = up(dop.r1_u, sizeof(double) * dop.A.n_cols, (const void**)&dop.r1_u);
    const double t_h2d = now_s();
    if (getenv("CHEB_DEBUG")) {
        cudaStreamSynchronize(st);
        fprintf(stderr, "[chebld] host call: arena %.1f ms, H2D %.1f ms (%zu B)\n", (t_h2d - t_alloc) * 1e3,
                (now_s() - t_h2d) * 1e3, used);
    }
    const double t_est = now_s();
    if (!rc) rc = logdet_device(&dop, a, b, degree, num_probes, seed, probe_block, out, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (getenv("CHEB_DEBUG")) fprintf(stderr, "[chebld] host call: estimate %.1f ms\n", (now_s() - t_est) * 1e3);
    out->elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

int cheb_bounds_btb(const cl_operator* op, double* ab_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if (op->kind != CL_OP_BTB) return fail(CL_EINVAL, "cheb_bounds_btb needs a CL_OP_BTB operator");
    if (!ab_out) return fail(CL_EINVAL, "ab_out is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf buf;
    CL_CUDA(cudaMalloc(&buf.p, 3 * sizeof(unsigned long long)));
    unsigned long long init[3] = {~0ull, 0ull, 0ull};
    CL_CUDA(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const int64_t d = op->A.n_rows;
    int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    bounds_btb_kernel<<<grid, kThreads, 0, st>>>(d, op->A.row_ptr, op->A.col_idx, op->A.val,
                                                  op->At.row_ptr, op->At.col_idx, op->At.val,
                                                  (unsigned long long*)buf.p);
    g_launches++;
    CL_CUDA(cudaGetLastError());
    unsigned long long h[3];
    CL_CUDA(cudaMemcpyAsync(h, buf.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    auto unkey = [](unsigned long long k) {
        unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        double x;
        memcpy(&x, &b, sizeof(x));
        return x;
    };
    const double smin = unkey(h[0]), rmax = unkey(h[1]), cmax = unkey(h[2]);
    if (!(smin > 0.0))
        return fail(CL_EINVAL, "Johnson lower bound on sigma_min is not positive (%g); supply [a,b]", smin);
    ab_out[0] = smin * smin;
    ab_out[1] = cmax * rmax;
    return CL_OK;
}

int cheb_probes(int64_t d, uint64_t seed, int64_t probe_begin, int32_t probe_block,
                double* v_out, void* stream) {
    if (d < 1 || d >= (int64_t(1) << 31)) return fail(CL_EDIM, "bad d");
    if (probe_begin < 0 || !valid_k(probe_block) || !v_out) return fail(CL_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    cl_operator op{};
    op.kind = CL_OP_CSR;
    op.A.n_rows = op.A.n_cols = d;
    const int sms = sm_count();
    const Layout L = plan(d, 0, probe_block, CL_OP_CSR, sms);
    DevBuf ws, mu;
    CL_CUDA(cudaMalloc(&ws.p, L.total));
    CL_CUDA(cudaMalloc(&mu.p, sizeof(double) * probe_block));
    CL_CUDA(cudaMemsetAsync((char*)ws.p + L.ticket, 0, 256, st));
    int rc;
    switch (probe_block) {
        case 8: rc = run_block<8, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 8, (char*)ws.p, L, (double*)mu.p, 1, st, sms, FusionPlan()); break;
        case 16: rc = run_block<16, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 16, (char*)ws.p, L, (double*)mu.p, 1, st, sms, FusionPlan()); break;
        case 32: rc = run_block<32, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 32, (char*)ws.p, L, (double*)mu.p, 1, st, sms, FusionPlan()); break;
        case 64: rc = run_block<64, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 64, (char*)ws.p, L, (double*)mu.p, 1, st, sms, FusionPlan()); break;
        default: rc = run_block<128, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 128, (char*)ws.p, L, (double*)mu.p, 1, st, sms, FusionPlan()); break;
    }
    if (rc) return rc;
    CL_CUDA(cudaMemcpyAsync(v_out, (char*)ws.p + L.w0, sizeof(double) * d * probe_block,
                            cudaMemcpyDeviceToDevice, st));
    CL_CUDA(cudaStreamSynchronize(st));
    return CL_OK;
}

}  // extern "C"
